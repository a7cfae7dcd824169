# x end taps by warp shuffle (ids 55-58) vs the same shapes with LDS: parity first, then sweeps
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.mem,power.limit,temperature.gpu --format=csv > gpurun_out/gpu_xsh.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "all_variants or ragged_nx or zchunking" > gpurun_out/pytest_xsh.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_xsh.log
if grep -q "pytest rc=0" gpurun_out/pytest_xsh.log; then
timeout 900 python tools/sweep.py --config 4 --ni 100 --repeat 3 --tiles 28,55,31,56,35,57 > gpurun_out/sweep_c4_xsh.log 2>&1
timeout 600 python tools/sweep.py --config 3 --ni 300 --repeat 3 --tiles 17,58,28,55 > gpurun_out/sweep_c3_xsh.log 2>&1
timeout 600 python tools/sweep.py --config 5 --ni 200 --repeat 2 --tiles 31,56,28,55 > gpurun_out/sweep_c5_xsh.log 2>&1
B="python bench.py --ncu --steps 1 --warmup 0 --nsteps 3 --config 4 --tile 55"
timeout 600 $B > gpurun_out/ncu_plain_c4_t55.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream -s 1 -c 1 -o gpurun_out/prof_xsh_c4_t55 $B > gpurun_out/ncu_xsh_c4_t55.log 2>&1
fi
echo done
