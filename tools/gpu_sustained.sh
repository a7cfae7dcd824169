# every single-step variant on C4 / C5 / C3 in sustained (long, interleaved) windows under the
# board's power cap: does the tuner's short-window lattice + refinement find the sustained best?
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=1,2,3,4,5,6,7,8,9,10,11,12,13,16,17,18,19,20,21,22,23,24,25,26,27,28,29,30,31,32,33,34,35,36,48,49,51,52,53,54
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.mem,power.limit,temperature.gpu --format=csv > gpurun_out/gpu_sust.txt
timeout 900 python tools/sweep.py --config 4 --ni 100 --repeat 3 --tiles $T > gpurun_out/sweep_c4_sust.log 2>&1
timeout 600 python tools/sweep.py --config 5 --ni 300 --repeat 2 --tiles $T > gpurun_out/sweep_c5_sust.log 2>&1
timeout 600 python tools/sweep.py --config 3 --ni 600 --repeat 2 --tiles $T > gpurun_out/sweep_c3_sust.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "bench_line" > gpurun_out/pytest_benchline.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_benchline.log
echo done
