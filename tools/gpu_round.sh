# full GPU round check: smoke, tests, bench (all configs + reference arm), ncu --set full of the
# two top single-step variants, ncu launch list of the default bench command
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r01g}
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.mem,power.limit --format=csv > gpurun_out/gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref_$TAG.log
for c in 3 5 2 1; do timeout 600 python bench.py --config $c --no-cpu > gpurun_out/bench_c${c}_$TAG.log 2>&1; done
for T in 35 28; do
  B="python bench.py --ncu --steps 1 --warmup 0 --nsteps 3 --tile $T"
  $B > gpurun_out/ncu_plain_${TAG}_t$T.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream -s 1 -c 1 -o gpurun_out/prof_c4_${TAG}_t$T $B > gpurun_out/ncu_full_${TAG}_t$T.log 2>&1
done
L="python bench.py --steps 3 --warmup 3 --no-cpu"
$L > gpurun_out/launch_plain_$TAG.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_$TAG.csv $L > gpurun_out/ncu_launch_$TAG.log 2>&1
echo done
