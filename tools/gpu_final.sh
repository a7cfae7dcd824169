# final validation of the committed build: smoke, the full -m gpu suite, the default bench line,
# the reference arm, and the ncu launch list of the bench's timed region (NVTX range bench_timed)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r02i}
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.mem,power.limit,temperature.gpu --format=csv > gpurun_out/gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py --steps 20 > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref_$TAG.log
L="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e"
$L > gpurun_out/launch_plain_$TAG.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "bench_timed/" --csv --log-file gpurun_out/launches_c4_${TAG}_timed.csv $L > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launch rc=$?" >> gpurun_out/ncu_launch_$TAG.log
echo done
