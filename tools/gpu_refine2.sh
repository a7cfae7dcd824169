# bench lines after the refinement change (6 finalists, >= 100 ms windows) + bench contract tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r02j}
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.mem,power.limit,temperature.gpu --format=csv > gpurun_out/gpu_$TAG.txt
timeout 900 python bench.py --steps 20 > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
for c in 3 5 2 1; do timeout 600 python bench.py --config $c --no-cpu > gpurun_out/bench_c${c}_$TAG.log 2>&1; done
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "bench" > gpurun_out/pytest_bench_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_bench_$TAG.log
echo done
