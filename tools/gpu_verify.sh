# re-verify a restored tree: smoke, gpu tests, default bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-v}
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.mem,power.limit --format=csv > gpurun_out/gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
echo done
