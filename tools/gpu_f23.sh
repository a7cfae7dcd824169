cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-x}
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "batch or autotune or variants or multislab or device_pointer" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
for a in "--config 2" "--config 2 --shots 16" "--config 1 --shots 64" "--config 3 --shots 4" "--config 1"; do
  echo "== $a" >> gpurun_out/bench_$TAG.log
  timeout 600 python bench.py $a --no-cpu --no-e2e >> gpurun_out/bench_$TAG.log 2>&1
done
echo done
