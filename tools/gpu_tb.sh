# two-step (k_tb2) check: parity tests, then C4 timing vs the single-step default
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-tb}
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "tb2 or all_variants" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
for t in ${TILES:-35 37 38 39 40}; do
  timeout 300 python bench.py --tile $t --no-cpu --no-e2e --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_t$t.log 2>&1; echo "rc=$?" >> gpurun_out/bench_${TAG}_t$t.log
done
echo done
