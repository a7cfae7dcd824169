# PDL on/off: parity test + per-config timing with the autotuned tile fixed per config
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-pdl}
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "pdl or graph_and_direct or multislab" > gpurun_out/pytest_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.log
for c in "2 23" "3 17" "4 28"; do set -- $c
  for p in 0 1 0 1; do
    timeout 300 python bench.py --config $1 --tile $2 --pdl $p --no-cpu --no-e2e --steps 5 > gpurun_out/bench_${TAG}_c$1_p$p.log 2>&1
    grep '^{' gpurun_out/bench_${TAG}_c$1_p$p.log >> gpurun_out/pdl_$TAG.jsonl
  done
done
echo done
