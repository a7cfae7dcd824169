# ncu --set full of one k_tb2 band launch (variant $T) on C4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-tbn}
T=${T:-39}
B="python bench.py --ncu --steps 1 --warmup 0 --nsteps 4 --tile $T"
timeout 300 $B > gpurun_out/ncu_plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tb2 -s 3 -c 1 -o gpurun_out/prof_$TAG $B > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full_$TAG.log
for t in ${TILES:-}; do
  timeout 300 python bench.py --tile $t --no-cpu --no-e2e --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_t$t.log 2>&1; echo "rc=$?" >> gpurun_out/bench_${TAG}_t$t.log
done
echo done
