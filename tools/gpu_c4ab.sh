cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.mem,power.limit,temperature.gpu --format=csv > gpurun_out/gpu_c4ab.txt
timeout 600 python tools/sweep.py --config 4 --ni 100 --repeat 6 --tiles 35,48 > gpurun_out/sweep_c4ab.log 2>&1
for t in 35 48 -1 35 48; do timeout 600 python bench.py --no-cpu --no-e2e --steps 10 --tile $t > gpurun_out/bench_c4ab_t$t.log 2>&1; grep '^{' gpurun_out/bench_c4ab_t$t.log >> gpurun_out/bench_c4ab.jsonl; done
echo done
