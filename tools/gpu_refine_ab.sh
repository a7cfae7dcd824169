# A/B of the tuner refinement on one box: --tune-refine 0 vs 6, alternated, C3 / C2 / C4; then
# ncu --set full of C3's sustained winner (stream64x14k8d4u4, tile 8)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.mem,power.limit,temperature.gpu --format=csv > gpurun_out/gpu_rab.txt
for c in 3 2 4; do for r in 0 6 0 6; do
  timeout 600 python bench.py --config $c --no-cpu --no-e2e --tune-refine $r > gpurun_out/rab_c${c}_r$r.log 2>&1
  grep '^{' gpurun_out/rab_c${c}_r$r.log | tail -1 | sed "s/^/c$c r$r /" >> gpurun_out/rab.jsonl
done; done
B="python bench.py --ncu --steps 1 --warmup 0 --nsteps 3 --config 3 --tile 8"
timeout 600 $B > gpurun_out/ncu_plain_c3_t8.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream -s 1 -c 1 -o gpurun_out/prof_final_c3_t8 $B > gpurun_out/ncu_final_c3_t8.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_final_c3_t8.log
echo done
