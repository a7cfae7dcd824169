# ncu --set full of each config's refinement winner on the final round-2 build (the bench's
# roofline.traffic source); each capture only after the same command exited 0 without ncu
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for ct in "4 28" "5 31" "3 17" "2 49"; do
  set -- $ct
  B="python bench.py --ncu --steps 1 --warmup 0 --nsteps 3 --config $1 --tile $2"
  timeout 600 $B > gpurun_out/ncu_plain_c$1_t$2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream -s 1 -c 1 \
      -o gpurun_out/prof_final_c$1_t$2 $B > gpurun_out/ncu_final_c$1_t$2.log 2>&1
  echo "c$1 t$2 rc=$?" >> gpurun_out/ncu_final_rc.log
done
echo done
