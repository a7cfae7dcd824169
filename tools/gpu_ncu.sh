cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --ncu --steps 1 --warmup 0 --nsteps 3"
$B > gpurun_out/ncu_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tiled -s 1 -c 1 -o gpurun_out/prof_c4_r01 $B > gpurun_out/ncu_full.log 2>&1
L="python bench.py --steps 3 --warmup 3"
$L > gpurun_out/launch_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_r01.csv $L > gpurun_out/ncu_launch.log 2>&1
echo done
