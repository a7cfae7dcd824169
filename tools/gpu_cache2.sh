cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > gpurun_out/c2_clk.txt
S="python tools/sweep.py --config 4 --ni 10 --tiles 1,8,3,5 --cache 0x41,0x141,0x241,0x341 --repeat 3"
$S > gpurun_out/cache2_sweep.log 2>&1
python tools/sweep.py --config 3 --ni 20 --tiles 1,8,3,5,2 --repeat 3 > gpurun_out/cache2_sweep_c3.log 2>&1
S2="python tools/sweep.py --config 4 --ni 2 --tiles 1,8 --cache 0x41,0x141,0x241,0x341"
$S2 > gpurun_out/cache2_plain.log 2>&1 && \
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/cache2_ncu.csv $S2 > gpurun_out/cache2_ncu.log 2>&1
echo done
