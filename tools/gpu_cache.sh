cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S="python tools/sweep.py --config 4 --ni 10 --tiles 1,2,8 --cache 0x41,0x00,0x42,0x21,0x81,0x45,0x49,0x4d,0x04"
$S > gpurun_out/cache_sweep.log 2>&1
S2="python tools/sweep.py --config 4 --ni 2 --tiles 1,2,8 --cache 0x41,0x00,0x42,0x45,0x49"
$S2 > gpurun_out/cache_sweep2_plain.log 2>&1 && \
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/cache_ncu.csv $S2 > gpurun_out/cache_ncu.log 2>&1
echo done
