cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S="python tools/sweep.py --config 4 --ni 2 --tiles 26,13 --zchunk 0,1024,512,256,128"
$S > gpurun_out/zc_plain.log 2>&1 && \
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/zc_ncu.csv $S > gpurun_out/zc_ncu.log 2>&1
python tools/sweep.py --config 4 --ni 10 --tiles 26,13 --zchunk 0,1024,512,256,128 --repeat 2 > gpurun_out/zc_sweep.log 2>&1
echo done
