cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S="python tools/sweep.py --config 4 --ni 2 --tiles 26,13 --cache 0x41,0x441,0x445,0x45"
$S > gpurun_out/cm_plain.log 2>&1 && \
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cm_ncu.csv $S > gpurun_out/cm_ncu.log 2>&1
python tools/sweep.py --config 4 --ni 10 --tiles 26,13 --cache 0x41,0x441,0x445,0x45 --repeat 2 > gpurun_out/cm_sweep.log 2>&1
python tools/sweep.py --config 3 --ni 20 --tiles 26,13,17 --cache 0x41,0x441,0x445 --repeat 2 > gpurun_out/cm_sweep3.log 2>&1
echo done
