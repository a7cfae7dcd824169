cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S="python tools/sweep.py --config 4 --ni 2 --tiles 35,28 --cache 0x41,0x441,0x445,0x45,0x40"
$S > gpurun_out/cm2_plain.log 2>&1 && \
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cm2_ncu.csv $S > gpurun_out/cm2_ncu.log 2>&1
python tools/sweep.py --config 4 --ni 10 --tiles 35,28,32 --cache 0x41,0x441,0x445,0x45,0x40 --repeat 3 > gpurun_out/cm2_sweep.log 2>&1
echo done
