cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/sweep.py --config 4 --ni 10 --tiles 28,31,32,33,34,35,36,27,17 --repeat 3 > gpurun_out/sweep_c4_s6.log 2>&1
python tools/sweep.py --config 3 --ni 20 --tiles 17,29,33,34,28 --repeat 3 > gpurun_out/sweep_c3_s6.log 2>&1
echo done
