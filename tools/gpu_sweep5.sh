cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/sweep.py --config 4 --ni 10 --tiles 13,26,17,27,28,29,30,18 --repeat 3 > gpurun_out/sweep_c4_s5.log 2>&1
python tools/sweep.py --config 3 --ni 20 --tiles 13,26,17,27,28,29,30,18 --repeat 3 > gpurun_out/sweep_c3_s5.log 2>&1
echo done
