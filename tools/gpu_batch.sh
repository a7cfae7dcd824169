cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/sweep.py --config 2 --ni 20 --shots 16 --tiles 13,10,8,16,17,18,20,22,23,24,25,26 --repeat 2 > gpurun_out/sweep_c2s16_b.log 2>&1
python tools/sweep.py --config 1 --ni 40 --shots 64 --tiles 13,10,8,16,17,18,20,22,23,24,25,26 --repeat 2 > gpurun_out/sweep_c1s64_b.log 2>&1
python tools/sweep.py --config 3 --ni 10 --shots 4 --tiles 13,10,8,16,17,18,20,22,23,24,25,26 --repeat 2 > gpurun_out/sweep_c3s4_b.log 2>&1
echo done
