# RTM_OPT_ZDIR bit 2 (odd z-chunks sweep downward: neighbouring chunks start / end on the planes
# they share) on single-step launches, interleaved with the default (2)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-zdir4}
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.mem,power.limit,temperature.gpu --format=csv > gpurun_out/gpu_$TAG.txt
timeout 600 python tools/sweep.py --config 2 --ni 400 --repeat 3 --tiles 49,10 --zdir 0,2,4,6 > gpurun_out/sweep_c2_$TAG.log 2>&1
timeout 600 python tools/sweep.py --config 3 --ni 40 --repeat 2 --tiles 17,35,28 --zdir 2,6 > gpurun_out/sweep_c3_$TAG.log 2>&1
timeout 600 python tools/sweep.py --config 5 --ni 20 --repeat 2 --tiles 31,28 --zdir 2,6 > gpurun_out/sweep_c5_$TAG.log 2>&1
timeout 600 python tools/sweep.py --config 4 --ni 20 --repeat 2 --tiles 28,35 --zdir 2,6 > gpurun_out/sweep_c4_$TAG.log 2>&1
echo done
