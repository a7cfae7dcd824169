cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "batch" > gpurun_out/pytest_shots.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_shots.log
python tools/sweep.py --config 2 --ni 20 --shots 16 --tiles 13,10,7,1 --shot-order 1,2 --repeat 2 > gpurun_out/sweep_c2s16_order.log 2>&1
python tools/sweep.py --config 3 --ni 10 --shots 4 --tiles 13,10,7 --shot-order 1,2 --repeat 2 > gpurun_out/sweep_c3s4_order.log 2>&1
python tools/sweep.py --config 1 --ni 40 --shots 64 --tiles 13,10,7 --shot-order 1,2 --repeat 2 > gpurun_out/sweep_c1s64_order.log 2>&1
echo done
