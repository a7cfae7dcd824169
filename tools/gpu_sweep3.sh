cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-x}
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "variants or batch or zchunk or graph or multislab or c1_full or one_step" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
python tools/sweep.py --config 4 --ni 10 --tiles 1,2,3,4,6,7,8,9,10,11,12,13 --repeat 2 > gpurun_out/sweep_c4_$TAG.log 2>&1
python tools/sweep.py --config 3 --ni 20 --tiles 1,3,4,7,8,9,10,11,12,13 --repeat 2 > gpurun_out/sweep_c3_$TAG.log 2>&1
python tools/sweep.py --config 2 --ni 20 --shots 16 --tiles 1,3,4,7,8,9,10,11,12,13 --repeat 2 > gpurun_out/sweep_c2s16_$TAG.log 2>&1
echo done
