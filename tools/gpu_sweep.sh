cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "variants or zchunk or graph or multislab or c1_full or one_step_random or device_pointer" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
timeout 600 python tools/sweep.py --config 4 --ni 10 > gpurun_out/sweep_c4.log 2>&1
timeout 600 python tools/sweep.py --config 3 --ni 20 > gpurun_out/sweep_c3.log 2>&1
echo done
