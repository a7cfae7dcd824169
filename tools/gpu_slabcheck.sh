cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python paper_1310_8232_b200/build.py > gpurun_out/g1_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_xproc.py -m gpu -q -p no:cacheprovider -k bench > gpurun_out/g1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g1_pytest.log
for H in 3 2; do
MASTER_ADDR=127.0.0.1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --peer --halo $H --config 3 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/g1_c3_h$H.log 2>&1; echo "rc=$?" >> gpurun_out/g1_c3_h$H.log
done
echo done
