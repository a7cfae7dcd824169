cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-q}
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider ${K:+-k "$K"} > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
echo done
