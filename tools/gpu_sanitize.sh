cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TOOL=${TOOL:-memcheck}
python tools/sanitize_case.py > gpurun_out/san_plain_$TOOL.log 2>&1 && \
timeout 1200 compute-sanitizer --tool $TOOL --print-limit 50 python tools/sanitize_case.py > gpurun_out/sanitizer_$TOOL.log 2>&1
echo "rc=$?" >> gpurun_out/sanitizer_$TOOL.log
