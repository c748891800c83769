set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/san
TOOL=$1
python scripts/sanitize_case.py > gpurun_out/san/plain_$TOOL.log 2>&1 && \
timeout 2400 /usr/local/cuda/bin/compute-sanitizer --tool $TOOL --print-limit 50 python scripts/sanitize_case.py > gpurun_out/san/$TOOL.log 2>&1
echo "rc=$?" >> gpurun_out/san/$TOOL.log
