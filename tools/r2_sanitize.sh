#!/bin/bash
# one compute-sanitizer tool per invocation (B200_PROFILING.md), tiny corpus
cd "$GRAFT_REPO_ROOT" || exit 1
TAG=$1; TOOL=$2
O=gpurun_out/$TAG
mkdir -p $O
python tools/sanitize_smoke.py > $O/plain_$TOOL.log 2>&1 && \
timeout 1200 compute-sanitizer --tool $TOOL --print-limit 50 --error-exitcode 9 python tools/sanitize_smoke.py > $O/sanitize_$TOOL.log 2>&1
echo "rc=$?" >> $O/sanitize_$TOOL.log
