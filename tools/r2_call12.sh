#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r2k
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gputests.log 2>&1
echo "rc=$?" >> $O/gputests.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.log 2>&1
echo "rc=$?" >> $O/bench.log
tools/r2_deflate.sh r2k
