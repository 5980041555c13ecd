#!/bin/bash
# one bench line (N=1) into gpurun_out/<tag>/bench.log
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/$1
mkdir -p $O
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench.log 2>&1
echo "rc=$?" >> $O/bench.log
