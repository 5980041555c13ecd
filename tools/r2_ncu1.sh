#!/bin/bash
# one ncu --set full capture (with source) of the first launch matching a regex
#   tools/r2_ncu1.sh <tag> <kernel regex> [launch skip]
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/$1
mkdir -p $O
ARGS="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks --no-train"
python bench.py $ARGS > $O/plain_n.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s ${3:-0} -c 1 \
  -o $O/k python bench.py $ARGS > $O/ncu_n.log 2>&1
echo "ncu rc=$?" >> $O/ncu_n.log
