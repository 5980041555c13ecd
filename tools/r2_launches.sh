#!/bin/bash
# ncu launch list (per-launch gpu__time_duration, serialised) of bench steps
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/$1
mkdir -p $O
ARGS="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks --no-train"
python bench.py $ARGS > $O/plain_l.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches.csv python bench.py $ARGS > $O/ncu_l.log 2>&1
echo "ncu rc=$?" >> $O/ncu_l.log
