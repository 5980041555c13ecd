#!/bin/bash
# ncu --set full of k_stage1 (current build), after a plain run
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/$1; mkdir -p $O
ARGS="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks --no-train"
python bench.py $ARGS > $O/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage1 -c 1 -o $O/stage1 python bench.py $ARGS > $O/ncu_stage1.log 2>&1
echo "rc=$?" >> $O/plain.log
