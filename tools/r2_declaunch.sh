#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/$1
mkdir -p $O
timeout 600 python tools/dec_prof.py > $O/dec_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/dec_launches.csv python tools/dec_prof.py > $O/ncu_dl.log 2>&1
echo "rc=$?" >> $O/ncu_dl.log
