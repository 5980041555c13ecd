#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/$1
mkdir -p $O
timeout 1500 python tools/cfg5_e2e.py > $O/cfg5_e2e.log 2>&1
echo "rc=$?" >> $O/cfg5_e2e.log
