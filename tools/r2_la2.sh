#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/$1; mkdir -p $O
for la in 12 10 11 12 10 11; do
  MLK_LOOKAHEAD=$la timeout 300 python tools/eb_trace.py >> $O/eb_$la.log 2>&1
done
