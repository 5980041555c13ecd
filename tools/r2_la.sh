#!/bin/bash
# search lookahead depth / levels per launch with the stored-reconstruction probes
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/la; mkdir -p $O
for cfg in "8 2" "12 3" "12 2" "9 3" "8 2" "12 3"; do
  set -- $cfg
  tag=${1}_${2}
  MLK_LOOKAHEAD=$1 MLK_PASS_LEVELS=$2 timeout 300 python tools/eb_trace.py >> $O/eb_$tag.log 2>&1
  MLK_LOOKAHEAD=$1 MLK_PASS_LEVELS=$2 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> $O/b_$tag.log 2>&1
done
