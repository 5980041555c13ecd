#!/bin/bash
# bench variants by environment (stage times in each line)
cd "$GRAFT_REPO_ROOT" || exit 1
TAG=$1; shift
O=gpurun_out/$TAG
mkdir -p $O
i=0
for spec in "$@"; do
  i=$((i+1))
  echo "== $spec" > $O/sweep_$i.log
  env $spec timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-train --no-clocks >> $O/sweep_$i.log 2>&1
done
