#!/bin/bash
# e2e compress A/B by environment (N=1)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/$1; shift
mkdir -p $O
i=0
for spec in "$@"; do
  i=$((i+1))
  echo "== $spec" > $O/e2e_$i.log
  env $spec timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-train --no-clocks >> $O/e2e_$i.log 2>&1
done
