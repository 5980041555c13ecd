#!/bin/bash
# bench variants by environment at N=4 (torchrun) and N=1
cd "$GRAFT_REPO_ROOT" || exit 1
TAG=$1; shift
O=gpurun_out/$TAG
mkdir -p $O
i=0
for spec in "$@"; do
  i=$((i+1))
  echo "== $spec" > $O/sweep4_$i.log
  env $spec timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
      --master-port $((29600 + i)) bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e --no-train --no-clocks >> $O/sweep4_$i.log 2>&1
  echo "== $spec" > $O/sweep1_$i.log
  env $spec timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-train --no-clocks >> $O/sweep1_$i.log 2>&1
done
