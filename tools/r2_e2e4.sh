#!/bin/bash
# compress_distributed phase trace at N = 4 (MLK_TRACE=1: synchronised phases)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/$1
mkdir -p $O
MLK_TRACE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29588 bench.py --gpus 4 --steps 3 --warmup 3 --no-train > $O/e2e4.log 2>&1
