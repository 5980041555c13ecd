#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/$1
mkdir -p $O
timeout 600 python tools/eb_trace.py > $O/eb_trace_1.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29555 tools/eb_trace.py > $O/eb_trace_4.log 2>&1
