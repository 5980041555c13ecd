#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/r2n
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 tools/debug_ddec.py > gpurun_out/r2n/ddec.log 2>&1
echo "rc=$?" >> gpurun_out/r2n/ddec.log
