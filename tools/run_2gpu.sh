#!/bin/bash
# 2-GPU checks: archive identity of compress_distributed vs compress(), bench at N=2
N=${1:-2}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 tools/check_distributed.py > gpurun_out/check${N}.log 2>&1
echo check=$?; grep -E "identical|ratio|qoi|Error" gpurun_out/check${N}.log | head
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N --no-clocks > gpurun_out/bench${N}.log 2>&1
echo bench=$?; tail -c 1500 gpurun_out/bench${N}.log
