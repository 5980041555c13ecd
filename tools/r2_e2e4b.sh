#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/$1
mkdir -p $O
timeout 900 python -m pytest tests/test_multi_gpu.py -m gpu -x -q -p no:cacheprovider > $O/multi_tests.log 2>&1
echo "rc=$?" >> $O/multi_tests.log
tools/r2_e2e4.sh $1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29591 bench.py --gpus 4 --steps 5 --warmup 3 > $O/bench_4.log 2>&1
