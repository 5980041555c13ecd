#!/bin/bash
# final round-2 evidence on one 4-GPU box: every GPU test, bench at N = 1, 2, 4
#   gpurun --gpus 4 -- tools/r2_final4.sh <tag>
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/$1; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1
echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 > $O/bench_1.log 2>&1
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29500 + N)) bench.py --gpus $N --steps 5 --warmup 3 > $O/bench_$N.log 2>&1
  echo "rc=$?" >> $O/bench_$N.log
done
MLK_LOOKAHEAD=8 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29555 bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_4_la8.log 2>&1
