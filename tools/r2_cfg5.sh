#!/bin/bash
# configs[4] (64 planes, device-generated f0) at N = 1, 2, 4
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/$1
mkdir -p $O
NG=$(nvidia-smi -L | wc -l)
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline > $O/cfg5_1.log 2>&1
for N in 2 4 8; do
  if [ "$N" -le "$NG" ]; then
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29700 + N)) bench.py --config cfg5 --gpus $N --steps 3 --warmup 3 > $O/cfg5_$N.log 2>&1
  fi
done
