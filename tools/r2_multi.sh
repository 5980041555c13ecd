#!/bin/bash
# multi-GPU evidence on one box: archive identity tests + bench at N = 1, 2, 4
#   gpurun --gpus 4 -- tools/r2_multi.sh <tag>
cd "$GRAFT_REPO_ROOT" || exit 1
TAG=$1
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 1500 python -m pytest tests/test_multi_gpu.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "multi or distributed or zlib or benchmark_configs" > $O/multi_tests.log 2>&1
echo "rc=$?" >> $O/multi_tests.log
NG=$(nvidia-smi -L | wc -l)
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-train > $O/bench_1.log 2>&1
for N in 2 4 8; do
  if [ "$N" -le "$NG" ]; then
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29500 + N)) bench.py --gpus $N --steps 5 --warmup 3 > $O/bench_$N.log 2>&1
    echo "rc=$?" >> $O/bench_$N.log
  fi
done
