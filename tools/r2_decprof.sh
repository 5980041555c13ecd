#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/$1
mkdir -p $O
timeout 900 python -m pytest tests/test_multi_gpu.py -m gpu -x -q -p no:cacheprovider -k "decompress or distributed" > $O/multi_tests.log 2>&1
echo "rc=$?" >> $O/multi_tests.log
timeout 600 python tools/dec_prof.py > $O/dec_prof_1.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29533 tools/dec_prof.py > $O/dec_prof_4.log 2>&1
