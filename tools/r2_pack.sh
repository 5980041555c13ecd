#!/bin/bash
# GPU tests + the pack-stage host timeline + bench
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/$1; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python tools/eb_trace.py > $O/eb.log 2>&1
for i in 1 2 3; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/b_$i.log 2>&1; done
