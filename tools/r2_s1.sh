#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/$1; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "compress_matches or benchmark_configs_match" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for i in 1 2 3; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/b_$i.log 2>&1; done
