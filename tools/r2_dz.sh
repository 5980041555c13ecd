#!/bin/bash
# DEFLATE iteration: byte-parity tests, per-phase cycle profile, bench
#   tools/r2_dz.sh <tag> [pytest -k expr]
cd "$GRAFT_REPO_ROOT" || exit 1
TAG=$1; KEXPR=${2:-"zlib or benchmark_configs or compress_matches"}
O=gpurun_out/$TAG
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$KEXPR" > $O/gputests.log 2>&1
echo "rc=$?" >> $O/gputests.log
timeout 600 python tools/deflate_prof.py > $O/deflate_prof.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench.log 2>&1
echo "rc=$?" >> $O/bench.log
