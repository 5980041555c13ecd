#!/bin/bash
# DEFLATE evidence: per-phase cycle breakdown + one ncu --set full capture of
# the main size tier ((1024, 1600] bytes, the 6th k_deflate_warp launch of a step)
cd "$GRAFT_REPO_ROOT" || exit 1
TAG=$1
O=gpurun_out/$TAG
mkdir -p $O
timeout 600 python tools/deflate_prof.py > $O/deflate_prof.log 2>&1
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks --no-train > $O/plain_d.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_deflate_warp -s 0 -c 14 \
  -o $O/deflate python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks --no-train > $O/ncu_d.log 2>&1
echo "ncu rc=$?" >> $O/ncu_d.log
