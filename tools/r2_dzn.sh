#!/bin/bash
# ncu --set full of the main DEFLATE size tier ((1024, 1600] bytes): its
# phase-1 and phase-2 launches (the 11th and 12th k_deflate_warp launches)
cd "$GRAFT_REPO_ROOT" || exit 1
TAG=$1
O=gpurun_out/$TAG
mkdir -p $O
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks --no-train > $O/plain_d.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_deflate_warp -s 10 -c 2 \
  -o $O/deflate python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks --no-train > $O/ncu_d.log 2>&1
echo "ncu rc=$?" >> $O/ncu_d.log
