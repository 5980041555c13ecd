#!/bin/bash
# Round profile evidence on one B200 (each ncu pass only after its command ran clean):
#   gpurun_out/bench_final.log  the default bench line
#   gpurun_out/launches.csv     ncu launch list of one timed step
#   gpurun_out/full_*.ncu-rep   --set full captures of one step's top kernels
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks"
timeout 600 python bench.py > gpurun_out/bench_final.log 2>&1; echo bench=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e \
  --no-cpu-baseline --no-clocks > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:'k_stage1|k_kmeans|k_project|k_probe_bins|k_pack_exc' --launch-skip 5 --launch-count 5 \
  -f -o gpurun_out/full_a $B > gpurun_out/ncu_a.log 2>&1; echo full_a=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_deflate_warp' \
  --launch-skip 7 --launch-count 7 -f -o gpurun_out/full_b $B > gpurun_out/ncu_b.log 2>&1; echo full_b=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_probe_level' \
  --launch-skip 12 --launch-count 12 -f -o gpurun_out/full_c $B > gpurun_out/ncu_c.log 2>&1; echo full_c=$?
ls -la gpurun_out/*.ncu-rep
# summaries on the box (the .ncu-rep files would exceed gpurun_out's 64 MiB)
python tools/ncu_summary.py gpurun_out/full_a.ncu-rep gpurun_out/full_b.ncu-rep \
  gpurun_out/full_c.ncu-rep --launches gpurun_out/launches.csv --out gpurun_out/prof; echo summary=$?
ncu -i gpurun_out/full_a.ncu-rep --page source --csv --print-units base > gpurun_out/src_a.csv 2>/dev/null
gzip -f gpurun_out/src_a.csv
[ $(stat -c %s gpurun_out/src_a.csv.gz) -gt 30000000 ] && rm -f gpurun_out/src_a.csv.gz
rm -f gpurun_out/full_*.ncu-rep
du -sh gpurun_out
