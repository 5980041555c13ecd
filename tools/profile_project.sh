#!/bin/bash
# one --set full capture of k_project with the CUDA-source view summarised on the box
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_project|k_stage1' \
  --launch-skip 2 --launch-count 2 -f -o gpurun_out/proj $B > gpurun_out/ncu_p.log 2>&1; echo cap=$?
ncu -i gpurun_out/proj.ncu-rep --page source --csv --print-source cuda --print-units base > gpurun_out/proj_src.csv 2>gpurun_out/proj_src.err
echo src=$?; ls -la gpurun_out/proj_src.csv; head -c 600 gpurun_out/proj_src.err
gzip -f gpurun_out/proj_src.csv; rm -f gpurun_out/proj.ncu-rep; du -sh gpurun_out
