#!/bin/bash
# round-2 GPU call 1: parity tests, FP64 peak, bench (both arms), k_project ncu
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r2a
mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
lscpu > $O/lscpu.txt 2>&1
tools/fp64_peak > $O/fp64_peak.json 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gputests.log 2>&1
echo "rc=$?" >> $O/gputests.log
timeout 600 python bench.py --steps 5 --warmup 3 > $O/bench.log 2>&1
echo "rc=$?" >> $O/bench.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/ref.log 2>&1
echo "rc=$?" >> $O/ref.log
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks --no-train > $O/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_project -c 1 \
  --metrics sm__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed_pipe_fp64.sum,sm__inst_executed.sum \
  -o $O/project python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks --no-train > $O/ncu.log 2>&1
echo "ncu rc=$?" >> $O/ncu.log
