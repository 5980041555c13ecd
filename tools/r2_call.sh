#!/bin/bash
# round-2 GPU iteration: parity tests, bench, one ncu capture of a kernel
#   tools/r2_call.sh <tag> <ncu kernel regex|none> [pytest -k expr]
cd "$GRAFT_REPO_ROOT" || exit 1
TAG=$1; KREGEX=$2; KEXPR=${3:-}
O=gpurun_out/$TAG
mkdir -p $O
if [ -n "$KEXPR" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$KEXPR" > $O/gputests.log 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gputests.log 2>&1
fi
echo "rc=$?" >> $O/gputests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench.log 2>&1
echo "rc=$?" >> $O/bench.log
if [ "$KREGEX" != "none" ]; then
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks --no-train > $O/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -c 1 \
  --metrics sm__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed.sum \
  -o $O/prof python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks --no-train > $O/ncu.log 2>&1
echo "ncu rc=$?" >> $O/ncu.log
fi
