#!/bin/bash
# device step vs bisection lookahead / levels per probe launch (config 3, 1 GPU)
for cfg in "12 2" "12 3" "8 2"; do
  set -- $cfg
  MLK_LOOKAHEAD=$1 MLK_PASS_LEVELS=$2 timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-clocks --steps 10 > gpurun_out/sw.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/sw.log').read().strip().splitlines()[-1]);print('lookahead $1 pass $2', round(d['ms_per_step'],3), 'eb_search', round(d['stage_ms']['eb_search'],3), 'rounds', d['probe_rounds'])"
done
