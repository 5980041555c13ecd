#!/bin/bash
# A/B of two engine.py versions (B in tools/_ab/engine_b.py), N=1, overlap off and on
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/$1
mkdir -p $O
for v in A B A B; do
  if [ $v = B ]; then cp paper_2212_10733_b200/engine.py /tmp/engine_a.py; cp tools/_ab/engine_b.py paper_2212_10733_b200/engine.py; fi
  for ov in 0 1; do
    echo "== $v overlap=$ov" >> $O/ab.log
    MLK_PROJECT_OVERLAP=$ov timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-train --no-clocks 2>/dev/null | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['stage_ms'].items() if k in ('compact','eb_search','newton','deflate_done')})" >> $O/ab.log
  done
  if [ $v = B ]; then cp /tmp/engine_a.py paper_2212_10733_b200/engine.py; fi
done
