#!/bin/bash
# A/B of dynamic DEFLATE tier balancing at N=1 and N=4 (config 3)
for dyn in 1 0; do
  MLK_DEFLATE_DYNAMIC=$dyn timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-clocks --steps 10 > gpurun_out/d1.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/d1.log').read().strip().splitlines()[-1]);print('dyn $dyn N=1', round(d['ms_per_step'],3), 'deflate', round(d['stage_ms']['deflate'],3))"
  MLK_DEFLATE_DYNAMIC=$dyn timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 --no-e2e --no-clocks --steps 10 > gpurun_out/d4.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/d4.log').read().strip().splitlines()[-1]);print('dyn $dyn N=4', round(d['ms_per_step'],3), 'deflate', [r['deflate'] for r in d['stage_ms_by_rank']])"
done
