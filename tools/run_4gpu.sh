#!/bin/bash
# N-GPU bench lines for config 3 and config 5 (split decomposition) + archive check
N=${1:-4}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29521 tools/check_distributed.py > gpurun_out/check${N}.log 2>&1
echo check=$?; grep -E "identical" gpurun_out/check${N}.log
for c in ${CFGS:-cfg3 cfg5}; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus $N --config $c --no-clocks > gpurun_out/bench${N}_$c.log 2>&1
echo $c=$?
python -c "import json;d=json.loads(open('gpurun_out/bench${N}_$c.log').read().strip().splitlines()[-1]);print('$c', d['ms_per_step'], d['value'], (d.get('e2e') or {}).get('seconds_per_step'));[print(r) for r in d['stage_ms_by_rank']]"
done
