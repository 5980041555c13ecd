#!/bin/bash
# GPU tests + A/B of stored reconstructions (probes and the residual projection)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/recon3; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for i in 1 2; do
  for r in 1 0; do
    MLK_PROBE_RECON=$r timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/b_${r}_$i.log 2>&1
  done
done
