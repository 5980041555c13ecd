#!/bin/bash
# A/B of the probes reading stored reconstructions (MLK_PROBE_RECON)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/recon; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for i in 1 2; do
  for r in 1 0; do
    MLK_PROBE_RECON=$r timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/b_${r}_$i.log 2>&1
  done
done
for r in 1 0; do
  MLK_PROBE_RECON=$r timeout 300 python tools/eb_trace.py > $O/eb_$r.log 2>&1
done
