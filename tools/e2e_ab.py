"""A/B of compress() options (pinned config-3 f0), interleaved to cancel drift."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
import bench
from paper_2212_10733_b200 import TimestepState, compress, hostio, pipeline, FDataset

spec = bench.CONFIGS['cfg3']
ds = bench.corpus(spec['P'], spec['N'])
pin = hostio.pinned_empty(ds.data.shape); pin[...] = ds.data
dsp = FDataset(grid=ds.grid, data=pin, timestep=ds.timestep)
st = TimestepState(models=bench.load_models(spec['golden']), timestep_index=1)
cfg = bench.pipeline_config(1e-3)
combos = [(p, h) for p in (True, False) for h in (True, False)]
ts = {c: [] for c in combos}
for c in combos * 2:
    pipeline.PLANE_STAGE1, pipeline.HOST_EXCEPTIONS = c
    compress(dsp, cfg, st)
for rep in range(6):
    for c in combos:
        pipeline.PLANE_STAGE1, pipeline.HOST_EXCEPTIONS = c
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        arc, _, _ = compress(dsp, cfg, st)
        ts[c].append(time.perf_counter() - t0)
        del arc
for c in combos:
    print(f"plane_stage1={c[0]!s:5} host_exceptions={c[1]!s:5} median {1e3*np.median(ts[c]):7.2f} ms"
          f"  min {1e3*min(ts[c]):7.2f}")
