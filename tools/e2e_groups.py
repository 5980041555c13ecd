"""compress() wall time (pinned config-3 f0) vs the shard-group pipelining depth."""
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
models = bench.load_models(spec['golden'])
cfg = bench.pipeline_config(1e-3)
st = TimestepState(models=models, timestep_index=1)
ref = None
for G in (1, 2, (1, 3, 4), 4, 2):
    pipeline.PIPELINE_GROUPS = G
    for name, d in (("pinned", dsp),) + ((("pageable", ds),) if G in (1, 2) else ()):
        arc, rep, _ = compress(d, cfg, st)
        if ref is None:
            ref = arc
        assert arc == ref, "archive depends on grouping"
        torch.cuda.synchronize()
        ts = []
        for _ in range(4):
            t0 = time.perf_counter()
            arc, rep, _ = compress(d, cfg, st)
            ts.append(time.perf_counter() - t0)
            del arc
        print(f"groups {G} {name:8s} median {1e3*np.median(ts):7.2f} ms  min {1e3*min(ts):7.2f}",
              {k: round(1e3 * v['sum'], 2) for k, v in rep.stage_timings.items()}, flush=True)
