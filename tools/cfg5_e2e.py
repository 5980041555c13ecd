"""configs[4] end to end through compress(): 64 planes x 16,395 nodes
(1,049,280 histograms, 12.8 GB) generated on the device, copied once into
page-locked host memory, then compress(ds, cfg, state) timed with the upload
streamed in shard groups (pipeline.PIPELINE_GROUPS = 1, 2, 4: group g + 1's
H2D under group g's compute).  The archives of every grouping must be
byte-identical."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2212_10733_b200 import FDataset, TimestepState, compress, hostio, pipeline

dev = torch.device("cuda", 0)
spec = bench.CONFIGS["cfg5"]
dc = bench.DeviceCorpus(spec["P"], spec["N"])
f0 = dc.device_planes(dev, 0, spec["P"])
D = 39 * 39
host = hostio.pinned_empty((spec["P"], spec["N"], 39, 39))
host.reshape(-1)[:] = f0[:spec["P"] * spec["N"] * D].cpu().numpy()
del f0
torch.cuda.empty_cache()
ds = FDataset._trusted(dc.grid, host, 0)
models = bench.load_models(spec["golden"])
cfg = bench.pipeline_config(1e-3)
st = TimestepState(models=models, timestep_index=1)
n = spec["P"] * spec["N"]
ref = None
for groups in (1, 2, 4):
    pipeline.PIPELINE_GROUPS = groups
    arc, _, _ = compress(ds, cfg, st)  # warm-up (workspaces, staging)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        arc, rep, _ = compress(ds, cfg, st)
        ts.append(time.perf_counter() - t0)
    same = ref is None or arc == ref
    ref = ref if ref is not None else arc
    t = min(ts)
    print(f"groups {groups}: {1e3 * t:.1f} ms per call = {n / t / 1e6:.2f} M hist/s "
          f"({n * D * 8 / t / 1e9:.1f} GB/s of f0), archive {len(arc)} B, identical {same}",
          flush=True)
