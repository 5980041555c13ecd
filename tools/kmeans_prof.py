"""Phase clocks of one k-means CTA (config 3, whole shards) after a device step."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2212_10733_b200 import engine, pipeline, _lib
from paper_2212_10733_b200.decomp import partition
dev = torch.device("cuda", 0)
spec = bench.CONFIGS["cfg3"]
ds = bench.corpus(spec["P"], spec["N"])
models = bench.load_models("cfg3")
cfg = bench.pipeline_config(1e-3)
shards = partition(ds.n_planes, ds.n_nodes, 8, "col")
f0 = pipeline.upload_f0(ds.data, dev)
dg = engine.DeviceGrid(ds.grid, dev)
works = engine.shard_layout(shards, models, ds.n_nodes, 39, 39)
for _ in range(2):
    out = engine.compress_device(f0, works, dg, cfg)
buf = (ctypes.c_int64 * 12)()
_lib.call("mlk_kmeans_prof", ctypes.addressof(buf))
ghz = 1.965
print("kmeans CTA0 cycles: load+distinct %d (%.1f us)  seeding %d (%.1f us)  lloyd %d (%.1f us)  sweeps %d"
      % (buf[0], buf[0] / ghz / 1e3, buf[1], buf[1] / ghz / 1e3, buf[2], buf[2] / ghz / 1e3, buf[3]))
names = ["seed: pairwise d2 sum", "seed: scan + choice", "lloyd: count + offsets",
         "lloyd: scatter", "lloyd: pairwise means", "lloyd: reseed + nearest"]
for k, nm in enumerate(names):
    print(f"  {nm:26s} {buf[4 + k] / ghz / 1e3:8.1f} us")
ki = out.host("kinfo").reshape(-1, 4)
print("sweeps per (shard, dim):", ki[:, 2].tolist())
print("choice(p) fallbacks per (shard, dim):", ki[:, 3].tolist())
