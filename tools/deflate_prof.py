"""Phase breakdown of the warp DEFLATE kernel on real residual streams (cfg3 tau=1e-3)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2212_10733_b200 import engine, pipeline
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
engine.compress_device(f0, works, dg, cfg)
prof = torch.zeros(16, dtype=torch.int64, device=dev)
engine.DEFLATE_PROF = prof
torch.cuda.synchronize(); t0 = time.perf_counter()
engine.compress_device(f0, works, dg, cfg)
torch.cuda.synchronize(); print("step", time.perf_counter() - t0)
p = prof.cpu().numpy().astype(float); n = p[7]
names = ["load+adler", "prev build (sort)", "p1 tail", "match loop", "  of which longest_match", "trees+emit"]
for i, nm in enumerate(names): print(f"{nm:28s} {p[i]/n:12.0f} cycles/stream")
print("calls/stream", p[6]/n, "streams", n, "bytes/stream", p[8]/n, "symbols/stream", p[9]/n,
      "match rounds/stream", p[10]/n, "candidates/stream", p[11]/n)
for i, nm in [(12, "  sort: histograms + scans"), (13, "  sort: pass 0"), (14, "  sort: pass 1")]:
    print(f"{nm:28s} {p[i]/n:12.0f} cycles/stream")
