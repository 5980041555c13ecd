"""Where one public-API compress() goes (config 3, pinned f0): per-phase wall
times with explicit synchronisation between phases (diagnostic only)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
import bench
from paper_2212_10733_b200 import TimestepState, compress, engine, hostio, pipeline, FDataset
from paper_2212_10733_b200.container import ArchivePreamble, archive_offsets
from paper_2212_10733_b200.decomp import partition

spec = bench.CONFIGS['cfg3']
ds = bench.corpus(spec['P'], spec['N'])
pin = hostio.pinned_empty(ds.data.shape); pin[...] = ds.data
ds = FDataset(grid=ds.grid, data=pin, timestep=ds.timestep)
models = bench.load_models(spec['golden'])
cfg = bench.pipeline_config(1e-3)
st = TimestepState(models=models, timestep_index=1)
dev = torch.device('cuda', 0)
for _ in range(2):
    compress(ds, cfg, st)
torch.cuda.synchronize()
T = {}
def tick(k, t0):
    torch.cuda.synchronize(); T.setdefault(k, []).append(time.perf_counter() - t0); return time.perf_counter()
for _ in range(4):
    t = time.perf_counter(); t_all = t
    f0 = pipeline.upload_f0(ds.data, dev); t = tick('upload', t)
    dgrid = engine.DeviceGrid(ds.grid, dev, cfg.latent_dim); t = tick('grid', t)
    shards = partition(ds.n_planes, ds.n_nodes, cfg.shards, cfg.mode)
    works = engine.shard_layout(shards, st.models, ds.n_nodes, 39, 39)
    out = engine.compress_device(f0, works, dgrid, cfg); t = tick('device', t)
    n = int(np.sum(out.blob_lens))
    stage = hostio.pinned('down0', n); stage[:n].copy_(out.blob_buf[:n], non_blocking=True); t = tick('d2h', t)
    arc = hostio.download_bytes(out.blob_buf, n, b'x' * 13000); t = tick('d2h+bytes', t)
    del arc
    t = time.perf_counter()
    arc, rep, _ = compress(ds, cfg, st); t = tick('compress_total', t)
    t = time.perf_counter()
    out.dataset_index = np.concatenate([np.arange(len(sh.members)) for sh in shards])
    pipeline.build_report(ds, arc, [out], cfg.tau, {}, 0.0); t = tick('report', t)
    del arc
for k, v in T.items():
    print(f"{k:16s} {1e3*np.median(v):8.2f} ms")
import os; print('cpus', os.cpu_count())
print(open('/sys/kernel/mm/transparent_hugepage/enabled').read())
