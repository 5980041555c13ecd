"""Diagnostics: DEFLATE phase cycles and stream-length distribution at cfg3."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import bench
from paper_2212_10733_b200 import engine, pipeline, distributed

dev = torch.device('cuda', 0)
spec = bench.CONFIGS['cfg3']
ds = bench.corpus(spec['P'], spec['N'])
models = bench.load_models(spec['golden'])
cfg = bench.pipeline_config(1e-3)
rp = distributed.plan(ds.n_planes, ds.n_nodes, cfg.shards, cfg.mode, 0, 1)
f0 = pipeline.upload_f0(ds.data, dev, (0, ds.n_nodes))
dgrid = engine.DeviceGrid(ds.grid, dev, cfg.latent_dim)
works = engine.shard_layout(rp.shards, models, ds.n_nodes, ds.grid.rows, ds.grid.cols)
out = engine.compress_device(f0, works, dgrid, cfg)
torch.cuda.synchronize()
engine.DEFLATE_PROF = torch.zeros(12, dtype=torch.int64, device=dev)
out = engine.compress_device(f0, works, dgrid, cfg)
torch.cuda.synchronize()
p = engine.DEFLATE_PROF.cpu().numpy().astype(np.float64)
names = ['load+adler', 'chains', 'p4', 'match loop', 'longest_match', 'trees+emit', 'n_calls', 'streams', 'bytes', 'symbols', 'rounds', 'cands']
for n_, v in zip(names, p):
    print(f"{n_:14s} {v:16.0f}  per-stream {v / max(p[7], 1):12.1f}")
ws = engine.Workspace.get(dev)
vlen = ws.bufs['vlen']
n_sel = int(p[7])
print('streams', n_sel)
engine.DEFLATE_PROF = None
# stream length histogram
vl = out.dev['vlen'][:] if hasattr(out, 'dev') and 'vlen' in out.dev else None
vl = ws.bufs['vlen'][:8 * n_sel].view(torch.int64)[:n_sel].cpu().numpy()
zl = ws.bufs['zlen'][:8 * n_sel].view(torch.int64)[:n_sel].cpu().numpy()
print('varint len: mean %.1f p50 %d p90 %d p99 %d max %d' % (vl.mean(), np.percentile(vl, 50), np.percentile(vl, 90), np.percentile(vl, 99), vl.max()))
print('zlib len  : mean %.1f ratio %.3f' % (zl.mean(), zl.sum() / vl.sum()))
tiers = (0,) + engine.DEFLATE_TIERS
for lo, hi in zip(tiers, tiers[1:]):
    print('tier', lo, hi, int(((vl > lo) & (vl <= hi)).sum()))
# per tier timing (isolated)
sms = torch.cuda.get_device_properties(dev).multi_processor_count
print('sms', sms)
