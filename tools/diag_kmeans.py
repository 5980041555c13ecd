import sys
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
print(out.dev['kinfo'].cpu().numpy().reshape(-1, 4))
