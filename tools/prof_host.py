"""cProfile of compress_device's host side on a small step (config 2: one
plane, 16,395 histograms = the per-rank size of config 3 at 8 GPUs)."""
import sys, cProfile, pstats
sys.path.insert(0, '.')
import torch
import bench
from paper_2212_10733_b200 import engine, pipeline
from paper_2212_10733_b200.decomp import partition
spec = bench.CONFIGS['cfg2']
ds = bench.corpus(spec['P'], spec['N'])
models = bench.load_models(spec['golden'])
cfg = bench.pipeline_config(1e-3)
dev = torch.device('cuda', 0)
f0 = pipeline.upload_f0(ds.data, dev)
dg = engine.DeviceGrid(ds.grid, dev, 4)
works = engine.shard_layout(partition(1, spec['N'], 8, 'col'), models, spec['N'], 39, 39)
for _ in range(3):
    engine.compress_device(f0, works, dg, cfg)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    engine.compress_device(f0, works, dg, cfg)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats('tottime').print_stats(30)
