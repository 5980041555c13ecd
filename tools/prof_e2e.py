import sys, cProfile, pstats
sys.path.insert(0, '.')
import torch
import bench
from paper_2212_10733_b200 import TimestepState, compress
spec = bench.CONFIGS['cfg3']
ds = bench.corpus(spec['P'], spec['N'])
models = bench.load_models(spec['golden'])
cfg = bench.pipeline_config(1e-3)
st = TimestepState(models=models, timestep_index=1)
compress(ds, cfg, st); compress(ds, cfg, st)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    compress(ds, cfg, st)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats('tottime').print_stats(25)
