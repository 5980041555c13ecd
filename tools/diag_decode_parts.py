import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import bench
from paper_2212_10733_b200 import engine, hostio, _lib, TimestepState, compress, decompress

spec = bench.CONFIGS['cfg3']
ds = bench.corpus(spec['P'], spec['N'])
models = bench.load_models(spec['golden'])
cfg = bench.pipeline_config(1e-3)
arc, _, _ = compress(ds, cfg, TimestepState(models=models, timestep_index=1))
dev = torch.device('cuda', 0)
decompress(arc)
# wrap call() and upload_bytes with sync timers
T = {}
orig_call = _lib.call
def timed_call(name, *a, **k):
    torch.cuda.synchronize(); t = time.perf_counter()
    orig_call(name, *a, **k)
    torch.cuda.synchronize(); T[name] = T.get(name, 0) + time.perf_counter() - t
engine.call = timed_call
orig_up = hostio.upload_bytes
def timed_up(*a):
    torch.cuda.synchronize(); t = time.perf_counter(); r = orig_up(*a); torch.cuda.synchronize()
    T['upload_bytes'] = T.get('upload_bytes', 0) + time.perf_counter() - t; return r
hostio.upload_bytes = timed_up
for rep in range(2):
    T.clear()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    engine.decode_archive(arc, dev)
    torch.cuda.synchronize(); tot = time.perf_counter() - t0
    print('total %.1f ms' % (1e3 * tot), {k: round(1e3 * v, 2) for k, v in T.items()})
t0 = time.perf_counter(); decompress(arc); print('decompress()', 1e3 * (time.perf_counter() - t0))
