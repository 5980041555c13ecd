"""Does a concurrent pinned H2D stream slow the device step?  compress_device
on resident f0, alone and while another stream uploads 80 MB chunks."""
import sys, time, threading
sys.path.insert(0, '.')
import numpy as np
import torch
import bench
from paper_2212_10733_b200 import engine, pipeline, hostio
from paper_2212_10733_b200.decomp import partition

spec = bench.CONFIGS['cfg3']
ds = bench.corpus(spec['P'], spec['N'])
models = bench.load_models(spec['golden'])
cfg = bench.pipeline_config(1e-3)
dev = torch.device('cuda', 0)
f0 = pipeline.upload_f0(ds.data, dev)
dgrid = engine.DeviceGrid(ds.grid, dev, 4)
shards = partition(8, 16395, 8, 'col')
works = engine.shard_layout(shards, models, 16395, 39, 39)
src = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
dst = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
cs = torch.cuda.Stream()

def step(tag=""):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    timer = engine.Timer(True)
    engine.compress_device(f0, works, dgrid, cfg, timer)
    timer.mark("end")
    torch.cuda.synchronize()
    r = timer.result()
    print(f"{tag:14s} {1e3*(time.perf_counter()-t0):7.2f} ms", {k: round(1e3*v, 2) for k, v in r.items()}, flush=True)

for _ in range(3):
    step("alone")
for chunk_mb, depth in ((80, 100), (2, 2)):
    stop = [False]
    def up():
        torch.cuda.set_device(dev)
        n = chunk_mb << 20
        q = []
        with torch.cuda.stream(cs):
            while not stop[0]:
                for a in range(0, (1 << 30) - n, n):
                    if len(q) >= depth:
                        q.pop(0).synchronize()
                    dst[a:a + n].copy_(src[a:a + n], non_blocking=True)
                    e = torch.cuda.Event(); e.record(cs); q.append(e)
                    if stop[0]:
                        break
        cs.synchronize()
    th = threading.Thread(target=up); th.start()
    time.sleep(0.05)
    for _ in range(3):
        step(f"h2d {chunk_mb}MBx{depth}")
    stop[0] = True; th.join()
# host-only contention: a busy python thread (GIL)
stop = [False]
def spin():
    x = 0
    while not stop[0]:
        x += 1
th = threading.Thread(target=spin); th.start()
for _ in range(2):
    step("gil spin")
stop[0] = True; th.join()
