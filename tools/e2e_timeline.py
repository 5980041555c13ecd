"""Timeline of one pipelined compress() (pinned config-3 f0): host times of
each group's upload-issued / compute start / compute return, and GPU times of
each group's upload-complete and compute-complete events (diagnostic)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
import bench
from paper_2212_10733_b200 import TimestepState, compress, engine, hostio, pipeline, FDataset

spec = bench.CONFIGS['cfg3']
ds = bench.corpus(spec['P'], spec['N'])
pin = hostio.pinned_empty(ds.data.shape); pin[...] = ds.data
dsp = FDataset(grid=ds.grid, data=pin, timestep=ds.timestep)
models = bench.load_models(spec['golden'])
cfg = bench.pipeline_config(1e-3)
st = TimestepState(models=models, timestep_index=1)
G = int(sys.argv[1]) if len(sys.argv) > 1 else 4
pipeline.PIPELINE_GROUPS = G
compress(dsp, cfg, st); compress(dsp, cfg, st)
torch.cuda.synchronize()
log = []
t0 = [0.0]
ev0 = [None]
orig_cd = engine.compress_device
orig_wait = hostio.PieceUpload.wait
orig_finish = hostio.ArchiveWriter.finish
marks = {}

def mark(name):
    e = torch.cuda.Event(enable_timing=True); e.record()
    log.append((name, time.perf_counter() - t0[0], e))

def cd(*a, **k):
    mark(f"dev{k.get('ws_tag')}>")
    r = orig_cd(*a, **k)
    mark(f"dev{k.get('ws_tag')}<")
    return r

import os
PRE = os.environ.get("PRE") == "1"

def wait(self, g):
    mark(f"wait{g}>")
    if PRE and g == 0:
        self.join()
        for i in range(len(self.events)):
            orig_wait(self, i)
        torch.cuda.synchronize()
    orig_wait(self, g)
    mark(f"wait{g}<")

def finish(self, head):
    mark("finish>")
    r = orig_finish(self, head)
    mark("finish<")
    return r

engine.compress_device = cd
pipeline.engine.compress_device = cd
hostio.PieceUpload.wait = wait
hostio.ArchiveWriter.finish = finish
for rep in range(2):
    log.clear()
    torch.cuda.synchronize()
    t0[0] = time.perf_counter()
    mark("start")
    arc, _, _ = compress(dsp, cfg, st)
    mark("end")
    torch.cuda.synchronize()
    e_start = log[0][2]
    print(f"--- G={G} total {1e3*(time.perf_counter()-t0[0]):.2f} ms")
    for name, th, e in log:
        print(f"{name:10s} host {1e3*th:8.2f}  gpu {e_start.elapsed_time(e):8.2f}")
