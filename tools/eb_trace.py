"""Host timeline of the error-bound search rounds inside compress_device
(config 3), per rank: staging, probe launches, the verdict sync, decisions.
Run with torchrun for N > 1."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import torch.distributed as dist
import bench
from paper_2212_10733_b200 import distributed, engine, pipeline

rank = int(os.environ.get("RANK", "0")); world = int(os.environ.get("WORLD_SIZE", "1"))
dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
torch.cuda.set_device(dev)
if world > 1:
    dist.init_process_group("nccl", device_id=dev)
spec = bench.CONFIGS["cfg3"]
ds = bench.corpus(spec["P"], spec["N"])
models = bench.load_models("cfg3")
cfg = bench.pipeline_config(1e-3)
sp = distributed.split_plan(ds.n_planes, ds.n_nodes, cfg.shards, cfg.mode, rank, world,
                            cfg.latent_dim, cfg.pq_bits)
f0 = pipeline.upload_f0(ds.data[sp.plane_lo:sp.plane_hi], dev)
dgrid = engine.DeviceGrid(ds.grid, dev, cfg.latent_dim)
works = engine.split_layout(sp, models, ds.grid.rows, ds.grid.cols)
comm = distributed.Comm(sp) if world > 1 else None
for _ in range(3):
    engine.compress_device(f0, works, dgrid, cfg, comm=comm)
torch.cuda.synchronize()
for rep in range(3):
    engine.EB_TRACE = []
    timer = engine.Timer(True)
    engine.compress_device(f0, works, dgrid, cfg, timer, comm=comm)
    engine.EB_TRACE.append(("returned", time.perf_counter()))
    torch.cuda.synchronize()
    engine.EB_TRACE.append(("gpu_done", time.perf_counter()))
    tr = engine.EB_TRACE
    engine.EB_TRACE = None
    t0 = tr[0][1]
    line = " ".join(f"{k}+{1e3 * (t - t0):.2f}" for k, t in tr)
    st = {k: round(1e3 * v, 2) for k, v in timer.result().items() if k in ("eb_search", "newton", "deflate", "pack")}
    print(f"rank {rank} rep {rep}: {line}  {st}", flush=True)
if world > 1:
    dist.destroy_process_group()
