"""cProfile of compress_device steps (config 3) on rank 0; run with torchrun
for N > 1.  Prints the top functions by own time and by cumulative time."""
import cProfile, io, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
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
kw = dict(comm=comm)
for _ in range(3):
    engine.compress_device(f0, works, dgrid, cfg, **kw)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    engine.compress_device(f0, works, dgrid, cfg, **kw)
torch.cuda.synchronize()
pr.disable()
if rank == 0:
    for key in ("tottime", "cumulative"):
        s = io.StringIO()
        pstats.Stats(pr, stream=s).sort_stats(key).print_stats(30)
        print(s.getvalue())
if world > 1:
    dist.destroy_process_group()
