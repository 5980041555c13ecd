"""Phase wall times of decompress_distributed on every rank (config 3):
   torchrun --nproc-per-node N tools/dec_prof.py  (N = 1 works without torchrun)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import torch.distributed as dist
import bench
from paper_2212_10733_b200 import engine, hostio, distributed, pipeline
from paper_2212_10733_b200.container import ArchivePreamble

rank = int(os.environ.get("RANK", "0")); world = int(os.environ.get("WORLD_SIZE", "1"))
dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
torch.cuda.set_device(dev)
if world > 1:
    dist.init_process_group("nccl", device_id=dev)
spec = bench.CONFIGS["cfg3"]
path = "/dev/shm/mlk_decprof_arc.bin"
if rank == 0:
    ds = bench.corpus(spec["P"], spec["N"])
    models = bench.load_models("cfg3")
    cfg = bench.pipeline_config(1e-3)
    from paper_2212_10733_b200 import compress, TimestepState
    arc, _, _ = compress(ds, cfg, TimestepState(models=models, timestep_index=1))
    open(path, "wb").write(arc)
if world > 1:
    dist.barrier()
arc = open(path, "rb").read()
out_path = "/dev/shm/mlk_decprof_out.f64"
pre, _ = ArchivePreamble.unpack(arc)
sp = distributed.split_plan(pre.n_planes, pre.n_nodes, pre.n_shards, pre.decomp_mode,
                            rank=rank, world=world, latent_dim=1, pq_bits=8)
g = pre.grid
nd = pre.n_nodes * g.rows * g.cols
total = pre.n_planes * nd * 8
for rep in range(4):
    if world > 1:
        dist.barrier()
    t = [time.perf_counter()]
    plan = engine.prepare_decode(arc, dev, sp); torch.cuda.synchronize(); t.append(time.perf_counter())
    out = engine.run_decode(plan); torch.cuda.synchronize(); t.append(time.perf_counter())
    mine = out[:plan.out_elems]
    bad = engine.decoded_negative(plan); t.append(time.perf_counter())
    if rank == 0:
        fd = os.open(out_path, os.O_RDWR | os.O_CREAT, 0o644); os.ftruncate(fd, total); os.close(fd)
    if world > 1:
        dist.barrier()
    t.append(time.perf_counter())
    h = hostio.download_pinned_array(mine, (plan.out_elems,)); t.append(time.perf_counter())
    fd = os.open(out_path, os.O_RDWR)
    t.append(time.perf_counter())
    hostio.download_to_file(mine, plan.out_elems * 8, fd, total, plan.plane_lo * nd * 8)
    t.append(time.perf_counter())
    os.close(fd)
    if world > 1:
        dist.barrier()
    t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    names = ["prepare", "run_decode", "neg check", "trunc+barrier", "D2H pinned (alt)", "open", "D2H into registered map", "barrier"]
    print(f"rank {rank} rep {rep}: " + "  ".join(f"{n} {x:.1f}" for n, x in zip(names, d)) + f"  total {sum(d) - d[4]:.1f} ms", flush=True)
# host parse vs upload inside prepare
t0 = time.perf_counter(); a_d = hostio.upload_bytes(arc, dev); torch.cuda.synchronize()
print(f"rank {rank}: upload_bytes of the whole archive {1e3 * (time.perf_counter() - t0):.1f} ms ({len(arc) / 1e6:.0f} MB); cpus {os.cpu_count()}", flush=True)
if world > 1:
    dist.barrier()
    dist.destroy_process_group()
hostio.release_maps()
if rank == 0:
    os.unlink(path)
    if os.path.exists(out_path):
        os.unlink(out_path)
