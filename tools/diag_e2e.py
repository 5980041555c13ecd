"""Where the end-to-end compress() time goes (host side)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch, struct
import bench
from paper_2212_10733_b200 import engine, pipeline, TimestepState
from paper_2212_10733_b200.container import ArchivePreamble, archive_offsets
from paper_2212_10733_b200.decomp import partition

spec = bench.CONFIGS['cfg3']
ds = bench.corpus(spec['P'], spec['N'])
models = bench.load_models(spec['golden'])
cfg = bench.pipeline_config(1e-3)
state = TimestepState(models=models, timestep_index=1)
dev = torch.device('cuda', 0)
pipeline.compress(ds, cfg, state)
torch.cuda.synchronize()
for rep in range(2):
    T = {}
    t = time.perf_counter()
    def mark(k):
        global t
        torch.cuda.synchronize()
        now = time.perf_counter(); T[k] = 1e3 * (now - t); t = now
    shards = partition(ds.n_planes, ds.n_nodes, cfg.shards, cfg.mode)
    f0 = pipeline.upload_f0(ds.data, dev); mark('upload')
    dgrid = engine.DeviceGrid(ds.grid, dev, cfg.latent_dim)
    works = engine.shard_layout(shards, state.models, ds.n_nodes, ds.grid.rows, ds.grid.cols); mark('grid+layout')
    out = engine.compress_device(f0, works, dgrid, cfg); mark('compress_device')
    preamble = ArchivePreamble(n_shards=len(shards), decomp_mode=cfg.mode, n_planes=ds.n_planes, n_nodes=ds.n_nodes, grid=ds.grid, timestep=ds.timestep, tau=cfg.tau, seed=cfg.seed, config_digest=cfg.digest())
    head = preamble.pack()
    offs = archive_offsets(len(head), [int(n) for n in out.blob_lens])
    from paper_2212_10733_b200 import hostio
    from paper_2212_10733_b200.decomp import shard_dataset_index
    archive = hostio.download_bytes(out.blob_buf, int(np.sum(out.blob_lens)), head + struct.pack(f"<{len(offs)}Q", *offs)); mark('archive bytes')
    out.dataset_index = np.concatenate([shard_dataset_index(sh, ds.n_nodes) for sh in shards]); mark('dataset_index')
    rep_ = pipeline.build_report(ds, archive, [out], cfg.tau, {}, 0.0); mark('report')
    print(rep, {k: round(v, 1) for k, v in T.items()}, 'total', round(sum(T.values()), 1))
t0 = time.perf_counter(); pipeline.compress(ds, cfg, state); torch.cuda.synchronize(); print('compress()', 1e3 * (time.perf_counter() - t0))
