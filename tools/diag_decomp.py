"""Where decompress() time goes."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import bench
from paper_2212_10733_b200 import engine, hostio, TimestepState, compress, decompress

spec = bench.CONFIGS['cfg3']
ds = bench.corpus(spec['P'], spec['N'])
models = bench.load_models(spec['golden'])
cfg = bench.pipeline_config(1e-3)
arc, _, _ = compress(ds, cfg, TimestepState(models=models, timestep_index=1))
dev = torch.device('cuda', 0)
decompress(arc)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dec = engine.decode_archive(arc, dev)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    pre = dec.preamble
    g = pre.grid
    out = hostio.download_array(dec.out[:pre.n_planes * pre.n_nodes * g.rows * g.cols],
                                (pre.n_planes, pre.n_nodes, g.rows, g.cols))
    t2 = time.perf_counter()
    print(f"decode {1e3*(t1-t0):.1f} ms  download {1e3*(t2-t1):.1f} ms")
t0 = time.perf_counter(); decompress(arc); print('decompress()', 1e3 * (time.perf_counter() - t0))
