"""torchrun --nproc-per-node 2 tools/debug_ddec.py: where decompress_distributed
differs from decompress (cfg3 archive)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
import bench
import paper_2212_10733_b200 as mb
from paper_2212_10733_b200 import pipeline
local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
spec = bench.CONFIGS["cfg3"]
ds = bench.corpus(spec["P"], spec["N"])
models = bench.load_models("cfg3")
cfg = bench.pipeline_config(1e-3)
st = mb.TimestepState(models=models, timestep_index=1)
path = "/dev/shm/ddec.mlk"
pipeline.compress_distributed(ds, cfg, st, out_path=path)
dist.barrier()
from pathlib import Path
arc = Path(path).read_bytes()
d = pipeline.decompress_distributed(arc).data
d2 = pipeline.decompress_distributed(arc).data
if dist.get_rank() == 0:
    print("repeat equal", bool(np.array_equal(d, d2)))
if dist.get_rank() == 0:
    s = mb.decompress(arc).data
    bad = np.argwhere(~(d == s).all(axis=(2, 3)))
    print("mismatched images", len(bad), bad[:10].tolist())
    if len(bad):
        p, n = bad[0]
        print("max rel", float(np.max(np.abs(d[p, n] - s[p, n]) / np.maximum(np.abs(s[p, n]), 1e-300))))
        planes = np.unique(bad[:, 0]); print("planes", planes.tolist())
        print("per plane counts", [int((bad[:, 0] == q).sum()) for q in planes])
dist.barrier()
dist.destroy_process_group()
