"""torchrun --nproc-per-node N tools/check_distributed_train.py: with no
trained models (state=None) compress_distributed trains every shard on every
rank; its archive and models equal single-process compress(ds, cfg, None)."""
import os, sys
sys.path.insert(0, '.')
import numpy as np, torch, torch.distributed as dist
import bench
from paper_2212_10733_b200 import compress, pipeline
rank = int(os.environ.get("RANK", 0)); local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
spec = bench.CONFIGS['cfg3']
ds = bench.corpus(spec['P'], spec['N'])
cfg = bench.pipeline_config(1e-3)
path = "/dev/shm/mlk_check_train.mlk"
_, rep, st = pipeline.compress_distributed(ds, cfg, None, out_path=path)
dist.barrier()
if rank == 0:
    got = open(path, "rb").read()
    arc, rep1, st1 = compress(ds, cfg, None)
    same_models = all(np.array_equal(a.weights, b.weights) and a.norm_mean == b.norm_mean
                      and a.norm_std == b.norm_std for a, b in zip(st.models, st1.models))
    print("identical:", got == arc, len(got), len(arc), "models identical:", same_models,
          "timestep", st.timestep_index, st1.timestep_index)
    print("ratio", rep.compression_ratio, rep1.compression_ratio)
    os.unlink(path)
dist.destroy_process_group()
