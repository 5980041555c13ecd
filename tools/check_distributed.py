"""torchrun --nproc-per-node N tools/check_distributed.py: the archive
compress_distributed writes equals single-process compress() bytes."""
import os, sys, hashlib
sys.path.insert(0, '.')
import numpy as np, torch, torch.distributed as dist
import bench
from paper_2212_10733_b200 import TimestepState, compress, pipeline
rank = int(os.environ.get("RANK", 0)); local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
spec = bench.CONFIGS['cfg3']
ds = bench.corpus(spec['P'], spec['N'])
models = bench.load_models(spec['golden'])
cfg = bench.pipeline_config(1e-3)
st = TimestepState(models=models, timestep_index=1)
path = "/dev/shm/mlk_check.mlk"
_, rep, _ = pipeline.compress_distributed(ds, cfg, st, out_path=path)
dist.barrier()
if rank == 0:
    got = open(path, "rb").read()
    arc, rep1, _ = compress(ds, cfg, st)
    print("identical:", got == arc, len(got), len(arc))
    print("ratio", rep.compression_ratio, rep1.compression_ratio, "exc", rep.exception_count,
          rep1.exception_count, "pd", rep.pd_nrmse, rep1.pd_nrmse)
    print("qoi", rep.max_qoi_nrmse, rep1.max_qoi_nrmse)
    os.unlink(path)
dist.destroy_process_group()
