"""torchrun: phase times of compress_distributed per rank (MLK_TRACE=1)."""
import os, sys
sys.path.insert(0, '.')
os.environ["MLK_TRACE"] = "1"
import torch, torch.distributed as dist
import bench
from paper_2212_10733_b200 import TimestepState, pipeline, FDataset
from paper_2212_10733_b200.hostio import pinned_empty
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
spec = bench.CONFIGS['cfg3']
ds = bench.corpus(spec['P'], spec['N'])
pin = pinned_empty(ds.data.shape); pin[...] = ds.data
ds = FDataset(grid=ds.grid, data=pin, timestep=ds.timestep)
st = TimestepState(models=bench.load_models('cfg3'), timestep_index=1)
cfg = bench.pipeline_config(1e-3)
for _ in range(3):
    pipeline.compress_distributed(ds, cfg, st, out_path="/dev/shm/mlk_trace.mlk")
dist.barrier()
dist.destroy_process_group()
