"""One process per GPU: shard ownership, archive offsets and report statistics.

The path is embarrassingly parallel over shards (pipeline.py:4-7; SURVEY
§8e): rank r of G owns shards [S r / G, S (r + 1) / G) -- a contiguous node
block in column mode -- and only that slab of f0 ever reaches its GPU.  The
only exchanges are tiny:
  * all_reduce(SUM) of per-shard blob sizes -> the archive's u64 offset index
    (container.py:182-195), identical to a single-process write_archive;
  * all_reduce SUM / MIN / MAX of the report's decomposable statistics
    (counts, squared-error sums, ranges; pipeline.py:367-391, qoi.py:79-133);
  * optionally a gather of blob bytes / per-image NRMSE to rank 0 when a
    caller wants the whole archive or the full report list in one process.
Works with NCCL (CUDA tensors) and gloo (CPU tensors, used by the tests).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .container import archive_offsets
from .decomp import partition, rank_shards

__all__ = ["RankPlan", "plan", "exchange_sizes", "reduce_stats", "gather_bytes"]


class RankPlan:
    """What rank `rank` of `world` owns of a (P, N) dataset split in S shards."""

    def __init__(self, n_planes, n_nodes, n_shards, mode, rank, world):
        self.shards = partition(n_planes, n_nodes, n_shards, mode)
        self.n_shards = len(self.shards)
        self.mine = rank_shards(self.n_shards, rank, world)
        self.rank, self.world = rank, world
        self.mode = mode
        own = [self.shards[i] for i in self.mine]
        if mode == "col" and own:
            self.node_range = (own[0].nodes_range[0], own[-1].nodes_range[1])
        else:
            self.node_range = (0, n_nodes)


def plan(n_planes, n_nodes, n_shards, mode, rank=None, world=None) -> RankPlan:
    if rank is None:
        rank = dist.get_rank() if dist.is_initialized() else 0
    if world is None:
        world = dist.get_world_size() if dist.is_initialized() else 1
    return RankPlan(n_planes, n_nodes, n_shards, mode, rank, world)


def _device_for(group=None):
    backend = dist.get_backend(group) if dist.is_initialized() else "gloo"
    return torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" \
        else torch.device("cpu")


def exchange_sizes(rp: RankPlan, local_sizes, head_len: int, group=None):
    """Blob sizes of every shard (shard order) and the archive offsets."""
    dev = _device_for(group)
    t = torch.zeros(rp.n_shards, dtype=torch.int64, device=dev)
    for k, sid in enumerate(rp.mine):
        t[sid] = int(local_sizes[k])
    if dist.is_initialized() and rp.world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    sizes = t.cpu().numpy()
    return sizes, np.asarray(archive_offsets(head_len, [int(x) for x in sizes]), dtype=np.int64)


def reduce_stats(local: dict, group=None) -> dict:
    """SUM / MIN / MAX reductions of the report statistics, one collective per
    operation (the values of each kind are packed into one tensor).

    `local` maps name -> (op, float64 array) with op in {"sum", "min", "max"}."""
    dev = _device_for(group)
    ops = {"sum": dist.ReduceOp.SUM, "min": dist.ReduceOp.MIN, "max": dist.ReduceOp.MAX}
    out = {}
    for op in ("sum", "min", "max"):
        names = [k for k, (o, _) in local.items() if o == op]
        if not names:
            continue
        parts = [np.atleast_1d(np.asarray(local[k][1], dtype=np.float64)) for k in names]
        t = torch.as_tensor(np.concatenate(parts), device=dev).clone()
        if dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(t, op=ops[op], group=group)
        flat = t.cpu().numpy()
        pos = 0
        for k, pa in zip(names, parts):
            out[k] = flat[pos:pos + pa.size]
            pos += pa.size
    return out


def gather_bytes(payload: bytes, group=None, dst=0):
    """Gather variable-length byte strings to `dst` (list in rank order there)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return [payload]
    objs = [None] * dist.get_world_size(group) if dist.get_rank(group) == dst else None
    dist.gather_object(payload, objs, dst=dst, group=group)
    return objs


def report_partials(out, tau):
    """Decomposable per-rank statistics of a CompressOut for reduce_stats,
    reduced on the device (one small D2H)."""
    from ._lib import F_EXCEPTION, F_EXC_OVERFLOW, F_NONFINITE, F_SELECTED
    d = out.dev
    flags, status, stats = d["flags"], d["status"], d["stats"]
    q_o, q_r = d["qoi"], d["fqoi"]
    mask = (q_o[:, 0] > 0).unsqueeze(1)
    f64 = torch.float64
    cnt = lambda m: m.sum().to(f64).reshape(1)
    dq = torch.where(mask, (q_o - q_r) ** 2, torch.zeros_like(q_o)).sum(0)
    qmax = torch.where(mask, q_o, torch.full_like(q_o, -np.inf)).amax(0)
    qmin = torch.where(mask, q_o, torch.full_like(q_o, np.inf)).amin(0)
    vals = torch.cat([
        torch.tensor([float(flags.numel())], dtype=f64, device=flags.device),
        cnt((flags & F_SELECTED) != 0), cnt((flags & F_EXCEPTION) != 0),
        cnt((status == 0) & ((flags & F_NONFINITE) == 0) & ((flags & F_EXC_OVERFLOW) == 0)),
        cnt((flags & (F_SELECTED | F_NONFINITE)) == 0), d["fsse"].sum().reshape(1),
        stats[:, 0].max().reshape(1), stats[:, 1].min().reshape(1), dq, mask.sum().to(f64)
        .reshape(1), qmax, qmin]).cpu().numpy()
    return {
        "n": ("sum", vals[0:1]), "selected": ("sum", vals[1:2]),
        "exceptions": ("sum", vals[2:3]), "converged": ("sum", vals[3:4]),
        "ae_ok": ("sum", vals[4:5]), "sse": ("sum", vals[5:6]),
        "data_max": ("max", vals[6:7]), "data_min": ("min", vals[7:8]),
        "qoi_sse": ("sum", vals[8:12]), "qoi_cnt": ("sum", vals[12:13]),
        "qoi_max": ("max", vals[13:17]), "qoi_min": ("min", vals[17:21]),
    }
