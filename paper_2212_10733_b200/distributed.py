"""One process per GPU: work split, archive offsets and report statistics.

The path is embarrassingly parallel over histograms (pipeline.py:4-7; SURVEY
§8e).  Two decompositions of the S shards (S is a configuration value, so
the archive never depends on the GPU count):

  * ``SplitPlan`` (the default): rank r of G processes the contiguous member
    range [n_s r / G, n_s (r + 1) / G) of EVERY shard s -- in column mode
    with P % G == 0 that is planes [P r / G, P (r + 1) / G) of every node
    block -- so the data-dependent residual / exception load (at config 3
    shard 7 holds 57 % of the payloads and 96 % of the exceptions) is spread
    evenly.  Per-shard decisions stay exact through tiny collectives inside
    compress_device: an all_gather of the 32-byte latents (each rank then
    runs the shard's k-means on identical inputs), all_reduce of the
    selection counts / eb_hi, one all_reduce of the probe verdicts per
    bisection round, and an all_gather of the per-rank section sizes from
    which every rank places its pieces of every shard blob;
  * ``RankPlan``: rank r owns whole shards [S r / G, S (r + 1) / G) -- a
    contiguous node block in column mode -- and only that slab of f0 ever
    reaches its GPU.

The exchanges of the archive and the report are tiny too:
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

__all__ = ["RankPlan", "SplitPlan", "plan", "split_plan", "exchange_sizes", "reduce_stats",
           "gather_bytes", "Comm"]


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


def _cut(n: int, r: int, world: int, bits_per_img: int) -> int:
    """Start of rank r's member range of an n-image shard: floor(n r / G),
    moved down so the packed PQ codes of the range start on a byte."""
    if r >= world:
        return n
    a = n * r // world
    while (a * bits_per_img) % 8:
        a -= 1
    return a


class SplitPlan:
    """Rank `rank` of `world` processes members [bounds[s][rank],
    bounds[s][rank + 1]) of every shard s (plane-major member order,
    decomp.py:102).  Its f0 slab is planes [plane_lo, plane_hi) x all nodes."""

    def __init__(self, n_planes, n_nodes, n_shards, mode, rank, world, latent_dim=4,
                 pq_bits=4):
        self.shards = partition(n_planes, n_nodes, n_shards, mode)
        self.n_shards = len(self.shards)
        self.rank, self.world, self.mode = rank, world, mode
        self.n_planes, self.n_nodes = n_planes, n_nodes
        bpi = latent_dim * pq_bits
        self.bounds = np.array([[_cut(len(sh.members), r, world, bpi) for r in range(world + 1)]
                                for sh in self.shards], dtype=np.int64)
        lo, hi = n_planes, 0
        for s, sh in enumerate(self.shards):
            a, e = self.range(s)
            if e > a:
                (p0, _), (x0, x1) = sh.planes_range, sh.nodes_range
                b = x1 - x0
                lo = min(lo, p0 + a // b)
                hi = max(hi, p0 + (e - 1) // b + 1)
        self.plane_lo, self.plane_hi = (lo, hi) if hi > lo else (0, 0)

    def range(self, s, rank=None):
        r = self.rank if rank is None else rank
        return int(self.bounds[s][r]), int(self.bounds[s][r + 1])

    def counts(self, rank=None):
        """Images of every shard that `rank` processes."""
        r = self.rank if rank is None else rank
        return (self.bounds[:, r + 1] - self.bounds[:, r]).astype(np.int64)

    @property
    def n_full(self):
        return self.bounds[:, -1].astype(np.int64)


def split_plan(n_planes, n_nodes, n_shards, mode, rank=None, world=None, latent_dim=4,
               pq_bits=4) -> SplitPlan:
    if rank is None:
        rank = dist.get_rank() if dist.is_initialized() else 0
    if world is None:
        world = dist.get_world_size() if dist.is_initialized() else 1
    return SplitPlan(n_planes, n_nodes, n_shards, mode, rank, world, latent_dim, pq_bits)


class Comm:
    """The collectives compress_device needs under a SplitPlan (NCCL on
    device tensors; gloo moves CPU copies).  Every method is called by all
    ranks in the same order."""

    def __init__(self, sp: SplitPlan, group=None):
        self.sp = sp
        self.group = group
        self.world = sp.world
        self._gidx = {}

    def _cpu(self):
        return dist.get_backend(self.group) != "nccl"

    def all_reduce_(self, t: torch.Tensor, op: str) -> torch.Tensor:
        ops = {"sum": dist.ReduceOp.SUM, "max": dist.ReduceOp.MAX, "min": dist.ReduceOp.MIN}
        if self.world == 1:
            return t
        if self._cpu():
            c = t.cpu()
            dist.all_reduce(c, op=ops[op], group=self.group)
            t.copy_(c)
        else:
            dist.all_reduce(t, op=ops[op], group=self.group)
        return t

    def all_gather(self, t: torch.Tensor) -> torch.Tensor:
        """(world, *t.shape): every rank's t (same shape on every rank)."""
        if self.world == 1:
            return t.unsqueeze(0)
        if self._cpu():
            c = t.cpu().contiguous()
            parts = [torch.empty_like(c) for _ in range(self.world)]
            dist.all_gather(parts, c, group=self.group)
            return torch.stack(parts).to(t.device)
        out = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t.contiguous(), group=self.group)
        return out

    def gather_index(self, dev) -> torch.Tensor:
        """Rows of the (world * max_local) gathered per-image array that form
        the full shards in member order (shard by shard, ranks in order)."""
        key = str(dev)
        if key not in self._gidx:
            sp = self.sp
            cnt = np.stack([sp.counts(r) for r in range(sp.world)])      # (G, S)
            loc_off = np.concatenate([np.zeros((sp.world, 1), np.int64),
                                      np.cumsum(cnt, axis=1)[:, :-1]], axis=1)
            m = int(cnt.sum(axis=1).max()) if cnt.size else 0
            idx = [np.arange(loc_off[r, s], loc_off[r, s] + cnt[r, s]) + r * m
                   for s in range(sp.n_shards) for r in range(sp.world)]
            self._gidx[key] = (torch.from_numpy(np.concatenate(idx).astype(np.int64)).to(dev),
                               max(1, m))
        return self._gidx[key]


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
    reduced on the device by mlk_report (csrc/report.cu; one small D2H).  A
    rank that owns no members contributes the identities (0 / -inf / +inf)."""
    from . import report as R
    v, _, n = R.finish(R.launch([out], False))
    return {
        "n": ("sum", np.array([float(n)])), "selected": ("sum", v[R.SEL:R.SEL + 1]),
        "exceptions": ("sum", v[R.EXC:R.EXC + 1]), "converged": ("sum", v[R.CONV:R.CONV + 1]),
        "ae_ok": ("sum", v[R.AE_OK:R.AE_OK + 1]), "sse": ("sum", v[R.SSE:R.SSE + 1]),
        "data_max": ("max", v[R.DMAX:R.DMAX + 1]), "data_min": ("min", v[R.DMIN:R.DMIN + 1]),
        "qoi_sse": ("sum", v[R.Q_D2]), "qoi_cnt": ("sum", v[R.QCNT:R.QCNT + 1]),
        "qoi_max": ("max", v[R.Q_MAX]), "qoi_min": ("min", v[R.Q_MIN]),
    }
