"""Public compress / decompress / evaluate (reference pipeline.py:29-491).

Same signatures, same archive bytes, same report fields as the reference
`mlk` package; every per-histogram stage runs on the current CUDA device
(``engine.compress_device`` / ``engine.decompress_device``).  Shard count
is a configuration value; the worker count only sets host threads, so
archives are identical for any worker or GPU count (pipeline.py:4-7).
"""

from __future__ import annotations

import ctypes
import hashlib
import json
import os
import struct
import time
from dataclasses import asdict, dataclass, field

import numpy as np
import torch

from . import engine, hostio
from . import report as _report
from . import autoencoder as ae
from .autoencoder import AEModel
from .container import ArchivePreamble, archive_offsets
from .decomp import (SelectionScheme, mix_seed, partition, select_training,
                     shard_dataset_index)
from .errors import ConfigError, DegenerateRangeError, DimensionError
from .fdata import FDataset, dataset_nbytes
from .lagrange import NewtonOptions
from .qoi import ErrorReport, compression_ratio, qoi_nrmse_from_moments

__all__ = ["PipelineConfig", "TimestepState", "compress", "compress_distributed", "decompress",
           "evaluate", "run_timesteps", "QOI_GATES"]

QOI_GATES = {"f32": 1e-8, "f64": 1e-12}
_STAGES = ("train", "encode", "pq", "find_eb", "newton", "pack", "other")


@dataclass(frozen=True)
class PipelineConfig:
    """Field-for-field the reference config (pipeline.py:36-89) so digests match."""

    workers: int = 4
    shards: int = 2
    mode: str = "col"
    scheme: str = "colrandind"
    tau: float = 1e-3
    latent_dim: int = 4
    pq_bits: int = 4
    lambda_precision: str = "f32"
    learning_rate: float = 0.001
    batch_size: int = 128
    epochs_full: int = 100
    epochs_incremental: int = 2
    retrain_period: int = 25
    static_model: bool = False
    newton: NewtonOptions = field(default_factory=NewtonOptions)
    seed: int = 0

    def __post_init__(self):
        if min(self.workers, self.shards, self.latent_dim, self.epochs_full,
               self.epochs_incremental, self.retrain_period, self.batch_size) < 1:
            raise ConfigError("all pipeline counts must be >= 1")
        if self.tau <= 0:
            raise ConfigError("tau must be positive")
        if self.pq_bits not in (4, 6, 8):
            raise ConfigError("pq_bits must be 4, 6, or 8")
        if self.lambda_precision not in ("f32", "f64"):
            raise ConfigError("lambda_precision must be 'f32' or 'f64'")
        if self.mode not in ("row", "col"):
            raise ConfigError("mode must be 'row' or 'col'")
        SelectionScheme(self.scheme)
        if self.seed < 0:
            raise ConfigError("seed must be non-negative")

    def to_dict(self) -> dict:
        return asdict(self)

    @classmethod
    def from_dict(cls, d: dict):
        d = dict(d)
        if isinstance(d.get("newton"), dict):
            d["newton"] = NewtonOptions(**d["newton"])
        return cls(**d)

    def digest(self) -> bytes:
        return hashlib.sha256(json.dumps(self.to_dict(), sort_keys=True).encode()).digest()

    @property
    def lambda_bytes(self) -> int:
        return 4 if self.lambda_precision == "f32" else 8


@dataclass
class TimestepState:
    """Per-shard models carried to the next timestep (pipeline.py:92-96)."""

    models: list
    timestep_index: int = 0


# ---------------------------------------------------------------------------
# device placement helpers

def _device():
    if not torch.cuda.is_available():
        from .errors import BackendError
        raise BackendError("no CUDA device: the B200 path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def upload_f0(data: np.ndarray, device, node_range=None) -> torch.Tensor:
    """(P, N, R, C) float64 host array -> flat device buffer (+16 B pad).

    node_range=(lo, hi) uploads only that node slab of every plane (the
    rank-local part of a column decomposition).  Pinned, chunked and
    overlapped with the host-side copy (hostio.upload_planes)."""
    if data.dtype != np.float64:
        data = data.astype(np.float64)
    return hostio.upload_planes(data, device, node_range)


def _check_state(config, state, n_shards):
    """Reference compress (pipeline.py:327-331): the shard count must match;
    returns train_full (None when the stored models are reused as they are)."""
    if state is not None and len(state.models) != n_shards:
        raise ConfigError("timestep state does not match the shard count")
    index = state.timestep_index if state is not None else 0
    train_full = (state is None) or (not config.static_model
                                     and index % config.retrain_period == 0)
    if state is not None and config.static_model:
        return None      # static mode reuses the models (pipeline.py:206-207)
    return train_full


def _train_models(f0, shards, ds, config, state, train_full, index=None):
    """Per-shard AE training on the device (pipeline.py:208-218): selection
    indices and PCG64 draws on the host, every shard's Adam run in ONE
    mlk_ae_train launch.  f0 = the device-resident dataset (flat, the
    dataset's own layout), or None: then only the selected training rows are
    gathered on the host and uploaded (compress_distributed, where a rank
    holds just its slab of planes and trains only its own shards).  index:
    the shard numbers of `shards` (their warm-start models in state)."""
    D = ds.grid.rows * ds.grid.cols
    epochs = config.epochs_full if train_full else config.epochs_incremental
    tc = ae.TrainConfig(learning_rate=config.learning_rate, batch_size=config.batch_size,
                        epochs=epochs, seed=0)
    sels = []
    for sh in shards:
        seed = mix_seed(config.seed, sh.worker_id)
        sels.append((seed, shard_dataset_index(sh, ds.n_nodes)[
            select_training(sh, config.scheme, ds.n_planes, seed)]))
    if f0 is None:
        idx = np.concatenate([ix for _, ix in sels])
        rows = np.ascontiguousarray(ds.data.reshape(-1, D)[idx], dtype=np.float64)
        f0 = torch.from_numpy(rows.reshape(-1)).to(_device())
        starts = np.cumsum([0] + [len(ix) for _, ix in sels])
        offs = [(starts[i] + np.arange(len(ix), dtype=np.int64)) * D
                for i, (_, ix) in enumerate(sels)]
    else:
        offs = [ix * D for _, ix in sels]
    index = list(range(len(shards))) if index is None else list(index)
    jobs = [ae.TrainJob(base=f0, row_off=o, epochs=epochs, seed=seed,
                        init=None if train_full else state.models[index[i]])
            for i, ((seed, _), o) in enumerate(zip(sels, offs))]
    return ae.train_jobs(jobs, tc, config.latent_dim, D)


def _train_distributed(ds, config, state, train_full, group=None):
    """compress_distributed's training: shard s is trained on rank s % G only
    (from the host rows of its selection), then its f32 weights and (mean,
    std) are broadcast from that rank, so every rank encodes with exactly the
    model rank 0 writes into the weights section -- no assumption that
    several GPUs reproduce one training run bit for bit."""
    import torch.distributed as dist

    from . import distributed as D_
    shards = partition(ds.n_planes, ds.n_nodes, config.shards, config.mode)
    on = dist.is_initialized()
    G = dist.get_world_size(group) if on else 1
    r = dist.get_rank(group) if on else 0
    mine = [s for s in range(len(shards)) if s % G == r]
    trained = {}
    if mine:
        got = _train_models(None, [shards[s] for s in mine], ds, config, state, train_full,
                            index=mine)
        trained = dict(zip(mine, got))
    L, D = config.latent_dim, ds.grid.rows * ds.grid.cols
    dev = D_._device_for(group)
    models = []
    for s in range(len(shards)):
        buf = torch.zeros(2 + L * D, dtype=torch.float64, device=dev)
        if s in trained:
            m = trained[s]
            buf[0], buf[1] = m.norm_mean, m.norm_std
            buf[2:] = torch.from_numpy(np.asarray(m.weights, np.float64).reshape(-1)).to(dev)
        if on and G > 1:
            src = s % G if group is None else dist.get_global_rank(group, s % G)
            dist.broadcast(buf, src=src, group=group)
        h = buf.cpu().numpy()
        models.append(AEModel(weights=h[2:].astype(np.float32).reshape(L, D),
                              norm_mean=float(h[0]), norm_std=float(h[1])))
    return models


# compress() can pipeline shard groups: group g's node blocks are uploaded
# while group g-1 runs on the device, and each group's blobs go D2H / into
# the archive bytes while the next group computes.  The archive does not
# depend on the grouping (shards are independent, pipeline.py:4-7).  Measured
# on the B200 box (tools/e2e_groups.py, config 3, pinned f0): 1 group 63 ms,
# 2 groups 65 ms, 4 groups 70 ms -- every group repeats the latency-bound
# k-means / bisection / DEFLATE tails and the device step slows while the
# upload streams in, so the default is one group (upload, then compute, with
# the archive bytes pre-faulted and filled by the pool as chunks land).
PIPELINE_GROUPS = 1
_GRIDS = {}
# bytes the last compress() moved over PCIe (diagnostics; bench.py's e2e)
LAST_CALL = {}
# stage 1 plane by plane under the upload (measured: 62.4 ms vs 61.5 ms without
# -- the upload then starts only after compress_device's own staging, which
# costs what the overlap gains; tools/e2e_ab.py); exception entries from the
# host f0 (61.5 vs 62.5 ms)
PLANE_STAGE1 = os.environ.get("MLK_PLANE_STAGE1", "0") == "1"
HOST_EXCEPTIONS = os.environ.get("MLK_HOST_EXCEPTIONS", "1") != "0"


def _device_grid(grid, dev, latent_dim):
    """DeviceGrid per (device, grid values, L): built once, reused by every call."""
    key = (dev.index, latent_dim, grid.rows, grid.cols, float(grid.mass),
           hashlib.sha1(np.ascontiguousarray(grid.vol).tobytes() + grid.v_par.tobytes()
                        + grid.v_perp.tobytes()).digest())
    g = _GRIDS.get(key)
    if g is None:
        if len(_GRIDS) > 16:
            _GRIDS.clear()
        g = _GRIDS[key] = engine.DeviceGrid(grid, dev, latent_dim)
    return g


def _groups(S, spec):
    """Shard groups: spec = a count (even split) or a tuple of group sizes."""
    if isinstance(spec, int):
        G = max(1, min(spec, S))
        return [list(range(S * g // G, S * (g + 1) // G)) for g in range(G)]
    out, lo = [], 0
    for n in spec:
        if lo < S:
            out.append(list(range(lo, min(S, lo + n))))
            lo += n
    if lo < S:
        out.append(list(range(lo, S)))
    return out


def _exception_fills(out, shards, data, ds):
    """Holes (buffer offset, length) of the exception entries of `out`'s
    shards and a fill(view, offset, length) that writes them from the host
    f0 with mlk_host_exception_entries in pool-sized chunks."""
    from ._lib import lib
    D = ds.grid.rows * ds.grid.cols
    row = 4 + 8 * D
    src = np.ascontiguousarray(data)
    holes, srcs = [], {}
    for (off, members), sh in zip(out.exceptions, shards):
        if members.size == 0:
            continue
        (p0, _), (x0, x1) = sh.planes_range, sh.nodes_range
        b = x1 - x0
        elem = ((p0 + members // b) * ds.n_nodes + x0 + members % b) * D
        holes.append((off, members.size * row))
        srcs[off] = (np.ascontiguousarray(elem, dtype=np.int64),
                     np.ascontiguousarray(members, dtype=np.uint32))

    def fill(view, off, length):
        elem, idx = srcs[off]
        n = idx.size
        per = max(1, (8 << 20) // row)

        def job(a):
            k = min(n, a + per) - a
            rc = lib().mlk_host_exception_entries(
                ctypes.c_void_p(view[off + a * row:].ctypes.data),
                ctypes.c_void_p(src.ctypes.data), ctypes.c_void_p(elem[a:].ctypes.data),
                ctypes.c_void_p(idx[a:].ctypes.data), k, D)
            if rc != 0:
                raise RuntimeError("mlk_host_exception_entries failed")

        return [hostio._pool().submit(job, a) for a in range(0, n, per)]

    return holes, fill


def _archive_bound(ds, config, n_shards, head_len):
    """Upper bound of the archive length: every image an exception AND a
    residual payload of maximal length (section codecs, pipeline.py:116-184)."""
    D = ds.grid.rows * ds.grid.cols
    n = ds.n_planes * ds.n_nodes
    per_img = (4 + 8 * D) + (21 + 10 * D + 64 + 16) + 64 + config.latent_dim * 2
    per_shard = 44 + 16 + 4 * config.latent_dim * D + 4 * config.latent_dim * 256 + 16
    return head_len + 8 * n_shards + n * per_img + n_shards * per_shard


def compress(ds: FDataset, config: PipelineConfig, state: TimestepState | None = None):
    """Run the five stages on the GPU; returns (archive bytes, report, new state)."""
    t_all = time.perf_counter()
    shards = partition(ds.n_planes, ds.n_nodes, config.shards, config.mode)
    train_full = _check_state(config, state, len(shards))
    dev = _device()
    data = ds.data if ds.data.dtype == np.float64 else ds.data.astype(np.float64)
    S = len(shards)
    # training needs every shard's f0 resident before the step: one group
    groups = _groups(S, PIPELINE_GROUPS if train_full is None else 1)
    pieces = [[(p, sh.nodes_range[0], sh.nodes_range[1]) for i in grp for sh in [shards[i]]
               for p in range(*sh.planes_range)] for grp in groups]
    plane_events = None
    if len(groups) == 1 and (not PLANE_STAGE1 or train_full is not None):
        f0 = upload_f0(data, dev)
        up = hostio.UploadDone(f0)
    elif len(groups) == 1:
        # stage 1 of plane p starts as soon as plane p has landed; the upload
        # is started by compress_device once its own small copies are queued
        f0 = hostio.device_planes_buffer(data, dev)
        up = hostio.UploadDone(f0)

        def plane_events():
            return list(enumerate(hostio.upload_planes(data, dev, plane_events=True,
                                                       into=f0)[1]))
    else:
        up = hostio.upload_pieces(data, dev, pieces)
        f0 = up.buf
    dgrid = _device_grid(ds.grid, dev, config.latent_dim)
    t_train = time.perf_counter()
    if train_full is None:
        models = list(state.models)
    else:
        models = _train_models(f0, shards, ds, config, state, train_full)
    t_train = time.perf_counter() - t_train
    works = engine.shard_layout(shards, models, ds.n_nodes, ds.grid.rows, ds.grid.cols)
    preamble = ArchivePreamble(n_shards=S, decomp_mode=config.mode,
                               n_planes=ds.n_planes, n_nodes=ds.n_nodes, grid=ds.grid,
                               timestep=ds.timestep, tau=config.tau, seed=config.seed,
                               config_digest=config.digest())
    head = preamble.pack()
    head_len = len(head) + 8 * S
    writer = hostio.ArchiveWriter(dev, _archive_bound(ds, config, S, len(head)), head_len)
    outs, lens, timers, stage_t = [], [], [], {}
    try:
        for g, grp in enumerate(groups):
            up.wait(g)
            timer = engine.Timer(True)
            out = engine.compress_device(f0, [works[i] for i in grp], dgrid, config, timer,
                                         ws_tag=g, plane_events=plane_events)
            timer.mark("end")
            timers.append(timer)
            out.dataset_index = np.concatenate([shard_dataset_index(shards[i], ds.n_nodes)
                                                for i in grp])
            outs.append(out)
            if g == len(groups) - 1:
                # the report needs only the archive length: its reductions and
                # small D2H go ahead of the last blob download
                rep_h = report_launch(outs)
            if out.exceptions is not None and HOST_EXCEPTIONS:
                # exception entries are the input's own bytes: written from
                # the host f0 by the pool, only the rest comes back over PCIe
                holes, fills = _exception_fills(out, [shards[i] for i in grp], data, ds)
                writer.add_with_host_rows(out.blob_buf, int(np.sum(out.blob_lens)), holes,
                                          fills)
            else:
                writer.add(out.blob_buf, int(np.sum(out.blob_lens)))
            lens += [int(x) for x in out.blob_lens]
    except BaseException:
        writer.drain()  # pool jobs still write into the archive object
        raise
    finally:
        up.join()
    t0 = time.perf_counter()
    offs = archive_offsets(len(head), lens)
    report = report_finish(rep_h, ds, offs[-1] + lens[-1], config.tau, stage_t, 0.0)
    archive = writer.finish(head + struct.pack(f"<{len(offs)}Q", *offs))
    LAST_CALL.update(h2d_bytes=int(data.nbytes), d2h_bytes=int(writer.d2h_bytes),
                     host_filled_bytes=len(archive) - int(writer.d2h_bytes))
    for timer in timers:
        for k, v in timer.result().items():
            stage_t[k] = stage_t.get(k, 0.0) + v
    stage_t["pack"] = stage_t.get("pack", 0.0) + time.perf_counter() - t0
    if train_full is not None:
        stage_t["train"] = t_train
    report.stage_timings = _timings(stage_t, time.perf_counter() - t_all)
    new_state = TimestepState(models=models,
                              timestep_index=(state.timestep_index if state else 0) + 1)
    return archive, report, new_state


class _Trace:
    """MLK_TRACE=1: print the wall time of each phase (synchronised)."""

    def __init__(self, tag):
        self.on = os.environ.get("MLK_TRACE") == "1"
        self.tag, self.t, self.parts = tag, time.perf_counter(), []

    def mark(self, name):
        if self.on:
            torch.cuda.synchronize()
            t = time.perf_counter()
            self.parts.append(f"{name} {1e3 * (t - self.t):.2f}")
            self.t = t

    def done(self):
        if self.on:
            print(f"[trace {self.tag}] " + " | ".join(self.parts), flush=True)


def compress_distributed(ds: FDataset, config: PipelineConfig, state: TimestepState | None,
                         out_path: str | None = None, group=None):
    """compress() with one process per GPU (torch.distributed initialised).

    Every rank passes the same dataset description and uploads only its
    slab: under distributed.SplitPlan rank r processes members
    [n_s r / G, n_s (r + 1) / G) of every shard s (whole planes when G
    divides the plane count).  The per-shard decisions are reduced across
    ranks inside compress_device, every rank learns the full blob sizes,
    and each writes its pieces of every shard blob with pwrite at their
    archive offsets into `out_path` (rank 0 also writes the preamble and the
    offset index); the report statistics are all-reduced.  Returns
    (out_path, report, new_state); the report's per_image_nrmse is empty
    (it would gather every image)."""
    import torch.distributed as dist

    from . import distributed as D_
    t_all = time.perf_counter()
    sp = D_.split_plan(ds.n_planes, ds.n_nodes, config.shards, config.mode,
                       latent_dim=config.latent_dim, pq_bits=config.pq_bits)
    train_full = _check_state(config, state, sp.n_shards)
    dev = _device()
    trace = _Trace(f"rank {sp.rank}")
    f0 = upload_f0(ds.data[sp.plane_lo:sp.plane_hi], dev)
    dgrid = _device_grid(ds.grid, dev, config.latent_dim)
    trace.mark("upload issued")
    if train_full is None:
        models = list(state.models)
    else:
        models = _train_distributed(ds, config, state, train_full, group)
        trace.mark("train")
    works = engine.split_layout(sp, models, ds.grid.rows, ds.grid.cols)
    out = engine.compress_device(f0, works, dgrid, config, comm=D_.Comm(sp, group))
    trace.mark("device")
    preamble = ArchivePreamble(n_shards=sp.n_shards, decomp_mode=config.mode,
                               n_planes=ds.n_planes, n_nodes=ds.n_nodes, grid=ds.grid,
                               timestep=ds.timestep, tau=config.tau, seed=config.seed,
                               config_digest=config.digest())
    head = preamble.pack()
    sizes = np.asarray(out.blob_lens, dtype=np.int64)
    offs = np.asarray(archive_offsets(len(head), [int(x) for x in sizes]), dtype=np.int64)
    if out_path is not None:
        nbytes = max([o + n for o, _, n in out.segments], default=0)
        # this rank's exception entries are its input's own histograms: they
        # are written into the file from the host f0, only the rest of its
        # pieces comes back over PCIe
        D = ds.grid.rows * ds.grid.cols
        row = 4 + 8 * D
        shards = partition(ds.n_planes, ds.n_nodes, config.shards, config.mode)
        holes = []  # (buffer offset, entries, member indices, shard)
        if HOST_EXCEPTIONS and out.exceptions is not None:
            for (off, members), sh in zip(out.exceptions, shards):
                if members.size:
                    holes.append((off, members.size * row, members, sh))
        holes.sort(key=lambda h: h[0])
        keep, at = [], 0  # buffer ranges that are not exception entries
        for off, ln, _, _ in holes:
            if off > at:
                keep.append((at, off))
            at = max(at, off + ln)
        if nbytes > at:
            keep.append((at, nbytes))
        body = hostio.download_ranges(out.blob_buf, nbytes, keep)
        if sp.rank == 0:
            # rewrite in place (no truncate-to-zero: an existing archive file's
            # pages are reused instead of re-allocated)
            fd = os.open(out_path, os.O_RDWR | os.O_CREAT, 0o644)
            try:
                os.pwrite(fd, head + struct.pack(f"<{len(offs)}Q", *[int(x) for x in offs]), 0)
                os.ftruncate(fd, int(offs[-1] + sizes[-1]))
            finally:
                os.close(fd)
        trace.mark("d2h + head")
        if dist.is_initialized():
            dist.barrier(group=group)
        trace.mark("barrier")
        # every rank copies its pieces into a shared mapping of the file from the
        # pool: pwrite()s to one file serialise on its inode lock across ranks
        fd = os.open(out_path, os.O_RDWR)
        try:
            total = int(offs[-1] + sizes[-1])
            dst = hostio.mapped_file(fd, total)
            base = int(offs[0])

            def to_file(o):  # buffer offset -> file offset (segments are disjoint)
                for lo, goff, n in out.segments:
                    if lo <= o < lo + n:
                        return base + goff + (o - lo)
                raise AssertionError("buffer offset outside every segment")

            spans = []
            for lo, goff, n in out.segments:
                for ka, kb in keep:
                    a0, b0 = max(lo, ka), min(lo + n, kb)
                    spans += [(c, base + goff + (c - lo), min(b0, c + (8 << 20)) - c)
                              for c in range(a0, b0, 8 << 20)]

            def put(x):
                dst[x[1]:x[1] + x[2]] = body[x[0]:x[0] + x[2]]

            jobs = [hostio._pool().submit(put, x) for x in spans]
            src = np.ascontiguousarray(ds.data)
            from ._lib import lib
            per = max(1, (8 << 20) // row)
            for off, ln, members, sh in holes:
                (p0, _), (x0, x1) = sh.planes_range, sh.nodes_range
                bn = x1 - x0
                elem = np.ascontiguousarray(((p0 + members // bn) * ds.n_nodes + x0
                                             + members % bn) * D, dtype=np.int64)
                idx = np.ascontiguousarray(members, dtype=np.uint32)
                fo = to_file(off)

                def fill(a, fo=fo, elem=elem, idx=idx):
                    k = min(idx.size, a + per) - a
                    if lib().mlk_host_exception_entries(
                            ctypes.c_void_p(dst[fo + a * row:].ctypes.data),
                            ctypes.c_void_p(src.ctypes.data),
                            ctypes.c_void_p(elem[a:].ctypes.data),
                            ctypes.c_void_p(idx[a:].ctypes.data), k, D) != 0:
                        raise RuntimeError("mlk_host_exception_entries failed")

                jobs += [hostio._pool().submit(fill, a) for a in range(0, idx.size, per)]
            for j in jobs:
                j.result()
            del dst
        finally:
            os.close(fd)
        trace.mark("pwrite")
        if dist.is_initialized():
            dist.barrier(group=group)
        trace.mark("barrier")
    st = D_.reduce_stats(D_.report_partials(out, config.tau), group)
    trace.mark("report")
    trace.done()
    n = float(st["n"][0])
    span = float(st["data_max"][0] - st["data_min"][0])
    names = ("n", "u_par", "t_perp", "t_par")
    qspan = st["qoi_max"] - st["qoi_min"]
    qerr = {nm: float(np.sqrt(st["qoi_sse"][k] / st["qoi_cnt"][0]) / qspan[k])
            for k, nm in enumerate(names)}
    total_bytes = len(head) + 8 * sp.n_shards + int(sizes.sum())
    report = ErrorReport(
        pd_nrmse=float(np.sqrt(st["sse"][0] / ds.data.size) / span) if span > 0 else 0.0,
        per_image_nrmse=[], qoi_nrmse=qerr, max_qoi_nrmse=max(qerr.values()),
        compression_ratio=compression_ratio(dataset_nbytes(ds), total_bytes),
        ae_accuracy=float(st["ae_ok"][0]) / n, residual_fraction=float(st["selected"][0]) / n,
        convergence_fraction=float(st["converged"][0]) / n,
        exception_count=int(st["exceptions"][0]),
        stage_timings={"other": {"sum": time.perf_counter() - t_all,
                                 "max": time.perf_counter() - t_all}})
    return out_path, report, TimestepState(models=models,
                                           timestep_index=(state.timestep_index if state
                                                           else 0) + 1)


def build_report(ds, archive_len, outs, tau, stage_t, wall) -> ErrorReport:
    """pipeline._build_report (pipeline.py:367-391): every statistic reduced on
    the device, one small D2H of scalars plus the per-image list (dataset
    order, as the reference reports it).  archive_len: the archive's length
    (or the archive itself)."""
    return report_finish(report_launch(outs), ds, archive_len, tau, stage_t, wall)


def report_launch(outs):
    """The device half of build_report: one mlk_report pass (csrc/report.cu)
    and one async D2H into page-locked memory, queued ahead of the archive
    download (the copy engine serves copies in order)."""
    return _report.launch(outs, True, _report.dataset_orders(outs))


def report_finish(handle, ds, archive_len, tau, stage_t, wall) -> ErrorReport:
    """The host half of build_report (waits for report_launch's copy)."""
    if not isinstance(archive_len, (int, np.integer)):
        archive_len = len(archive_len)
    v, per, n_tot = _report.finish(handle)
    span = float(v[_report.DMAX] - v[_report.DMIN])
    pd = float(np.sqrt(v[_report.SSE] / ds.data.size) / span) if span > 0 else 0.0
    cnt = v[_report.QCNT]
    d2_h, qhi_h, qlo_h = v[_report.Q_D2], v[_report.Q_MAX], v[_report.Q_MIN]
    names = ("n", "u_par", "t_perp", "t_par")
    qerr = {}
    for k, nm in enumerate(names):
        rng_k = float(qhi_h[k] - qlo_h[k])
        if cnt == 0:
            raise DimensionError("nrmse needs two equal-length, non-empty arrays")
        if rng_k == 0.0:
            if d2_h[k] != 0.0:
                raise DegenerateRangeError("reference range is zero but arrays differ")
            qerr[nm] = 0.0
        else:
            qerr[nm] = float(np.sqrt(d2_h[k] / cnt) / rng_k)
    return ErrorReport(
        pd_nrmse=pd, per_image_nrmse=per.tolist(), qoi_nrmse=qerr,
        max_qoi_nrmse=max(qerr.values()),
        compression_ratio=compression_ratio(dataset_nbytes(ds), archive_len),
        ae_accuracy=float(v[_report.AE_OK]) / n_tot,
        residual_fraction=float(v[_report.SEL]) / n_tot,
        convergence_fraction=float(v[_report.CONV]) / n_tot,
        exception_count=int(v[_report.EXC]), stage_timings=_timings(stage_t, wall))


def _timings(stage_t, wall):
    timings = {s: {"sum": 0.0, "max": 0.0} for s in _STAGES}
    for k, v in stage_t.items():
        if k in timings:
            timings[k] = {"sum": v, "max": v}
    rest = max(0.0, wall - sum(v for v in stage_t.values()))
    timings["other"] = {"sum": rest, "max": rest}
    return timings


# ---------------------------------------------------------------------------
# decompress (pipeline.py:397-440)

def decompress(archive: bytes) -> FDataset:
    """Invert compress(); exception images are reproduced verbatim."""
    pre, _ = ArchivePreamble.unpack(archive)
    data = engine.decompress_device(archive, _device())
    return FDataset._trusted(pre.grid, data, pre.timestep)


def decompress_distributed(archive: bytes, group=None, gather: bool = True,
                           out_path: str | None = None):
    """decompress() with one process per GPU (torch.distributed initialised).

    The reference decodes every shard independently (pipeline.py:430-440);
    here rank r decodes members [n_s r / G, n_s (r + 1) / G) of every shard
    (the member ranges compress_distributed gave it), i.e. planes
    [P r / G, P (r + 1) / G) of f0, into its own HBM.  gather=True: the slabs
    are all-gathered over NCCL (NVLink) and every rank returns the whole
    FDataset, as decompress() does; gather=False: returns (FDataset of the
    rank's planes, (plane_lo, plane_hi)); out_path: every rank copies its
    planes straight into that file (the (P, N, rows, cols) little-endian
    float64 payload, created by rank 0) over its own PCIe link, and every rank
    returns (out_path, (plane_lo, plane_hi)).  Needs G to divide the plane
    count (each rank's slab is then whole planes)."""
    import torch.distributed as dist

    from . import distributed as D_
    pre, _ = ArchivePreamble.unpack(archive)
    on = dist.is_initialized()
    # member ranges exactly [n_s r / G, n_s (r + 1) / G): the decode needs no
    # byte alignment of the packed codes (bits per image 8 -> no cut)
    sp = D_.split_plan(pre.n_planes, pre.n_nodes, pre.n_shards, pre.decomp_mode,
                       rank=dist.get_rank(group) if on else 0,
                       world=dist.get_world_size(group) if on else 1, latent_dim=1, pq_bits=8)
    if pre.decomp_mode != "col" or pre.n_planes % sp.world:
        raise ConfigError("decompress_distributed needs col mode and a plane count divisible "
                          "by the number of ranks")
    dev = _device()
    plan = engine.prepare_decode(archive, dev, sp)
    out = engine.run_decode(plan)
    g = pre.grid
    nd = pre.n_nodes * g.rows * g.cols
    mine = out[:plan.out_elems]
    if engine.decoded_negative(plan):
        raise ConfigError("histogram values must be non-negative")
    if out_path is not None:
        total = pre.n_planes * nd * 8
        if sp.rank == 0:
            fd = os.open(out_path, os.O_RDWR | os.O_CREAT, 0o644)
            try:
                os.ftruncate(fd, total)
            finally:
                os.close(fd)
        if on and sp.world > 1:
            dist.barrier(group=group)
        fd = os.open(out_path, os.O_RDWR)
        try:
            hostio.download_to_file(mine, plan.out_elems * 8, fd, total, plan.plane_lo * nd * 8)
        finally:
            os.close(fd)
        if on and sp.world > 1:
            dist.barrier(group=group)
        return out_path, (plan.plane_lo, plan.plane_hi)
    if not gather:
        data = hostio.download_pinned_array(mine, (plan.plane_hi - plan.plane_lo, pre.n_nodes,
                                                   g.rows, g.cols))
        return FDataset._trusted(pre.grid, data, pre.timestep), (plan.plane_lo, plan.plane_hi)
    full = torch.empty(pre.n_planes * nd, dtype=torch.float64, device=dev)
    if sp.world > 1:
        dist.all_gather_into_tensor(full, mine.contiguous(), group=group)
    else:
        full.copy_(mine)
    data = hostio.download_pinned_array(full, (pre.n_planes, pre.n_nodes, g.rows, g.cols))
    return FDataset._trusted(pre.grid, data, pre.timestep)


def evaluate(orig: FDataset, archive: bytes) -> ErrorReport:
    """Decompress and fill a full error report with gate verdicts (pipeline.py:443-491)."""
    t0 = time.perf_counter()
    preamble, _ = ArchivePreamble.unpack(archive)
    if (preamble.n_planes, preamble.n_nodes) != (orig.n_planes, orig.n_nodes) or \
            (preamble.grid.rows, preamble.grid.cols) != (orig.grid.rows, orig.grid.cols):
        raise ConfigError("archive dimensions do not match the dataset")
    dev = _device()
    dec = engine.decode_archive(archive, dev)
    torch.cuda.synchronize(dev)
    decode_time = time.perf_counter() - t0
    t1 = time.perf_counter()
    ev = engine.evaluate_device(orig, dec, dev)
    qerr, qmax = qoi_nrmse_from_moments(ev["q_orig"], ev["q_rec"])
    tau = preamble.tau
    gate = QOI_GATES["f32" if dec.lam_bytes == 4 else "f64"]
    per_image = ev["per_image"]
    ae = ev["ae_err"]
    fin = np.where(np.isfinite(ae), ae, np.inf)
    return ErrorReport(
        pd_nrmse=ev["pd_nrmse"], per_image_nrmse=per_image.tolist(), qoi_nrmse=qerr,
        max_qoi_nrmse=qmax,
        compression_ratio=compression_ratio(dataset_nbytes(orig), len(archive)),
        ae_accuracy=float(np.mean(fin <= tau)), residual_fraction=float(np.mean(fin > tau)),
        stage_timings={"decode": {"sum": decode_time, "max": decode_time},
                       "metrics": {"sum": time.perf_counter() - t1,
                                   "max": time.perf_counter() - t1}},
        gates={"pd_per_image": bool(np.all(per_image <= tau)), "qoi": bool(qmax <= gate)})


def run_timesteps(datasets, config: PipelineConfig, models=None):
    """Compress a sequence; full training every retrain_period steps (pipeline.py:494-515).

    Returns a list of (archive, report, mode), mode in {"full", "incremental",
    "static"}.  ``models`` (optional, an extension of the reference API) seeds
    the state with trained per-shard models instead of training at step 0."""
    if not datasets:
        raise ConfigError("need at least one timestep")
    state = TimestepState(models=list(models), timestep_index=0) if models else None
    out = []
    for index, ds in enumerate(datasets):
        if state is None:
            mode = "full"
        elif config.static_model:
            mode = "static"
        elif index % config.retrain_period == 0:
            mode = "full"
        else:
            mode = "incremental"
        archive, report, state = compress(ds, config, state)
        out.append((archive, report, mode))
    return out
