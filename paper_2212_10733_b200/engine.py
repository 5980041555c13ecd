"""Device orchestration of the per-histogram compress / decompress path.

One call processes every shard a rank owns: each kernel launch covers all of
them (the shard id of an image is found from the shard table).  The host
only (a) precomputes exact tables and the PCG64 draws of the k-means
seeding, (b) drives the error-bound bisection with numpy's own log/exp, and
(c) assembles the byte sections around device-produced payloads.

Reference map: pipeline._compress_shard (pipeline.py:196-320) and
pipeline._decode_shard (pipeline.py:397-427).
"""

from __future__ import annotations

import ctypes
import functools
import os
import struct
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, hostio
from ._lib import MlkGrid, MlkNewton, MlkShard, call
from .decomp import mix_seed
from .errors import ConfigError, FormatError, SizeMismatchError

SPAN = 2.0 ** -20
STEPS = 20
LOOKAHEAD = int(os.environ.get("MLK_LOOKAHEAD", 12))  # levels per host round trip
PASS_LEVELS = int(os.environ.get("MLK_PASS_LEVELS", 2))  # levels per probe launch
PROBE_RECON = os.environ.get("MLK_PROBE_RECON", "1") != "0"  # probes read stored reconstructions
EB_TRACE = None  # a list: the search appends (event, host time) per round (diagnostics)
_PAYLOAD_HEAD = struct.Struct("<BHHd")


# ---------------------------------------------------------------------------
# host BLAS order (the decode bracketing the reference inherits from numpy)

@functools.lru_cache(maxsize=None)
def decode_tree_cols(d: int, l: int) -> bytes:
    """Columns where numpy/OpenBLAS sums the L=4 decode products as
    (p0+p1)+(p2+p3) in its blocked kernel (autoencoder.py:109); probed once,
    on one BLAS thread."""
    out = np.zeros(d, dtype=np.uint8)
    if l != 4:
        return out.tobytes()
    rng = np.random.default_rng(20221221)
    n = max(512, int(1e6 // (l * d)) + 64)
    w = rng.standard_normal((l, d)).astype(np.float32).astype(np.float64)
    z = (rng.standard_normal((n, l)) * 37.0).astype(np.float32).astype(np.float64)
    # the reference's orders are single-threaded OpenBLAS's: probe
    # that kernel whatever this process's BLAS thread count is (a threaded
    # run partitions the product differently)
    try:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=1, user_api="blas"):
            ref = z @ w
    except ImportError:  # pragma: no cover - threadpoolctl ships with the image
        ref = z @ w
    p = [z[:, k:k + 1] * w[k][None, :] for k in range(4)]
    seq = ((p[0] + p[1]) + p[2]) + p[3]
    tree = (p[0] + p[1]) + (p[2] + p[3])
    for j in np.flatnonzero((seq != ref).any(axis=0)):
        if (tree[:, j] == ref[:, j]).all():
            out[j] = 1
    return out.tobytes()


# ---------------------------------------------------------------------------
# grid tables

# Separable grids take the exponent-table Newton (project.cu); tests switch it
# off to exercise the per-cell path on the same fixtures.
SEPARABLE_NEWTON = True


class DeviceGrid:
    """Exact grid tables on device (lagrange.py:68-80, 163-173, 199-204)."""

    def __init__(self, grid, device, latent_dim: int = 4):
        r, c = grid.rows, grid.cols
        self.D = r * c
        vol = grid.vol.reshape(-1)
        vpar = np.broadcast_to(grid.v_par, (r, c)).reshape(-1)
        vperp = np.broadcast_to(grid.v_perp[:, None], (r, c)).reshape(-1)
        half_m = 0.5 * grid.mass
        rows = [vol, vol * vpar, half_m * vol * vperp ** 2]
        scales = [float(np.max(np.abs(x))) for x in rows]
        ash = np.concatenate([x / s for x, s in zip(rows, scales)])
        tc = np.frombuffer(decode_tree_cols(self.D, latent_dim), dtype=np.uint8)

        def dev(a, dt=torch.float64):
            return torch.from_numpy(np.ascontiguousarray(a)).to(device=device, dtype=dt)

        self.t = dict(vol=dev(vol), vpar=dev(vpar), vperp2=dev(vperp ** 2),
                      hmvol=dev(half_m * vol), ash=dev(ash), tree=dev(tc.copy(), torch.uint8))
        self.mass = grid.mass
        # separable trapezoid volumes (make_grid): vol depends on edge class only
        re_ = np.zeros(r, dtype=int)
        re_[[0, -1]] = 1
        ce_ = np.zeros(c, dtype=int)
        ce_[[0, -1]] = 1
        cls = 2 * re_[:, None] + ce_[None, :]
        vcls = [grid.vol[cls == k][0] if np.any(cls == k) else 0.0 for k in range(4)]
        sep = int(all(np.all(grid.vol[cls == k] == vcls[k]) for k in range(4) if np.any(cls == k)))
        # the factorised Newton sums also need vol ~= dlt * w_r * w_c
        if sep and vcls[0] > 0:
            wc_, wr_ = vcls[1] / vcls[0], vcls[2] / vcls[0]
            sep = int(abs(vcls[3] - vcls[0] * wr_ * wc_) <= 1e-12 * abs(vcls[3]))
        sep = int(sep and SEPARABLE_NEWTON)
        self.struct = MlkGrid(rows=r, cols=c, D=self.D, pad=0, mass=grid.mass,
                              vol=self.t["vol"].data_ptr(), vpar=self.t["vpar"].data_ptr(),
                              vperp2=self.t["vperp2"].data_ptr(),
                              hmvol=self.t["hmvol"].data_ptr(), ash=self.t["ash"].data_ptr(),
                              tree_cols=self.t["tree"].data_ptr(), s0=scales[0], s1=scales[1],
                              s2=scales[2], sep=sep, pad2=0)
        for k in range(4):
            self.struct.vcls[k] = float(vcls[k])

    @property
    def addr(self) -> int:
        return ctypes.addressof(self.struct)


# ---------------------------------------------------------------------------
# error-bound search (residual.py:129-173) as an explicit state machine so a
# whole subtree of candidate bounds can be probed in one launch

@dataclass(frozen=True)
class _Search:
    stage: str            # "hi" | "bis" | "low" | "done"
    eb_hi: float
    lo: object = None
    hi: object = None
    best: object = None
    step: int = 0
    result: tuple = None

    def query(self):
        if self.stage == "hi":
            return self.eb_hi
        if self.stage == "bis":
            return np.exp(0.5 * (self.lo + self.hi))
        if self.stage == "low":
            return self.eb_hi * SPAN
        return None

    def advance(self, ok: bool) -> "_Search":
        if self.stage == "hi":
            if ok:
                return _Search("done", self.eb_hi, result=(self.eb_hi, False))
            return _Search("bis", self.eb_hi, np.log(self.eb_hi * SPAN), np.log(self.eb_hi),
                           None, 0)._settle()
        if self.stage == "bis":
            mid = 0.5 * (self.lo + self.hi)
            if ok:
                nxt = _Search("bis", self.eb_hi, mid, self.hi, np.exp(mid), self.step + 1)
            else:
                nxt = _Search("bis", self.eb_hi, self.lo, mid, self.best, self.step + 1)
            return nxt._settle()
        if self.stage == "low":
            low = self.eb_hi * SPAN
            return _Search("done", self.eb_hi, result=(float(low), not ok))
        raise AssertionError("search already done")

    def _settle(self) -> "_Search":
        if self.stage == "bis" and self.step == STEPS:
            if self.best is not None:
                return _Search("done", self.eb_hi, result=(float(self.best), False))
            return _Search("low", self.eb_hi)
        return self


def _search_heap(states, depth: int) -> np.ndarray:
    """Candidate bounds of the next `depth` decisions of each search, in heap
    order: column 1 is the state's query, 2i / 2i+1 the next query after node
    i is accepted / rejected; NaN where the search has ended.  The tree's
    structure and log-space midpoints come from mlk_search_tree (host C, the
    scalar machine's own additions and halvings); the bounds are numpy's
    exp of those midpoints and the same eb_hi / eb_hi 2^-20 products as
    _Search.query -- bit-identical values (compress_device re-checks every
    root against _Search.query; tests/test_host_logic.py pins whole trees)."""
    n = 1 << depth
    S = len(states)
    codes = {"done": 0, "hi": 1, "bis": 2, "low": 3}
    kind0 = np.array([codes[st.stage] for st in states], dtype=np.int8)
    step0 = np.array([st.step if st.stage == "bis" else 0 for st in states], dtype=np.int32)
    best0 = np.array([st.best is not None for st in states], dtype=np.uint8)
    lo0 = np.array([st.lo if st.stage == "bis" else 0.0 for st in states], dtype=np.float64)
    hi0 = np.array([st.hi if st.stage == "bis" else 0.0 for st in states], dtype=np.float64)
    eb_hi = np.array([st.eb_hi for st in states], dtype=np.float64)
    lo_end, hi_end = np.log(eb_hi * SPAN), np.log(eb_hi)
    kind = np.empty((S, n), dtype=np.int8)
    mid = np.empty((S, n), dtype=np.float64)
    if S:
        rc = _lib.host_lib().mlk_search_tree(
            kind0.ctypes.data, step0.ctypes.data, best0.ctypes.data, lo0.ctypes.data,
            hi0.ctypes.data, lo_end.ctypes.data, hi_end.ctypes.data, S, depth, STEPS,
            kind.ctypes.data, mid.ctypes.data)
        if rc != 0:
            raise ConfigError("search tree depth out of range")
    out = np.full((S, n), np.nan)
    b = kind == 2
    out[b] = np.exp(mid[b])
    ebc = np.broadcast_to(eb_hi[:, None], (S, n))
    h = kind == 1
    out[h] = ebc[h]
    lw = kind == 3
    out[lw] = (ebc * SPAN)[lw]
    return out


# ---------------------------------------------------------------------------
# compress

@dataclass
class ShardWork:
    """A shard as the device sees it plus its model."""

    wid: int
    n_img: int
    base: int              # element offset of image 0 in the rank's f0 buffer
    plane_stride: int
    block: int
    model: object          # AEModel
    rows: int = 39
    cols: int = 39
    j0: int = 0            # member index of image 0 (split shards, distributed.SplitPlan)
    n_full: int = -1       # images of the whole shard (-1: n_img)
    plane0: int = 0        # plane of member 0 (plane-wise stage 1)

    @property
    def n_total(self) -> int:
        return self.n_img if self.n_full < 0 else self.n_full


@dataclass
class CompressOut:
    """Device-resident result of compress_device: the rank's shard blobs back
    to back in `blob_buf` plus the per-image arrays the report needs."""

    specs: list
    blob_buf: torch.Tensor
    blob_lens: np.ndarray  # whole shard blobs (every rank's pieces)
    dev: dict
    sel_count: np.ndarray
    eb: list
    lossless: list
    rows_cols: tuple
    img_off: list
    segments: list = field(default_factory=list)  # (buf offset, blob-region offset, length)
    exceptions: list = None  # per shard (buf offset of its entries, member indices)
    timings: dict = field(default_factory=dict)
    _host: dict = field(default_factory=dict)

    def host(self, name):
        if name not in self._host:
            self.fetch(name)
        return self._host[name]

    def fetch(self, *names):
        """Bring several per-image arrays to the host with one copy."""
        need = [n for n in names if n not in self._host]
        if not need:
            return
        ts = [self.dev[n].contiguous() for n in need]
        flat = torch.cat([t.reshape(-1).view(torch.uint8) for t in ts])
        raw = hostio.download_view(flat, flat.numel())
        pos = 0
        for n, t in zip(need, ts):
            nb = t.numel() * t.element_size()
            dt = torch.empty((), dtype=t.dtype).numpy().dtype
            self._host[n] = raw[pos:pos + nb].view(dt).reshape(tuple(t.shape)).copy()
            pos += nb

    def blobs(self) -> list:
        raw = self.blob_buf.cpu().numpy().tobytes()
        out, pos = [], 0
        for n in self.blob_lens:
            out.append(raw[pos:pos + int(n)])
            pos += int(n)
        return out


class Timer:
    """Stage timer: CUDA events on the current stream; MLK_TIMING=sync adds a
    device synchronize per mark and reports host wall intervals instead
    (diagnostics: exposes host-side stalls inside a stage)."""

    def __init__(self, enabled=True):
        import os
        self.enabled = enabled
        self.sync = os.environ.get("MLK_TIMING") == "sync"
        self.marks = []
        self.points = []
        self.spans = []

    def span_start(self, stream):
        """An event on `stream` opening a span (span_end closes it)."""
        if not self.enabled or self.sync:
            return None
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        return ev

    def span_end(self, name, stream, ev0):
        """Report the time between ev0 and now on `stream` as `name` (one
        launch's in-situ duration on its own stream)."""
        if ev0 is None:
            return
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        self.spans.append((name, ev0, ev))

    def point(self, name, stream, since):
        """An event on `stream`, reported as ms after the mark `since`
        (points of concurrent streams: which one a join waited for)."""
        if not self.enabled or self.sync:
            return
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        self.points.append((name, ev, since))

    def mark(self, name):
        if not self.enabled:
            return
        if self.sync:
            import time
            torch.cuda.synchronize()
            self.marks.append((name, time.perf_counter()))
            return
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self.marks.append((name, ev))

    def result(self):
        if not self.enabled or len(self.marks) < 2:
            return {}
        torch.cuda.synchronize()
        out = {}
        for (n0, e0), (_, e1) in zip(self.marks, self.marks[1:]):
            dt = (e1 - e0) if self.sync else e0.elapsed_time(e1) / 1e3
            out[n0] = out.get(n0, 0.0) + dt
        base = dict(self.marks)
        for name, ev, since in self.points:
            if since in base and not self.sync:
                out[name] = out.get(name, 0.0) + base[since].elapsed_time(ev) / 1e3
        for name, ev0, ev1 in self.spans:
            out[name] = out.get(name, 0.0) + ev0.elapsed_time(ev1) / 1e3
        return out


def _shard_table(specs, D, L, full=False):
    """MlkShard table of a rank's (pieces of) shards; full=True describes the
    whole shards instead (the k-means input after the latents all_gather)."""
    arr = (MlkShard * len(specs))()
    off = 0
    for i, sp in enumerate(specs):
        n = sp.n_total if full else sp.n_img
        # the encode order is the one numpy picks for the whole shard's matmul
        small = sp.n_total * L * D <= 1e6
        arr[i] = MlkShard(base=sp.base, plane_stride=sp.plane_stride, block=sp.block,
                          n_img=n, img_off=off, small_blas=int(small),
                          mean=float(sp.model.norm_mean), std=float(sp.model.norm_std), eb=0.0,
                          lossless=0, w_off=i * L * D, j0=0 if full else sp.j0, pad=0)
        off += n
    return arr


def _upload_shards(arr, device):
    raw = np.frombuffer(bytes(arr), dtype=np.uint8).copy()
    return torch.from_numpy(raw).to(device)


_GRAMS = {}


def _gram(models):
    """Per-shard [W W^T, row sums, row norms, max |W|] (cached on the weight
    bytes: the models are the same every timestep in static mode)."""
    # identity + address + a checksum of each weight array (a model mutated in
    # place changes its sum)
    key = tuple((id(m.weights), m.weights.ctypes.data, float(np.sum(m.weights, dtype=np.float64)))
                for m in models)
    g = _GRAMS.get(key)
    if g is None:
        if len(_GRAMS) > 64:
            _GRAMS.clear()
        g = _GRAMS[key] = _gram_compute(models)
    return g


def _gram_compute(models):
    rows = []
    for m in models:
        w = m.weights.astype(np.float64)
        rows.append(np.concatenate([(w @ w.T).reshape(-1), w.sum(axis=1),
                                    np.sqrt((w * w).sum(axis=1)), np.abs(w).max(axis=1)]))
    return np.stack(rows)


@functools.lru_cache(maxsize=4096)
def kmeans_draws(n: int, k: int, seed: int):
    """The PCG64 draws quantizer.kmeans_1d consumes (quantizer.py:68,77): a pure
    function of (n, k, seed), so it is cached."""
    g = np.random.Generator(np.random.PCG64(seed))
    first = int(g.integers(n))
    return first, tuple(g.random() for _ in range(k - 1))


_NP2TORCH = {}


class Workspace:
    """Per-device persistent buffers: grow-only device arenas by name and a
    pinned host staging arena whose contents reach the device with one async
    copy per flush (no pageable, stream-draining H2D on the hot path)."""

    _by_dev = {}

    def __init__(self, dev, cap=1 << 26):
        self.dev = dev
        self.bufs = {}
        self.views = {}
        self._alloc(cap)
        self.pending = []
        self.ready = None

    def _alloc(self, cap):
        self.h = torch.empty(cap, dtype=torch.uint8).pin_memory()
        self.hn = self.h.numpy()
        self.d = torch.empty(cap, dtype=torch.uint8, device=self.dev)
        self.pos = 0

    @classmethod
    def get(cls, dev, tag=0):
        """The workspace `tag` of a device (compress() pipelines shard groups
        through separate workspaces so a group's results outlive the next)."""
        ws = cls._by_dev.get((dev.index, tag))
        if ws is None:
            ws = cls._by_dev[(dev.index, tag)] = Workspace(dev)
        return ws

    _ESIZE = {}

    def tensor(self, name, shape, dtype):
        """A typed view of the grow-only buffer `name` (views are cached per
        (name, shape, dtype) while the buffer stays the same)."""
        key = (name, shape, dtype)
        hit = self.views.get(key)
        b = self.bufs.get(name)
        if hit is not None and hit[0] is b:
            return hit[1]
        es = self._ESIZE.get(dtype)
        if es is None:
            es = self._ESIZE[dtype] = torch.empty((), dtype=dtype).element_size()
        n = int(np.prod(shape)) if shape else 1
        nbytes = max(16, n * es)
        if b is None or b.numel() < nbytes:
            self.bufs[name] = b = torch.empty(int(nbytes * 1.25) + 64, dtype=torch.uint8,
                                              device=self.dev)
        v = b[:nbytes].view(dtype)[:n].view(shape)
        if len(self.views) > 512:  # data-dependent shapes: keep the cache bounded
            self.views.clear()
        self.views[key] = (b, v)
        return v

    def reset(self):
        """Start of a call: the previous call's staged copies must have landed
        before the arena is rewritten (device views of one call stay valid for
        the whole call because positions only grow within it)."""
        if self.ready is not None:
            self.ready.synchronize()
            self.ready = None
        self.pos = 0

    def begin(self):
        pass

    def stage(self, arr):
        """Queue a host array; returns its device view after the next flush()."""
        a = np.ascontiguousarray(arr)
        nb = a.nbytes
        if self.pos + nb + 16 > self.h.numel():
            # grow (rare): everything staged so far must reach the device first
            if self.pending:
                raise MemoryError("staging arena exhausted inside a flush group")
            torch.cuda.synchronize(self.dev)
            self._alloc(max(2 * self.h.numel(), nb + (1 << 20)))
        self.hn[self.pos:self.pos + nb] = a.reshape(-1).view(np.uint8)
        view = self.d[self.pos:self.pos + max(nb, 1)]
        td = _NP2TORCH.get(a.dtype)
        if td is None:
            td = _NP2TORCH[a.dtype] = torch.from_numpy(a[:0].copy()).dtype
        out = view[:nb].view(td).view(a.shape) if nb else view
        self.pending.append((self.pos, nb))
        self.pos = (self.pos + nb + 15) & ~15
        return out

    def flush(self):
        if self.pending:
            lo = self.pending[0][0]
            self.d[lo:self.pos].copy_(self.h[lo:self.pos], non_blocking=True)
            self.pending = []
            ev = torch.cuda.Event()
            ev.record()
            self.ready = ev


def _d2h(*tensors):
    """One synchronisation point for several small device results."""
    return [t.cpu().numpy() for t in tensors]


def compress_device(f0: torch.Tensor, specs, dgrid: DeviceGrid, cfg, timer: Timer | None = None,
                    zlib_level: int = 6, comm=None, ws_tag=0, plane_events=None) -> CompressOut:
    """Run stages 2-5 of pipeline._compress_shard for every shard in `specs`.

    f0 is a flat float64 CUDA tensor holding the rank's histograms; image j
    of spec s is member g = j0 + j of its shard, at
    base + (g // block) * plane_stride + (g % block) * D.
    comm (distributed.Comm): the specs are this rank's member ranges of every
    shard (distributed.SplitPlan); the per-shard decisions are made on
    collectively reduced inputs, so every rank's pieces are exactly those of
    the single-process blobs.
    plane_events: a callable that starts the upload of f0 and returns
    [(plane, cuda event)] (hostio.upload_planes(..., plane_events=True)): it
    is called once this call's own small host->device copies are queued (the
    copy engine serves copies in order, so they must not wait behind the
    upload), and stage 1 then runs plane by plane as each lands, everything
    after it in stream order behind them all.
    Device arrays in the result stay valid until the next call on the device
    with the same ws_tag.
    """
    dev = f0.device
    D, L, K = dgrid.D, cfg.latent_dim, 2 ** cfg.pq_bits
    S = len(specs)
    timer = timer or Timer(False)
    for sp in specs:
        if sp.model.latent_dim != L or sp.model.input_dim != D:
            raise ConfigError("shard model does not match the configuration/grid")
    ws = Workspace.get(dev, ws_tag)
    ws.reset()
    T = ws.tensor
    f64, i32, i64 = torch.float64, torch.int32, torch.int64
    table = _shard_table(specs, D, L)
    total = sum(sp.n_img for sp in specs)
    sh_d = ws.stage(np.frombuffer(bytes(table), dtype=np.uint8))
    W = ws.stage(np.stack([sp.model.weights for sp in specs]).astype(np.float32))
    first, draws = [], []
    for sp in specs:
        seed = mix_seed(cfg.seed, sp.wid)
        for d in range(L):
            f, u = kmeans_draws(sp.n_total, K, seed + d)
            first.append(f)
            draws.extend(u)
    first_d = ws.stage(np.asarray(first, dtype=np.int64))
    draws_d = ws.stage(np.asarray(draws, dtype=np.float64))
    gram = ws.stage(_gram([sp.model for sp in specs]))
    if comm is not None:
        table_full = _shard_table(specs, D, L, full=True)
        shf_d = ws.stage(np.frombuffer(bytes(table_full), dtype=np.uint8))
    else:
        table_full, shf_d = table, sh_d
    plane_tabs = []
    planes = list(range(max((sp.plane0 + sp.n_img // max(1, sp.block) for sp in specs),
                            default=0))) if plane_events is not None else []
    for p in planes:
        # the members of every shard that lie on plane p (plane-major order)
        ents = []
        for si, sp in enumerate(specs):
            q = p - sp.plane0
            if sp.n_img % sp.block or sp.j0 % sp.block or not 0 <= q < sp.n_img // sp.block:
                continue
            e = MlkShard.from_buffer_copy(table[si])
            e.n_img, e.img_off, e.j0 = sp.block, e.img_off + q * sp.block, e.j0 + q * sp.block
            ents.append(e)
        arr = (MlkShard * max(1, len(ents)))(*ents)
        plane_tabs.append((p, ws.stage(np.frombuffer(bytes(arr), dtype=np.uint8)), len(ents),
                           sum(e.n_img for e in ents)))
    if plane_tabs and sum(t[3] for t in plane_tabs) != total:
        raise ConfigError("plane-wise stage 1 needs shards made of whole planes")
    ws.flush()
    if plane_events is not None:
        evs = dict(plane_events())
        plane_tabs = [(evs[p], tab_d, n_ent, n_pl) for p, tab_d, n_ent, n_pl in plane_tabs]

    timer.mark("encode")
    lat = T("lat", (total, L), f64)
    stats = T("stats", (total, 4), f64)
    qoi = T("qoi", (total, 4), f64)
    if plane_tabs:
        main = torch.cuda.current_stream(dev)
        for ev, tab_d, n_ent, n_pl in plane_tabs:
            main.wait_event(ev)
            if n_ent:
                call("mlk_stage1", f0, tab_d, n_ent, n_pl, dgrid.addr, W, L, lat, stats, qoi)
    else:
        call("mlk_stage1", f0, sh_d, S, total, dgrid.addr, W, L, lat, stats, qoi)

    timer.mark("pq")
    lat_km, total_km = lat, total
    if comm is not None:
        # every rank's latents, rearranged into whole shards (32 B per image)
        gidx, m = comm.gather_index(dev)
        lat_pad = T("lat_pad", (m, L), f64)
        lat_pad[:total].copy_(lat)
        lat_km = comm.all_gather(lat_pad).reshape(-1, L).index_select(0, gidx)
        total_km = lat_km.shape[0]
    scratch = T("km_scratch", (4 * L * total_km,), f64)
    cents = T("cents", (S, L, K), torch.float32)
    kinfo = T("kinfo", (S, L, 4), i32)
    call("mlk_kmeans", lat_km, shf_d, ctypes.addressof(table_full), S, L, K, first_d, draws_d,
         scratch, cents, None, kinfo)

    timer.mark("find_eb")
    codes = T("codes", (total, L), torch.uint8)
    flags = T("flags", (total,), torch.uint8)
    err_a = T("err_a", (total,), f64)
    rbound = T("rbound", (total,), f64)
    call("mlk_select", lat, stats, sh_d, S, total, dgrid.addr, cents, L, K, gram, cfg.tau, codes,
         flags, err_a, rbound)
    timer.mark("recheck")
    err_x = T("err_x", (total,), f64)
    call("mlk_recheck", f0, stats, sh_d, S, total, dgrid.addr, W, L, cents, K, codes, cfg.tau,
         flags, err_x)
    timer.mark("compact")
    sel = T("sel", (total,), i32)
    sel_rank = T("sel_rank", (total,), i32)
    sel_rng = T("sel_rng", (total,), i32)
    sel_cnt = T("sel_cnt", (S,), i32)
    eb_hi = T("eb_hi", (S,), f64)
    call("mlk_compact", flags, stats, sh_d, S, cfg.tau, sel, sel_rank, sel_rng, sel_cnt, eb_hi)
    if comm is not None:
        # eb_hi = tau * max range over the whole shard's selection (residual.py:143)
        cnt_g = sel_cnt.clone()
        comm.all_reduce_(cnt_g, "sum")
        comm.all_reduce_(eb_hi, "max")
        cnt_h, cntg_h, ebhi_h = _d2h(sel_cnt, cnt_g, eb_hi)
    else:
        cnt_h, ebhi_h = _d2h(sel_cnt, eb_hi)
        cntg_h = cnt_h

    # ---- projection of the images WITHOUT residuals does not need the error
    #      bounds: it runs on a side stream under the error-bound search
    #      (capped CTAs per SM leave room for the probe kernels)
    n_sel = int(cnt_h.sum())
    vcap = ((10 * D + 15) // 16) * 16
    varint = T("varint", (max(1, n_sel) * vcap,), torch.uint8)
    vlen = T("vlen", (max(1, n_sel),), i64)
    opts = MlkNewton(step=cfg.newton.step, max_iter=cfg.newton.max_iter,
                     retry=int(cfg.newton.retry), tol=cfg.newton.tol, floor=cfg.newton.floor,
                     retry_step=cfg.newton.retry_step, retry_max_iter=cfg.newton.retry_max_iter,
                     lam_f32=int(cfg.lambda_precision == "f32"), tau=cfg.tau)
    lam = T("lam", (total, 4), f64)
    qst = T("qst", (total, 4), f64)
    status = T("status", (total,), i32)
    iters = T("iters", (total,), i32)
    ferr = T("ferr", (total,), f64)
    fqoi = T("fqoi", (total, 4), f64)
    fsse = T("fsse", (total,), f64)
    errf = T("errf", (1,), i32)
    errf.zero_()
    list_sel = T("list_sel", (max(1, total),), i32)
    list_non = T("list_non", (max(1, total),), i32)
    nsel_d = T("nsel_d", (1,), i32)
    call("mlk_split_flags", flags, total, _lib.F_SELECTED, list_sel, list_non, nsel_d)
    main = torch.cuda.current_stream(dev)
    side = _side_stream(dev) if PROJECT_OVERLAP else main
    if side is not main:
        ev_split = torch.cuda.Event()
        ev_split.record(main)
        side.wait_event(ev_split)
    sp_non = timer.span_start(side)
    call("mlk_project", f0, stats, qoi, sh_d, S, total, dgrid.addr, W, L, cents, K, codes,
         sel_rank, None, ctypes.addressof(opts), flags, lam, qst, status, iters, ferr, fqoi,
         fsse, varint, vcap, vlen, errf, list_non, total - n_sel, None, stream=side.cuda_stream)
    timer.span_end("project_non_launch", side, sp_non)
    ev_non = torch.cuda.Event()
    ev_non.record(side)

    timer.mark("eb_search")
    # the search is a chain of small launches and host round trips: on a
    # high-priority stream its CTAs go first whenever the side stream's
    # projection CTAs retire
    hi_ctx = None
    if side is not main:
        hi = _hi_stream(dev)
        hi.wait_stream(main)
        hi_ctx = torch.cuda.stream(hi)
        hi_ctx.__enter__()
    # ---- error-bound search, LOOKAHEAD levels per launch
    states = []
    for s in range(S):
        if cntg_h[s] == 0:
            states.append(None)
            continue
        eb_hi_s = float(ebhi_h[s])
        if eb_hi_s <= 0:
            states.append(_Search("done", eb_hi_s, result=(eb_hi_s, True)))
        else:
            states.append(_Search("hi", eb_hi_s))
    n_sel_all = int(cnt_h.sum())
    bins = T("probe_bins", (max(1, total) * 68,), f64)
    # the selected images' reconstructions, stored once for the probes
    recon = (T("probe_recon", (max(1, n_sel_all) * ((D + 1) & ~1),), f64) if PROBE_RECON
             else None)
    call("mlk_probe_bins", f0, sh_d, S, dgrid.addr, W, L, cents, K, codes, sel_rng, sel_cnt,
         n_sel_all, eb_hi, bins, sel_rank, recon)
    n_nodes = 1 << LOOKAHEAD
    rounds = 0
    fail = T("fail", (S, n_nodes), i32)
    zero_start = ws.stage(np.zeros(S, dtype=np.int32))
    ws.flush()
    # each round's lookahead tree and work offsets: one pinned host block and
    # one copy into fixed device views (the previous round's copy has landed:
    # its verdicts were read back)
    nb_cand = 8 * S * n_nodes
    h_round = hostio.pinned(f"eb_round{dev.index}", nb_cand + 4 * (S + 1))
    d_round = T("eb_round", (nb_cand + 4 * (S + 1),), torch.uint8)
    h_cand = h_round.numpy()[:nb_cand].view(np.float64).reshape(S, n_nodes)
    h_off = h_round.numpy()[nb_cand:nb_cand + 4 * (S + 1)].view(np.int32)
    cand_d = d_round[:nb_cand].view(torch.float64).view(S, n_nodes)
    off_d = d_round[nb_cand:].view(torch.int32)
    tr = EB_TRACE.append if EB_TRACE is not None else None
    while any(st is not None and st.stage != "done" for st in states):
        rounds += 1
        if tr:
            tr(("round", time.perf_counter()))
        cnt_act = np.zeros(S, dtype=np.int32)
        live = []
        for s, st in enumerate(states):
            if st is not None and st.stage != "done":
                live.append(s)
                cnt_act[s] = int(cnt_h[s])
        cand = h_cand
        cand.fill(np.nan)
        cand[live] = _search_heap([states[s] for s in live], LOOKAHEAD)
        if tr:
            tr(("tree", time.perf_counter()))
        off = h_off
        off[0] = 0
        np.cumsum(cnt_act, out=off[1:])
        d_round.copy_(h_round[:nb_cand + 4 * (S + 1)], non_blocking=True)
        if tr:
            tr(("flush", time.perf_counter()))
        fail.zero_()
        if tr:
            tr(("staged", time.perf_counter()))
        for level in range(0, LOOKAHEAD, PASS_LEVELS):  # several levels per pass
            call("mlk_probe", f0, stats, sh_d, S, dgrid.addr, W, L, cents, K, codes, sel_rng,
                 off_d, zero_start, int(off[-1]), rbound, cfg.tau, cand_d, n_nodes, level,
                 min(PASS_LEVELS, LOOKAHEAD - level), fail, bins, eb_hi,
                 sel_cnt if recon is not None else None, sel_rank, recon)
        if tr:
            tr(("launched", time.perf_counter()))
        if comm is not None:
            comm.all_reduce_(fail, "max")
        (fail_h,) = _d2h(fail)
        if tr:
            tr(("synced", time.perf_counter()))
        for s, st in enumerate(states):
            if st is None or st.stage == "done":
                continue
            node = 1
            for level in range(LOOKAHEAD):
                if st.stage == "done":
                    break
                # the tree was built with the state machine's own float
                # operations (tests/test_host_logic.py pins it level by level);
                # the root of every round is re-checked here
                if level == 0 and st.query() != cand[s, node]:
                    raise AssertionError("lookahead tree out of step with the search")
                ok = fail_h[s, node] == 0
                st = st.advance(ok)
                node = 2 * node + (0 if ok else 1)
            states[s] = st
        if tr:
            tr(("decided", time.perf_counter()))
    eb = [0.0] * S
    lossless = [False] * S
    for s, st in enumerate(states):
        if st is not None:
            eb[s], lossless[s] = st.result
    for s in range(S):
        table[s].eb = eb[s]
        table[s].lossless = int(lossless[s])

    timer.mark("newton")
    slot_base_h = np.concatenate([[0], np.cumsum(cnt_h)[:-1]]).astype(np.int32)
    ws.begin()
    sh_d = ws.stage(np.frombuffer(bytes(table), dtype=np.uint8))
    slot_base = ws.stage(slot_base_h)
    ws.flush()
    if n_sel:
        # the residual images feed DEFLATE (the critical path): still on the
        # high-priority stream, ahead of the side stream's remaining CTAs
        sp_sel = timer.span_start(torch.cuda.current_stream(dev))
        call("mlk_project", f0, stats, qoi, sh_d, S, total, dgrid.addr, W, L, cents, K, codes,
             sel_rank, slot_base, ctypes.addressof(opts), flags, lam, qst, status, iters, ferr,
             fqoi, fsse, varint, vcap, vlen, errf, list_sel, n_sel, recon)
        timer.span_end("project_sel_launch", torch.cuda.current_stream(dev), sp_sel)
    if hi_ctx is not None:
        hi_ctx.__exit__(None, None, None)
        main.wait_stream(hi)
    timer.mark("deflate")
    # DEFLATE needs only the residual images' varint streams: it starts while
    # the side stream may still be projecting the others
    zout, zoff, zlen = deflate_launch(ws, varint, vcap, vlen, n_sel, dev)
    timer.point("deflate_done", main, "deflate")
    if side is not main:
        timer.point("project_rest_done", side, "deflate")
    main.wait_event(ev_non)
    exc_list = T("exc_list", (total,), i32)
    exc_cnt = T("exc_cnt", (S,), i32)
    call("mlk_list_flags", flags, sh_d, S, _lib.F_EXCEPTION, exc_list, exc_cnt)
    # while DEFLATE runs: the host copies of what the pack stage stages that
    # does not depend on the compressed sizes (weights sections, entry shards,
    # each shard's entry range)
    own0 = comm is None or comm.sp.rank == 0
    ws.begin()
    wraw = [sp.model.to_bytes() for sp in specs] if own0 else []
    w_d = ws.stage(np.frombuffer(b"".join(wraw), dtype=np.uint8)) if own0 else None
    ent_shard = ws.stage(np.repeat(np.arange(S, dtype=np.int32), cnt_h))
    e_lo = slot_base_h.astype(np.int64)
    rng_d = ws.stage(np.concatenate([e_lo, e_lo + cnt_h]))
    ws.flush()
    # entry bytes (21-byte header + zlib body) prefix-summed on the device:
    # the host reads back only each shard's total and the smallest length
    zinc = T("zinc", (n_sel + 1,), i64)
    zsm = T("zsmall", (S + 1,), i64)
    zinc[:1].zero_()
    if n_sel:
        torch.cumsum(zlen[:n_sel] + 21, 0, out=zinc[1:])
        torch.sub(zinc.index_select(0, rng_d[S:]), zinc.index_select(0, rng_d[:S]), out=zsm[:S])
        zsm[S:].copy_(zlen[:n_sel].amin().view(1))
    else:
        zsm.zero_()
    # (the exception lists too: callers write those entries from host f0)
    zsm_h, exc_h, errf_h, excl_h = _d2h(zsm, exc_cnt, errf, exc_list)
    if tr:
        tr(("zlen_synced", time.perf_counter()))
    res_h = zsm_h[:S].astype(np.int64)
    bad = [int(errf_h[0]), int(n_sel > 0 and zsm_h[S] < 0)]
    ranks = None
    if comm is not None:
        # every rank's section sizes: where its pieces go in each shard blob
        mine = np.concatenate([[sp.n_img for sp in specs], cnt_h, res_h, exc_h, bad]).astype(
            np.int64)
        allr = comm.all_gather(torch.from_numpy(mine).to(dev)).cpu().numpy()
        ranks = dict(rank=comm.sp.rank, n=allr[:, :S], cnt=allr[:, S:2 * S],
                     res=allr[:, 2 * S:3 * S], exc=allr[:, 3 * S:4 * S])
        bad = allr[:, 4 * S:].max(axis=0).tolist()
    if bad[0]:
        raise ConfigError("error bound too small for this residual range")
    if bad[1]:
        raise ConfigError("residual stream exceeds the device DEFLATE limits")

    timer.mark("pack")
    lay = blob_layout(specs, cfg, D, cnt_h, None, exc_h, ranks, res_h=res_h)
    if tr:
        tr(("layout", time.perf_counter()))
    buf = T("blob", (max(1, lay["total"]),), torch.uint8)
    # fixed pieces (rank 0 of a split): 44-byte header, residual / exception
    # section prefixes; the weights sections from the copy staged above
    pieces, src, ln, dst = [], [], [], []
    pos = 0
    for s, sp in enumerate(specs):
        if lay["hdr_off"][s] < 0:
            continue
        for off, raw in ((lay["hdr_off"][s], lay["header"][s]),
                         (lay["res_pre_off"][s], struct.pack("<dI", eb[s], int(cntg_h[s]))),
                         (lay["exc_pre_off"][s], struct.pack("<I", int(lay["exc_total"][s])))):
            pieces.append(raw)
            src.append(pos)
            ln.append(len(raw))
            dst.append(off)
            pos += len(raw)
    pq_s = [s for s in range(S) if lay["pq_off"][s] >= 0]
    ws.begin()
    if pieces:
        stage = ws.stage(np.frombuffer(b"".join(pieces), dtype=np.uint8))
        src_d = ws.stage(np.asarray(src, np.int64))
        ln_d = ws.stage(np.asarray(ln, np.int64))
        dst_d = ws.stage(np.asarray(dst, np.int64))
        pq_src = ws.stage(np.asarray([4 * L * K * s for s in pq_s], dtype=np.int64))
        pq_len = ws.stage(np.full(len(pq_s), 4 * L * K, dtype=np.int64))
        pq_off = ws.stage(lay["pq_off"][pq_s])
        w_len = np.array([len(w) for w in wraw], dtype=np.int64)
        w_src = ws.stage(np.concatenate([[0], np.cumsum(w_len)[:-1]]).astype(np.int64))
        w_ln = ws.stage(w_len)
        w_dst = ws.stage(lay["hdr_off"] + 44)
    # each entry's buffer offset: its shard's first entry + the prefix sum
    ent_base = ws.stage(lay["ent_off"] - np.concatenate([[0], np.cumsum(res_h)[:-1]]))
    lam_off = ws.stage(lay["lam_off"])
    exc_base = ws.stage(np.concatenate([[0], np.cumsum(exc_h)]).astype(np.int32))
    exc_off = ws.stage(lay["exc_base"])
    ws.flush()
    if tr:
        tr(("pack_staged", time.perf_counter()))
    if pieces:
        call("mlk_gather_segments", stage, src_d, ln_d, len(pieces), buf, dst_d)
        call("mlk_gather_segments", w_d, w_src, w_ln, S, buf, w_dst)
        call("mlk_gather_segments", cents.view(torch.uint8).reshape(-1), pq_src, pq_len,
             len(pq_s), buf, pq_off)
    # codes: pack_indices straight into the blob (each piece starts on a byte)
    c16 = T("codes16", (total * L,), torch.int16)
    c16.copy_(codes.reshape(-1))
    bad_d = T("bad", (1,), i32)
    base = buf.data_ptr()
    for s, sp in enumerate(specs):
        if sp.n_img == 0:
            continue
        off = table[s].img_off
        call("mlk_pack_indices", c16[off * L:(off + sp.n_img) * L], sp.n_img * L, cfg.pq_bits,
             base + int(lay["codes_off"][s]), bad_d)
    if n_sel:
        entry_off = T("entry_off", (n_sel,), i64)
        torch.add(zinc[:n_sel], ent_base.index_select(0, ent_shard), out=entry_off)
        call("mlk_pack_residuals", sel, sh_d, ent_shard, entry_off, zoff, zlen, zout, slot_base,
             dgrid.struct.rows, dgrid.struct.cols, n_sel, buf)
    call("mlk_pack_lambdas", lam, qst, sh_d, S, total, lam_off,
         int(cfg.lambda_precision == "f32"), buf)
    call("mlk_pack_exceptions", f0, sh_d, S, exc_list, exc_base, exc_off, int(exc_h.sum()), D,
         buf)
    if tr:
        tr(("pack_launched", time.perf_counter()))
    out = CompressOut(specs=specs, blob_buf=buf, blob_lens=lay["blob_len"],
                      dev=dict(codes=codes, cents=cents, flags=flags, lam=lam, qst=qst,
                               status=status, iters=iters, ferr=ferr, fqoi=fqoi, fsse=fsse,
                               qoi=qoi, stats=stats, sel=sel, kinfo=kinfo),
                      sel_count=cnt_h, eb=eb, lossless=lossless, rows_cols=(
                          dgrid.struct.rows, dgrid.struct.cols), img_off=[t.img_off for t in table],
                      segments=lay["segments"])
    if excl_h is not None:
        # where each shard's exception entries sit in blob_buf, and whose they
        # are (member indices), for callers that fill them from host f0
        out.exceptions = [(int(lay["exc_base"][s]) + 4,
                           excl_h[table[s].img_off:table[s].img_off + int(exc_h[s])].astype(np.int64)
                           + table[s].j0) for s in range(S)]
    out.timings = {"probe_rounds": rounds}
    return out


def blob_layout(specs, cfg, D, cnt_h, zlen_h, exc_h, ranks=None, res_h=None):
    """Byte layout of every shard blob (container.py:30-95, pipeline.py:116-184)
    and of the pieces of it this rank writes.

    ranks=None: the rank holds whole shards.  Otherwise a dict of (G, S)
    arrays over every rank -- n (images), cnt (residual entries), res (entry
    bytes), exc (exceptions) -- and `rank`: the blob sizes are those of the
    whole shards, and this rank writes its member range of the codes, lambda,
    residual-entry and exception sections (rank 0 also the header, weights,
    PQ table and section prefixes).  Pieces are laid out in the rank's buffer
    in blob order; `segments` maps (buffer offset, blob-region offset, length).
    With one rank the buffer IS the blob region (a single segment).

    zlen_h (zlib body length per residual entry) gives `entry_off`, every
    entry's buffer offset; zlen_h=None with res_h (this rank's entry bytes per
    shard, 21 + body each) skips it -- the caller derives the offsets from
    `ent_off` (each shard's first entry) and its own prefix sums."""
    from .container import ShardHeader, SCHEME_FULL
    L, bits, K = cfg.latent_dim, cfg.pq_bits, 2 ** cfg.pq_bits
    lb = 4 if cfg.lambda_precision == "f32" else 8
    S = len(specs)
    cnt = np.asarray(cnt_h, dtype=np.int64)
    e_start = np.concatenate([[0], np.cumsum(cnt)[:-1]]).astype(np.int64)
    if zlen_h is not None:
        # entry bytes (21-byte entry header + zlib body), prefix-summed once
        zcs = np.concatenate([[0], np.cumsum(21 + np.asarray(zlen_h, dtype=np.int64))])
        zl_sum = zcs[e_start + cnt] - zcs[e_start]
    else:
        zl_sum = np.asarray(res_h, dtype=np.int64)
    if ranks is None:
        ranks = dict(rank=0, n=np.array([[sp.n_img for sp in specs]], dtype=np.int64),
                     cnt=cnt[None], res=zl_sum[None], exc=np.asarray(exc_h, np.int64)[None])
    r = ranks["rank"]
    n_all, res_all, exc_all = ranks["n"], ranks["res"], ranks["exc"]
    # per-shard totals over every rank and the parts of the ranks before r
    n_tot, n_pre, n_own = (n_all.sum(0).tolist(), n_all[:r].sum(0).tolist(),
                           n_all[r].tolist())
    res_tot, res_pre, res_own = (res_all.sum(0).tolist(), res_all[:r].sum(0).tolist(),
                                 res_all[r].tolist())
    exc_tot, exc_pre, exc_own = (exc_all.sum(0).tolist(), exc_all[:r].sum(0).tolist(),
                                 exc_all[r].tolist())
    cnt_l, e_start_l = cnt.tolist(), e_start.tolist()
    keys = ("blob_off", "blob_len", "hdr_off", "codes_off", "pq_off", "res_pre_off", "ent_off",
            "lam_off", "exc_pre_off", "exc_base", "exc_total")
    lay = {k: np.full(S, -1, dtype=np.int64) for k in keys}
    lay["header"] = []
    entry_off = np.zeros(len(zlen_h), dtype=np.int64) if zlen_h is not None else None
    segs = []
    cur = [0]

    def put(goff, n):
        """Reserve n buffer bytes for blob-region bytes [goff, goff + n)."""
        o = cur[0]
        if n <= 0:
            return o
        if segs and segs[-1][0] + segs[-1][2] == o and segs[-1][1] + segs[-1][2] == goff:
            segs[-1][2] += n
        else:
            segs.append([o, goff, n])
        cur[0] += n
        return o

    gpos = 0
    rec = 4 + 8 * D
    for s, sp in enumerate(specs):
        n = n_tot[s]
        a = n_pre[s]          # first member of this rank's range
        m = n_own[s]
        n_exc = exc_tot[s]
        sec = (16 + 4 * L * D, (n * L * bits + 7) // 8, 4 * L * K, 12 + res_tot[s], n * 8 * lb,
               4 + n_exc * rec)
        g_codes = gpos + 44 + sec[0]
        g_pq = g_codes + sec[1]
        g_res = g_pq + sec[2]
        g_lam = g_res + sec[3]
        g_exc = g_lam + sec[4]
        own0 = r == 0
        if own0:
            lay["hdr_off"][s] = put(gpos, 44 + sec[0])
        c_lo = a * L * bits // 8
        c_hi = sec[1] if a + m == n else (a + m) * L * bits // 8
        lay["codes_off"][s] = put(g_codes + c_lo, c_hi - c_lo)
        if own0:
            lay["pq_off"][s] = put(g_pq, sec[2])
            lay["res_pre_off"][s] = put(g_res, 12)
        ent = put(g_res + 12 + res_pre[s], res_own[s])
        lay["ent_off"][s] = ent
        c, e0 = cnt_l[s], e_start_l[s]
        if c and entry_off is not None:
            entry_off[e0:e0 + c] = ent + (zcs[e0:e0 + c] - zcs[e0])
        lay["lam_off"][s] = put(g_lam + a * 8 * lb, m * 8 * lb)
        if own0:
            lay["exc_pre_off"][s] = put(g_exc, 4)
        lay["exc_base"][s] = put(g_exc + 4 + exc_pre[s] * rec, exc_own[s] * rec) - 4
        lay["exc_total"][s] = n_exc
        lay["blob_off"][s] = gpos
        blen = 44 + sum(sec)
        lay["blob_len"][s] = blen
        lay["header"].append(ShardHeader(scheme=SCHEME_FULL, lambda_precision=lb,
                                         section_lengths=sec, n_images=n,
                                         img_rows=specs[s].rows, img_cols=specs[s].cols,
                                         latent_dim=L, pq_bits=bits).pack())
        gpos += blen
    lay["entry_off"] = entry_off
    lay["total"] = cur[0]
    lay["segments"] = [tuple(x) for x in segs]
    return lay


# ---------------------------------------------------------------------------
# DEFLATE on device (zlib.compress(x, 6) byte-exact, csrc/zlib6.h)

_DEFLATE_POOLS = {}
DEFLATE_WORK = 1 << 18
_SCRATCH = {}


def _scratch(dev, name, nbytes):
    """Grow-only named device scratch (uint8), reused across calls."""
    key = (dev.index, name)
    buf = _SCRATCH.get(key)
    if buf is None or buf.numel() < nbytes:
        _SCRATCH[key] = buf = torch.empty(max(1, int(nbytes * 1.25)), dtype=torch.uint8,
                                          device=dev)
    return buf


# project the residual-free images on a low-priority side stream under the
# error-bound search
PROJECT_OVERLAP = os.environ.get("MLK_PROJECT_OVERLAP", "1") != "0"
_SIDE_STREAMS = {}


def _side_stream(dev):
    s = _SIDE_STREAMS.get(dev.index)
    if s is None:
        s = _SIDE_STREAMS[dev.index] = torch.cuda.Stream(device=dev, priority=0)
    return s


_HI_STREAMS = {}


def _hi_stream(dev):
    s = _HI_STREAMS.get(dev.index)
    if s is None:
        lo, hi = torch.cuda.Stream.priority_range()
        s = _HI_STREAMS[dev.index] = torch.cuda.Stream(device=dev, priority=hi)
    return s


def _deflate_pool(dev, n_workers):
    key = (dev.index, n_workers)
    if key not in _DEFLATE_POOLS:
        _DEFLATE_POOLS.clear()
        _DEFLATE_POOLS[key] = torch.zeros(n_workers * DEFLATE_WORK, dtype=torch.uint8, device=dev)
    return _DEFLATE_POOLS[key]


DEFLATE_TIERS = (1024, 1600, 2048, 3072, 4096, 8192, 16000)


DEFLATE_PROF = None   # set to a (16,) uint64 CUDA tensor to collect phase cycles
# tier warps claim streams from an atomic counter (dynamic balance)
DEFLATE_DYNAMIC = os.environ.get("MLK_DEFLATE_DYNAMIC", "1") != "0"


_TIER_STREAMS = {}


_SMS = {}


def _sm_count(dev):
    n = _SMS.get(dev.index)
    if n is None:
        n = _SMS[dev.index] = torch.cuda.get_device_properties(dev).multi_processor_count
    return n


def _tier_streams(dev, n):
    key = dev.index
    if key not in _TIER_STREAMS:
        # high priority: DEFLATE is the tail of the step; the residual-free
        # projection on the low-priority side stream fills in around it
        hi = torch.cuda.Stream.priority_range()[1]
        _TIER_STREAMS[key] = [torch.cuda.Stream(device=dev, priority=hi) for _ in range(n)]
    return _TIER_STREAMS[key]


def _run_deflate(ws, varint, in_off, vlen, n, zout, zoff, zcap, zlen, dev, max_workers=2048):
    """Warp-cooperative kernel per size tier, the tiers concurrently on their own
    streams (a sparse tier is bounded by single-stream latency, not throughput);
    one thread per stream beyond the last tier."""
    sms = _sm_count(dev)
    sym_cap = 3 * DEFLATE_TIERS[-1] + 32  # symbols + the 16-byte phase-1 record
    sym = ws.tensor("deflate_sym", (n * sym_cap,), torch.uint8)
    main = torch.cuda.current_stream(dev)
    streams = _tier_streams(dev, len(DEFLATE_TIERS) + 1)
    ctr = ws.tensor("deflate_ctr", (len(DEFLATE_TIERS) + 1,), torch.int32)
    ctr.zero_()
    ev0 = torch.cuda.Event()
    ev0.record(main)
    bounds = list(zip((0,) + DEFLATE_TIERS, DEFLATE_TIERS + (None,)))
    # largest streams first: the few long, latency-bound streams of the upper
    # tiers start at once and overlap the bulk tier instead of trailing it
    # (launched on the tier streams by handle: no current-stream switching)
    for k in reversed(range(len(bounds))):
        lo, hi = bounds[k]
        st = streams[k]
        st.wait_event(ev0)
        if hi is None:
            workers = min(n, max_workers)
            call("mlk_zlib_compress6", varint, in_off, vlen, n, zout, zoff, zcap, zlen,
                 _deflate_pool(dev, workers), workers, lo, stream=st.cuda_stream)
        else:
            nb = 2 * sms if k < 3 else sms
            if DEFLATE_DYNAMIC:
                call("mlk_zlib_compress6_warp_dyn", varint, in_off, vlen, n, lo, hi, zout, zoff,
                     zcap, zlen, nb, sym, sym_cap, DEFLATE_PROF, ctr[k:k + 1],
                     stream=st.cuda_stream)
            else:
                call("mlk_zlib_compress6_warp", varint, in_off, vlen, n, lo, hi, zout, zoff,
                     zcap, zlen, nb, sym, sym_cap, DEFLATE_PROF, stream=st.cuda_stream)
        ev = torch.cuda.Event()
        ev.record(st)
        main.wait_event(ev)


def deflate_launch(ws, varint, vcap, vlen, n, dev):
    """Launch zlib-6 over every varint slot; returns device (zout, zoff, zlen)."""
    i64 = torch.int64
    zcap = vcap + 64
    m = max(1, n)
    zout = ws.tensor("zout", (m * zcap,), torch.uint8)
    zlen = ws.tensor("zlen", (m,), i64)
    in_off = ws.tensor("in_off", (m,), i64)
    zoff = ws.tensor("zoff", (m,), i64)
    torch.arange(0, m * vcap, vcap, out=in_off)
    torch.arange(0, m * zcap, zcap, out=zoff)
    if n:
        _run_deflate(ws, varint, in_off, vlen[:n], n, zout, zoff, zcap, zlen, dev)
    return zout, zoff, zlen


def deflate_device(varint, vcap, vlen, n, dev):
    """zlib-6 every varint slot; returns (zout, zoff, zlen) on device + zlen host."""
    ws = Workspace.get(dev)
    zout, zoff, zlen = deflate_launch(ws, varint, vcap, vlen, n, dev)
    zlen_h = zlen[:n].cpu().numpy()
    if np.any(zlen_h < 0):
        raise ConfigError("residual stream exceeds the device DEFLATE limits")
    return zout, zoff, zlen, zlen_h


def deflate_slots(varint, vcap, vlen, n, dev):
    """zlib-6 every varint slot on device; returns the packed bodies (host),
    their offsets and lengths."""
    if n == 0:
        return np.zeros(0, np.uint8), np.zeros(0, np.int64), np.zeros(0, np.int64)
    zout, zoff, zlen, zlen_h = deflate_device(varint, vcap, vlen, n, dev)
    dst_h = np.concatenate([[0], np.cumsum(zlen_h)[:-1]]).astype(np.int64)
    comp = torch.empty(max(1, int(zlen_h.sum())), dtype=torch.uint8, device=dev)
    call("mlk_gather_segments", zout, zoff, zlen, n, comp, torch.from_numpy(dst_h).to(dev))
    return comp.cpu().numpy(), dst_h, zlen_h


# ---------------------------------------------------------------------------
# decompress (pipeline.py:397-440)

def _unzigzag_host(z):
    return ((z >> np.uint64(1)) ^ (np.uint64(0) - (z & np.uint64(1)))).astype(np.int64)


_WHY = {1: "residual section truncated", 2: "residual section has trailing bytes",
        3: "residual payload shorter than its header",
        4: "residual payload dims do not match the shard",
        5: "unknown residual payload mode", 6: "residual entry image index out of range",
        7: "residual section lists more entries than images"}


@dataclass
class DecodedArchive:
    """An archive decoded on the device (pipeline.py:397-440)."""

    preamble: object
    shards: list
    out: torch.Tensor          # (P*N*D) float64 on the device, dataset order
    specs: list
    table: object
    sh_d: torch.Tensor
    W: torch.Tensor
    cents: torch.Tensor
    codes: torch.Tensor
    L: int
    K: int
    lam_bytes: int
    dgrid: "DeviceGrid"


@dataclass
class DecodePlan:
    """An archive parsed on the host and staged on the device: everything
    run_decode's launches read (prepare_decode)."""

    preamble: object
    shards: list
    specs: list
    table: object
    models: list
    total: int
    n_res: int
    n_exc: int
    L: int
    K: int
    bits: int
    lam_bytes: int
    arc_d: torch.Tensor
    sh_d: torch.Tensor
    W: torch.Tensor
    cents: torch.Tensor
    res_slot: torch.Tensor
    exc_slot: torch.Tensor
    lam_seg: torch.Tensor
    lam_len: torch.Tensor
    lam_dst: torch.Tensor
    code_src: list          # per shard (archive offset, n_images, first member, count)
    img_off: np.ndarray
    body: tuple             # (off, len, eb, mode) device tensors of the kept entries
    exc_seg: tuple          # (src, len, dst)
    dgrid: "DeviceGrid"
    out_elems: int
    dev: torch.device
    plane_lo: int = 0
    plane_hi: int = 0
    codes: object = None    # the unpacked codes of the last run_decode
    neg: object = None      # device flag: the last run_decode wrote a value < 0


def prepare_decode(archive, dev, sp=None) -> DecodePlan:
    """Parse an archive (pipeline.py:397-440) and stage what the device
    decode needs.  sp: a distributed.SplitPlan -- decode only rank sp.rank's
    members [n_s r/G, n_s (r+1)/G) of every shard into its slab of planes
    [sp.plane_lo, sp.plane_hi) (decompress_distributed); None: everything.

    The host reads only the preamble, the shard index, the 44-byte shard
    headers, the small weight / codebook sections and the residual entry
    chain (mlk_parse_residual_section, in place over the archive bytes);
    the archive goes to the device in one pinned copy and every per-image
    byte -- codes, lambdas, zlib bodies, exception images -- is read there."""
    from .autoencoder import AEModel
    from .container import HEADER_SIZE, SECTIONS, ArchivePreamble, ShardHeader
    from .decomp import partition
    from .quantizer import PQCodebook

    raw = memoryview(archive).cast("B")
    pre, off = ArchivePreamble.unpack(archive)
    n_sh = pre.n_shards
    if len(raw) < off + 8 * n_sh:
        raise FormatError("archive shard index truncated")
    offs = list(struct.unpack_from(f"<{n_sh}Q", raw, off)) + [len(raw)]
    shards = partition(pre.n_planes, pre.n_nodes, n_sh, pre.decomp_mode)
    if len(shards) != n_sh:
        raise FormatError("archive shard count disagrees with the partition")
    P, N = pre.n_planes, pre.n_nodes
    rows, cols = pre.grid.rows, pre.grid.cols
    D = rows * cols
    heads, secs = [], []
    for i in range(n_sh):
        a_, b_ = offs[i], offs[i + 1]
        if not (off + 8 * n_sh <= a_ < b_ <= len(raw)):
            raise FormatError(f"corrupt shard offset index at entry {i}")
        h = ShardHeader.unpack(raw[a_:a_ + HEADER_SIZE])
        if b_ - a_ != HEADER_SIZE + sum(h.section_lengths):
            raise FormatError(f"shard {i} length disagrees with its header")
        if h.n_images != len(shards[i].members):
            raise FormatError("shard image count disagrees with the partition")
        if (h.img_rows, h.img_cols) != (rows, cols):
            raise FormatError("shard image dims disagree with the archive grid")
        o, d = a_ + HEADER_SIZE, {}
        for name, ln in zip(SECTIONS, h.section_lengths):
            d[name] = (o, ln)
            o += ln
        heads.append(h)
        secs.append(d)
    L, bits = heads[0].latent_dim, heads[0].pq_bits
    K = 1 << bits
    if any(h.latent_dim != L or h.pq_bits != bits for h in heads):
        raise FormatError("mixed latent/codebook shapes across shards are not supported")
    lam_bytes = heads[-1].lambda_precision
    if any(h.lambda_precision != lam_bytes for h in heads):
        raise FormatError("mixed lambda precisions across shards are not supported")
    # the member range [lo_s, hi_s) of every shard this call decodes
    rng_ = [sp.range(s) for s in range(n_sh)] if sp is not None else \
        [(0, h.n_images) for h in heads]
    so = _lib.lib()
    arr = np.frombuffer(archive, dtype=np.uint8)
    base_ptr = arr.ctypes.data
    models, cents = [], []
    res_idx, res_off, res_len, res_eb, res_mode = [], [], [], [], []
    exc_idx, exc_src = [], []
    cnt = ctypes.c_int32()
    why = ctypes.c_int32()
    for s, (h, d) in enumerate(zip(heads, secs)):
        n = h.n_images
        lo_s, hi_s = rng_[s]
        wo, wl = d["weights"]
        models.append(AEModel.from_bytes(bytes(raw[wo:wo + wl]), L, D))
        po, pl = d["pq_table"]
        cents.append(PQCodebook.from_bytes(bytes(raw[po:po + pl]), L, K).centroids)
        if d["codes"][1] != (n * L * bits + 7) // 8:
            raise SizeMismatchError(f"code stream is {d['codes'][1]} bytes, expected "
                                    f"{(n * L * bits + 7) // 8}")
        if d["lambdas"][1] != n * 8 * h.lambda_precision:
            raise FormatError("lambda section length mismatch")
        ro, rl = d["residuals"]
        cap = n
        idx = np.empty(cap, np.int32)
        bo = np.empty(cap, np.int64)
        bl = np.empty(cap, np.int64)
        eb = np.empty(cap, np.float64)
        md = np.empty(cap, np.uint8)
        rc = so.mlk_parse_residual_section(
            ctypes.c_void_p(base_ptr + ro), rl, n, rows, cols, ro, cap,
            idx.ctypes.data, bo.ctypes.data, bl.ctypes.data, eb.ctypes.data, md.ctypes.data,
            ctypes.byref(cnt), ctypes.byref(why))
        if rc != 0:
            raise FormatError(_WHY.get(why.value, "corrupt residual section"))
        k = cnt.value
        keep = (idx[:k] >= lo_s) & (idx[:k] < hi_s)
        res_idx.append(idx[:k][keep] - lo_s)
        res_off.append(bo[:k][keep])
        res_len.append(bl[:k][keep])
        res_eb.append(eb[:k][keep])
        res_mode.append(md[:k][keep])
        eo, el = d["exceptions"]
        if el < 4:
            raise FormatError("exceptions section truncated")
        ne = struct.unpack_from("<I", raw, eo)[0]
        rec = 4 + 8 * D
        if el != 4 + ne * rec:
            raise FormatError("exceptions section truncated" if el < 4 + ne * rec
                              else "exceptions section has trailing bytes")
        if ne:
            starts = eo + 4 + rec * np.arange(ne, dtype=np.int64)
            ei = np.frombuffer(archive, np.uint8, ne * rec, eo + 4).reshape(ne, rec)[:, :4]
            ei = np.ascontiguousarray(ei).view("<u4").reshape(-1).astype(np.int64)
            if np.any(ei >= n):
                raise FormatError("exception index out of range")
            keep = (ei >= lo_s) & (ei < hi_s)
            exc_idx.append(ei[keep] - lo_s)
            exc_src.append(starts[keep] + 4)
        else:
            exc_idx.append(np.zeros(0, np.int64))
            exc_src.append(np.zeros(0, np.int64))
    n_res = sum(len(x) for x in res_idx)
    n_exc = sum(len(x) for x in exc_idx)
    # everything but the exception images of members outside the range (the
    # sorted exception list makes this rank's records one run per shard)
    ranges, at = [], 0
    for s, d in enumerate(secs):
        eo = d["exceptions"][0] + 4
        ranges.append((at, eo))
        if len(exc_src[s]):
            ranges.append((int(exc_src[s][0]) - 4, int(exc_src[s][-1]) + 8 * D))
        at = eo + d["exceptions"][1] - 4
    ranges.append((at, len(raw)))
    ranges = [(a_, b_) for a_, b_ in ranges if b_ > a_]
    arc_d = hostio.upload_bytes(archive, dev, ranges if sp is not None else None)
    if sp is not None:
        specs = split_layout(sp, models, rows, cols)
        plane_lo, plane_hi = sp.plane_lo, sp.plane_hi
    else:
        specs = shard_layout(shards, models, N, rows, cols)
        plane_lo, plane_hi = 0, P
    table = _shard_table(specs, D, L)
    img_off = np.array([t.img_off for t in table], dtype=np.int64)
    total = sum(sp_.n_img for sp_ in specs)
    ws = Workspace.get(dev)
    ws.reset()
    # per-image slots and the small host-built tables, one staged copy
    res_slot = np.full(max(total, 1), -1, np.int32)
    if n_res:
        gi = np.concatenate([img_off[s] + res_idx[s] for s in range(n_sh)])
        res_slot[gi] = np.arange(n_res, dtype=np.int32)
    exc_slot = np.full(max(total, 1), -1, np.int32)
    if n_exc:
        gi = np.concatenate([img_off[s] + exc_idx[s] for s in range(n_sh)])
        exc_slot[gi] = np.arange(n_exc, dtype=np.int32)
    lrec = 8 * lam_bytes
    sh_d = ws.stage(np.frombuffer(bytes(table), dtype=np.uint8))
    W = ws.stage(np.stack([m.weights for m in models]).astype(np.float32))
    cents_d = ws.stage(np.stack(cents))
    res_slot_d = ws.stage(res_slot)
    exc_slot_d = ws.stage(exc_slot)
    lam_seg = ws.stage(np.array([d["lambdas"][0] + lrec * rng_[s][0]
                                 for s, d in enumerate(secs)], np.int64))
    lam_len = ws.stage(np.array([lrec * (b_ - a_) for a_, b_ in rng_], np.int64))
    lam_dst = ws.stage(lrec * img_off)
    body = exc_seg = None
    if n_res:
        body = (ws.stage(np.concatenate(res_off)), ws.stage(np.concatenate(res_len)),
                ws.stage(np.concatenate(res_eb)), ws.stage(np.concatenate(res_mode)))
    if n_exc:
        exc_seg = (ws.stage(np.concatenate(exc_src)), ws.stage(np.full(n_exc, 8 * D, np.int64)),
                   ws.stage(8 * D * np.arange(n_exc, dtype=np.int64)))
    ws.flush()
    code_src = [(d["codes"][0], h.n_images, rng_[s][0], rng_[s][1] - rng_[s][0])
                for s, (h, d) in enumerate(zip(heads, secs))]
    return DecodePlan(preamble=pre, shards=shards, specs=specs, table=table, models=models,
                      total=total, n_res=n_res, n_exc=n_exc, L=L, K=K, bits=bits,
                      lam_bytes=lam_bytes, arc_d=arc_d, sh_d=sh_d, W=W, cents=cents_d,
                      res_slot=res_slot_d, exc_slot=exc_slot_d, lam_seg=lam_seg,
                      lam_len=lam_len, lam_dst=lam_dst, code_src=code_src, img_off=img_off,
                      body=body, exc_seg=exc_seg, dgrid=DeviceGrid(pre.grid, dev, L),
                      out_elems=(plane_hi - plane_lo) * N * D, dev=dev, plane_lo=plane_lo,
                      plane_hi=plane_hi)


def run_decode(pl: DecodePlan, check: bool = True, out: torch.Tensor | None = None):
    """The device half of the decode: unpack codes, gather lambdas, inflate +
    varint-decode the residual bodies, gather the exception images, then
    mlk_decode writes every image at its dataset address in `out` (flat,
    the plan's planes x all nodes).  check: raise FormatError on corrupt
    residual streams (one small D2H); the timed device loop passes False
    after a checked run."""
    dev = pl.dev
    D = pl.preamble.grid.rows * pl.preamble.grid.cols
    L, total = pl.L, pl.total
    i64 = dict(dtype=torch.int64, device=dev)
    ws = Workspace.get(dev)
    codes16 = ws.tensor("dec_codes16", (max(1, total) * L,), torch.int16)
    for s, (co, n_img, lo_s, cnt_s) in enumerate(pl.code_src):
        if not cnt_s:
            continue
        o = int(pl.img_off[s]) * L
        if lo_s == 0 and cnt_s == n_img:
            call("mlk_unpack_indices", pl.arc_d.data_ptr() + co, n_img * L, pl.bits,
                 codes16.data_ptr() + 2 * o)
        else:
            full = ws.tensor(f"dec_codes_full{s}", (n_img * L,), torch.int16)
            call("mlk_unpack_indices", pl.arc_d.data_ptr() + co, n_img * L, pl.bits,
                 full.data_ptr())
            codes16[o:o + cnt_s * L].copy_(full[lo_s * L:(lo_s + cnt_s) * L])
    codes = ws.tensor("dec_codes", (max(1, total) * L,), torch.uint8)
    codes.copy_(codes16)
    pl.codes = codes
    lam_raw = ws.tensor("dec_lamraw", (max(1, total) * 8 * pl.lam_bytes,), torch.uint8)
    call("mlk_gather_segments", pl.arc_d, pl.lam_seg, pl.lam_len, len(pl.code_src), lam_raw,
         pl.lam_dst)
    lamq = lam_raw.view(torch.float32 if pl.lam_bytes == 4 else torch.float64).to(torch.float64)
    n_res = pl.n_res
    if n_res:
        body_off, body_len, res_eb_d, res_mode_d = pl.body
        icap = 10 * D + 64
        raw_d = ws.tensor("dec_inflate", (n_res * icap,), torch.uint8)
        raw_off = torch.arange(0, n_res * icap, icap, **i64)
        raw_len = ws.tensor("dec_rawlen", (n_res,), torch.int64)
        call("mlk_zlib_decompress", pl.arc_d, body_off, body_len, n_res, raw_d, raw_off, icap,
             raw_len)
        vals = ws.tensor("dec_vals", (n_res * D,), torch.int64)
        consumed = ws.tensor("dec_consumed", (n_res,), torch.int64)
        call("mlk_varint_decode_batch", raw_d, raw_off, raw_len, n_res,
             torch.full((n_res,), D, **i64), vals, torch.arange(0, n_res * D, D, **i64),
             consumed)
        if check:
            rl, con = _d2h(raw_len, consumed)
            if np.any(rl < 0):
                raise FormatError("corrupt residual stream")
            if np.any(con == -1):
                raise FormatError("varint stream truncated")
            if np.any(con == -2):
                raise FormatError("varint value exceeds 64 bits")
            if np.any(con != rl):
                raise FormatError("residual stream has trailing bytes")
    else:
        vals = torch.zeros(1, **i64)
        res_eb_d = torch.zeros(1, dtype=torch.float64, device=dev)
        res_mode_d = torch.zeros(1, dtype=torch.uint8, device=dev)
    exc_img = ws.tensor("dec_exc", (max(1, pl.n_exc) * D,), torch.float64)
    if pl.n_exc:
        ex_src, ex_len, ex_dst = pl.exc_seg
        call("mlk_gather_segments", pl.arc_d, ex_src, ex_len, pl.n_exc,
             exc_img.view(torch.uint8), ex_dst)
    if out is None:
        out = torch.empty(pl.out_elems + 2, dtype=torch.float64, device=dev)
    pl.neg = ws.tensor("dec_neg", (1,), torch.int32)
    pl.neg.zero_()
    if total:
        call("mlk_decode", pl.sh_d, len(pl.specs), total, pl.dgrid.addr, pl.W, L, pl.cents,
             pl.K, codes, pl.res_slot, vals, res_eb_d, res_mode_d, lamq, pl.exc_slot, exc_img,
             1e-12, out, pl.neg)
    return out


def decoded_negative(pl: DecodePlan) -> bool:
    """Whether the last run_decode of `pl` wrote a value < 0 (one int D2H)."""
    return bool(int(pl.neg.item()))


def decode_archive(archive, dev) -> DecodedArchive:
    """Parse and decode a whole archive on `dev` (prepare_decode + run_decode)."""
    pl = prepare_decode(archive, dev)
    out = run_decode(pl)
    return DecodedArchive(preamble=pl.preamble, shards=pl.shards, out=out, specs=pl.specs,
                          table=pl.table, sh_d=pl.sh_d, W=pl.W, cents=pl.cents, codes=pl.codes,
                          L=pl.L, K=pl.K, lam_bytes=pl.lam_bytes, dgrid=pl.dgrid)


def decompress_device(archive, dev) -> np.ndarray:
    """Decode an archive on `dev`; returns the (P, N, R, C) array.  Raises
    ConfigError, like FDataset (fdata.py:70-103), if a value is negative --
    checked on the device, so the host never rescans the array."""
    pl = prepare_decode(archive, dev)
    out = run_decode(pl)
    pre = pl.preamble
    g = pre.grid
    if decoded_negative(pl):
        raise ConfigError("histogram values must be non-negative")
    return hostio.download_pinned_array(out[:pre.n_planes * pre.n_nodes * g.rows * g.cols],
                                        (pre.n_planes, pre.n_nodes, g.rows, g.cols))


def shard_layout(shards, models, n_nodes, rows, cols, node_lo=0):
    """Device addressing of each shard in a (P, n_nodes, rows*cols) buffer whose
    first node is `node_lo` (a rank's node slab)."""
    D = rows * cols
    out = []
    for sh, m in zip(shards, models):
        (p0, p1), (x0, x1) = sh.planes_range, sh.nodes_range
        out.append(ShardWork(wid=sh.worker_id, n_img=len(sh.members),
                             base=(p0 * n_nodes + (x0 - node_lo)) * D,
                             plane_stride=n_nodes * D, block=x1 - x0, model=m, rows=rows,
                             cols=cols, plane0=p0))
    return out


def split_layout(sp, models, rows, cols):
    """ShardWork of rank sp.rank's member range of every shard
    (distributed.SplitPlan) in an f0 buffer holding planes
    [sp.plane_lo, sp.plane_hi) x all nodes."""
    D = rows * cols
    N = sp.n_nodes
    out = []
    for s, sh in enumerate(sp.shards):
        a, e = sp.range(s)
        (p0, _), (x0, x1) = sh.planes_range, sh.nodes_range
        out.append(ShardWork(wid=sh.worker_id, n_img=e - a,
                             base=((p0 - sp.plane_lo) * N + x0) * D, plane_stride=N * D,
                             block=x1 - x0, model=models[s], rows=rows, cols=cols, j0=a,
                             n_full=len(sh.members)))
    return out


def evaluate_device(orig, dec: DecodedArchive, dev) -> dict:
    """Per-image final errors, AE-only errors and moments for evaluate(),
    against the archive decoded on the device (no host round trip)."""
    P, N = orig.n_planes, orig.n_nodes
    D = orig.grid.rows * orig.grid.cols
    total = P * N
    dgrid = dec.dgrid
    a = hostio.upload_planes(np.ascontiguousarray(orig.data, dtype=np.float64), dev)
    b = dec.out
    f64 = dict(dtype=torch.float64, device=dev)
    err = torch.empty(total, **f64)
    sse = torch.empty(total, **f64)
    qa = torch.empty((total, 4), **f64)
    qb = torch.empty((total, 4), **f64)
    ext = torch.empty((total, 2), **f64)
    call("mlk_compare", a, b, total, dgrid.addr, err, sse, qa, qb, ext)
    # AE-only errors through the exact recheck kernel (shard order)
    from .decomp import shard_dataset_index
    order = np.concatenate([shard_dataset_index(sh, N) for sh in dec.shards])
    order_d = torch.from_numpy(order).to(dev)
    stats = torch.zeros((total, 4), **f64)
    stats[:, 0] = ext[order_d, 0]
    stats[:, 1] = ext[order_d, 1]
    flags = torch.full((total,), 4, dtype=torch.uint8, device=dev)
    ae = torch.empty(total, **f64)
    call("mlk_recheck", a, stats, dec.sh_d, len(dec.specs), total, dgrid.addr, dec.W, dec.L,
         dec.cents, dec.K, dec.codes, dec.preamble.tau, flags, ae)
    span = float(ext[:, 0].max() - ext[:, 1].min())
    pd = float(np.sqrt(float(sse.sum()) / orig.data.size) / span) if span > 0 else 0.0
    ae_h = np.empty(total)
    ae_h[order] = ae.cpu().numpy()
    return {"per_image": err.cpu().numpy(), "q_orig": qa.cpu().numpy(),
            "q_rec": qb.cpu().numpy(), "pd_nrmse": pd, "ae_err": ae_h}


