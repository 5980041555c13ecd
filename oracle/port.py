"""numpy restatement of the reference compress/decompress path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Every function cites the
reference file:line it restates (paths relative to
/root/reference/pkg/src/mlk/).  Inputs are plain numpy arrays so the checker
shares no code with the product package.

Host-dependent arithmetic the reference inherits from numpy, and how this
restatement pins it:
  * AE encode/decode matmuls -> explicit OpenBLAS orders in ckernels.c
    (oracle_encode / oracle_decode); the decode tree columns are probed from
    this host's numpy at first use (``decode_tree_cols``);
  * per-image NRMSE / sums -> numpy's own pairwise reductions (same calls);
  * exp/log scalars and arrays -> numpy (same calls as the reference);
  * DEFLATE -> the host's zlib 1.3 at level 6 (same call as the reference).
"""

from __future__ import annotations

import functools
import hashlib
import json
import struct
import zlib
from dataclasses import dataclass, field

import numpy as np

from oracle import native

CONVERGED, MAX_ITER, DEGENERATE = 0, 1, 2
FLOOR = 1e-12
KMEANS_ITERS = 25
SPAN = 2.0 ** -20
STEPS = 20


# ---------------------------------------------------------------------------
# configuration mirror (pipeline.py:36-89, lagrange.py:42-56)

@dataclass(frozen=True)
class Newton:
    step: float = 1.0
    max_iter: int = 50
    tol: float = 1e-13
    floor: float = FLOOR
    retry: bool = False
    retry_step: float = 0.01
    retry_max_iter: int = 400


@dataclass(frozen=True)
class Cfg:
    shards: int = 2
    mode: str = "col"
    tau: float = 1e-3
    latent_dim: int = 4
    pq_bits: int = 4
    lambda_precision: str = "f32"
    seed: int = 0
    newton: Newton = field(default_factory=Newton)
    digest: bytes = b"\0" * 32     # PipelineConfig.digest() of the caller's config


@dataclass
class Grid:
    v_perp: np.ndarray
    v_par: np.ndarray
    vol: np.ndarray
    mass: float

    @property
    def shape(self):
        return self.vol.shape

    def cells(self):
        r, c = self.vol.shape
        vpar = np.broadcast_to(self.v_par, (r, c)).reshape(-1)
        vperp = np.broadcast_to(self.v_perp[:, None], (r, c)).reshape(-1)
        return self.vol.reshape(-1), vpar, vperp


# ---------------------------------------------------------------------------
# decomposition (decomp.py:61-113)

def blocks(count: int, parts: int):
    """decomp.py:61-70 -- first count % parts blocks get one extra."""
    q, r = divmod(count, parts)
    out, lo = [], 0
    for i in range(parts):
        hi = lo + q + (i < r)
        out.append((lo, hi))
        lo = hi
    return out


def shard_members(n_planes: int, n_nodes: int, n_shards: int, mode: str):
    """decomp.py:73-105 as (planes, nodes) index arrays per shard."""
    out = []
    if mode == "col":
        for lo, hi in blocks(n_nodes, n_shards):
            nodes = np.arange(lo, hi)
            out.append((np.repeat(np.arange(n_planes), hi - lo), np.tile(nodes, n_planes)))
        return out
    per_plane = [n_shards // n_planes + (p < n_shards % n_planes) for p in range(n_planes)]
    for p, k in enumerate(per_plane):
        for lo, hi in blocks(n_nodes, k):
            out.append((np.full(hi - lo, p), np.arange(lo, hi)))
    return out


def mix_seed(seed: int, wid: int) -> int:
    """decomp.py:108-113 (SplitMix64 finaliser)."""
    m = (1 << 64) - 1
    z = (seed + 0x9E3779B97F4A7C15 * (wid + 1)) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


# ---------------------------------------------------------------------------
# AE training: selection + Adam, autoencoder.py:77-177

def select_training(planes, nodes, scheme: str, n_planes: int, seed: int, wid: int):
    """decomp.py:116-153 on a shard given as (plane, node) member arrays."""
    rng = np.random.Generator(np.random.PCG64(mix_seed(seed, wid)))
    n = len(planes)
    row_based = scheme.startswith("row")
    single = len(set(planes.tolist())) == 1
    if row_based and not single and n_planes > 1:
        raise ValueError("row scheme needs row-wise shards")
    if not row_based and single and n_planes > 1:
        raise ValueError("col scheme needs column-wise shards")
    frac = int(scheme[-2:]) / 100 if scheme[-2:].isdigit() else None
    if scheme in ("row", "col"):
        return np.arange(n)
    if row_based:
        return np.sort(rng.choice(n, size=max(1, int(n * frac)), replace=False))
    block = sorted(set(nodes.tolist()))
    if scheme == "colfst":
        return np.nonzero(planes == min(planes))[0]
    if scheme == "colrand":
        return np.sort(rng.choice(n, size=len(block), replace=False))
    pos = {x: j for j, x in enumerate(block)}
    by_node = [[] for _ in block]
    for i, x in enumerate(nodes.tolist()):
        by_node[pos[x]].append(i)
    picks = np.array([c[rng.integers(len(c))] for c in by_node])
    if scheme == "colrandind":
        return np.sort(picks)
    return np.sort(rng.choice(picks, size=max(1, int(len(block) * frac)), replace=False))


def ae_train(images, lr=0.001, batch=128, epochs=100, beta1=0.9, beta2=0.999, eps=1e-8,
             seed=0, init_w=None, latent_dim=4):
    """autoencoder.train (137-177) with fit_normalizer (77-84) and
    _loss_and_grad_normalized (127-134); returns (W f32, mean, std) or
    raises FloatingPointError(epoch, mse) where the reference raises
    TrainingDivergedError."""
    x = np.asarray(images, dtype=np.float64)
    x = x.reshape(len(x), -1)
    mean = float(np.mean(x))
    std = max(float(np.std(x)), 1e-30)
    x = (x - mean) / std
    n, d = x.shape
    rng = np.random.Generator(np.random.PCG64(seed))
    if init_w is not None:
        w = np.asarray(init_w, dtype=np.float32).astype(np.float64)
    else:
        bound = np.sqrt(6.0 / (latent_dim + d))
        w = rng.uniform(-bound, bound, size=(latent_dim, d))
    m = np.zeros_like(w)
    v = np.zeros_like(w)
    t = 0
    for epoch in range(epochs):
        order = rng.permutation(n)
        for start in range(0, n, batch):
            xb = x[order[start:start + batch]]
            b = len(xb)
            z = xb @ w.T
            err = z @ w - xb
            mse = float(np.mean(err ** 2))
            grad = 2.0 / (b * d) * (z.T @ err + (err @ w.T).T @ xb)
            if not np.isfinite(mse):
                raise FloatingPointError(epoch, mse)
            t += 1
            m = beta1 * m + (1 - beta1) * grad
            v = beta2 * v + (1 - beta2) * grad ** 2
            mhat = m / (1 - beta1 ** t)
            vhat = v / (1 - beta2 ** t)
            w -= lr * mhat / (np.sqrt(vhat) + eps)
    return w.astype(np.float32), mean, std


# ---------------------------------------------------------------------------
# autoencoder contractions (autoencoder.py:99-110)

@functools.lru_cache(maxsize=None)
def decode_tree_cols(d: int, l: int) -> bytes:
    """Columns where this host's OpenBLAS sums the L=4 decode products as
    (p0+p1)+(p2+p3) instead of left to right (blocked-kernel path)."""
    out = np.zeros(d, dtype=np.uint8)
    if l != 4:
        return out.tobytes()
    rng = np.random.default_rng(20221221)
    n = max(512, int(1e6 // (l * d)) + 64)
    w = rng.standard_normal((l, d)).astype(np.float32).astype(np.float64)
    z = (rng.standard_normal((n, l)) * 37.0).astype(np.float32).astype(np.float64)
    from threadpoolctl import threadpool_limits  # the reference ran on one BLAS thread
    with threadpool_limits(limits=1, user_api="blas"):
        ref = z @ w
    p = [z[:, k:k + 1] * w[k][None, :] for k in range(4)]
    seq = ((p[0] + p[1]) + p[2]) + p[3]
    tree = (p[0] + p[1]) + (p[2] + p[3])
    for j in np.flatnonzero((seq != ref).any(axis=0)):
        if (tree[:, j] == ref[:, j]).all():
            out[j] = 1
    return out.tobytes()


def ae_encode(w32, mean, std, flat):
    """autoencoder.py:99-103 with OpenBLAS's accumulation order."""
    return native.encode(flat, w32, mean, std)


def ae_decode(w32, mean, std, lat):
    """autoencoder.py:106-110 with OpenBLAS's bracketing."""
    n, l = lat.shape
    d = w32.shape[1]
    tc = np.frombuffer(decode_tree_cols(d, l), dtype=np.uint8)
    if n * l * d <= 1e6:
        tc = np.zeros_like(tc)
    return native.decode(lat, w32, mean, std, tc)


# ---------------------------------------------------------------------------
# product quantiser (quantizer.py:53-138)

def nearest(v, c):
    """quantizer.py:94-96 -- first minimum wins."""
    return np.argmin(np.abs(v[:, None] - c[None, :]), axis=1)


def kmeans_draws(n: int, k: int, seed: int):
    """The PCG64 draws kmeans_1d consumes (quantizer.py:68,77): one bounded
    integer, then one double per Generator.choice call."""
    g = np.random.Generator(np.random.PCG64(seed))
    first = int(g.integers(n))
    return first, np.array([g.random() for _ in range(k - 1)])


def kmeans(values, k: int, seed: int):
    """quantizer.py:53-91, with Generator.choice(p=...) written out as
    searchsorted(cumsum(p)/cumsum(p)[-1], u, 'right') on the same draws."""
    v = np.asarray(values, dtype=np.float64).ravel()
    uniq = np.unique(v)
    if uniq.size <= k:
        return np.sort(np.concatenate([uniq, np.repeat(uniq[-1], k - uniq.size)]))
    first, us = kmeans_draws(v.size, k, seed)
    cent = np.empty(k)
    cent[0] = v[first]
    d2 = (v - cent[0]) ** 2
    for i in range(1, k):
        tot = d2.sum()
        if tot <= 0:
            cent[i:] = cent[0]
            break
        cdf = np.cumsum(d2 / tot)
        cdf /= cdf[-1]
        cent[i] = v[int(np.searchsorted(cdf, us[i - 1], side="right"))]
        d2 = np.minimum(d2, (v - cent[i]) ** 2)
    lab = nearest(v, cent)
    for _ in range(KMEANS_ITERS):
        for j in range(k):
            hit = lab == j
            if hit.any():
                cent[j] = v[hit].mean()
            else:
                cent[j] = v[np.argmax(np.abs(v - cent[lab]))]
        nxt = nearest(v, cent)
        if np.array_equal(nxt, lab):
            break
        lab = nxt
    return np.sort(cent)


def pq_codebook(lat, k: int, seed: int):
    """quantizer.py:99-108 -> (L, k) float32."""
    return np.array([kmeans(lat[:, d], k, seed + d) for d in range(lat.shape[1])],
                    dtype=np.float32)


def pq_indices(cents32, lat):
    """quantizer.py:111-120 before packing -> (N, L) uint16."""
    c = cents32.astype(np.float64)
    return np.stack([nearest(lat[:, d], c[d]) for d in range(lat.shape[1])],
                    axis=1).astype(np.uint16)


def pq_lookup(cents32, idx):
    """quantizer.py:123-138 after unpacking."""
    c = cents32.astype(np.float64)
    return np.stack([c[d][idx[:, d]] for d in range(idx.shape[1])], axis=1)


# ---------------------------------------------------------------------------
# metrics (qoi.py:60-119)

def nrmse_rows(orig, rec):
    """qoi.py:107-119 (numpy pairwise mean, same calls)."""
    n = orig.shape[0]
    o = orig.reshape(n, -1)
    r = rec.reshape(n, -1)
    span = o.max(axis=1) - o.min(axis=1)
    rms = np.sqrt(np.mean((o - r) ** 2, axis=1))
    out = np.empty(n)
    ok = span > 0
    out[ok] = rms[ok] / span[ok]
    out[~ok] = np.where(rms[~ok] == 0.0, 0.0, np.inf)
    return out


def nrmse_flat(u, f):
    """qoi.py:79-90."""
    u = np.asarray(u, dtype=np.float64).ravel()
    f = np.asarray(f, dtype=np.float64).ravel()
    span = float(np.max(u) - np.min(u))
    if span == 0.0:
        if np.array_equal(u, f):
            return 0.0
        raise ValueError("reference range is zero but arrays differ")
    return float(np.sqrt(np.mean((u - f) ** 2)) / span)


def moments(images, grid: Grid):
    """qoi.py:60-76 -> (N, 4) [n, u_par, t_perp, t_par], NaN where n <= 0."""
    fv = images * grid.vol
    n = np.einsum("irc->i", fv)
    m = grid.mass
    with np.errstate(invalid="ignore", divide="ignore"):
        u = np.einsum("irc,c->i", fv, grid.v_par) / n
        tp = 0.5 * m * np.einsum("irc,r->i", fv, grid.v_perp ** 2) / n
        dv = grid.v_par[None, None, :] - u[:, None, None]
        tl = 0.5 * m * np.einsum("irc,irc->i", fv, dv ** 2) / n
    out = np.stack([n, u, tp, tl], axis=1)
    out[~(n > 0), 1:] = np.nan
    return out


# ---------------------------------------------------------------------------
# residual stage (residual.py:60-191)

_PAYLOAD_HEAD = struct.Struct("<BHHd")


def zigzag(q):
    q = np.asarray(q, dtype=np.int64)
    return ((q << 1) ^ (q >> 63)).astype(np.uint64)


def unzigzag(z):
    z = np.asarray(z, dtype=np.uint64)
    return ((z >> np.uint64(1)) ^ (np.uint64(0) - (z & np.uint64(1)))).astype(np.int64)


def payload_quantized(r, eb):
    """residual.py:60-72."""
    q = np.rint(r / (2.0 * eb))
    if np.any(np.abs(q) >= 2.0 ** 62):
        raise ValueError("error bound too small for this residual range")
    body = zlib.compress(native.varint_encode(zigzag(q.astype(np.int64).reshape(-1))), 6)
    return _PAYLOAD_HEAD.pack(0, r.shape[0], r.shape[1], eb) + body


def payload_lossless(r):
    """residual.py:74-79."""
    bits = np.ascontiguousarray(r, dtype="<f8").reshape(-1).view(np.uint64)
    body = zlib.compress(native.varint_encode(bits), 6)
    return _PAYLOAD_HEAD.pack(1, r.shape[0], r.shape[1], 0.0) + body


def payload_decode(p: bytes):
    """residual.py:81-98."""
    if len(p) < _PAYLOAD_HEAD.size:
        raise ValueError("residual payload shorter than its header")
    mode, rows, cols, eb = _PAYLOAD_HEAD.unpack_from(p, 0)
    raw = zlib.decompress(p[_PAYLOAD_HEAD.size:])
    codes, used = native.varint_decode(raw, rows * cols)
    if used != len(raw):
        raise ValueError("residual stream has trailing bytes")
    if mode == 0:
        return (unzigzag(codes).astype(np.float64) * (2.0 * eb)).reshape(rows, cols)
    if mode == 1:
        return codes.view(np.float64).reshape(rows, cols).copy()
    raise ValueError(f"unknown residual payload mode {mode}")


def search_bound(orig, rec, tau):
    """residual.py:129-173; returns (eb, lossless, probes)."""
    n = len(orig)
    fo = orig.reshape(n, -1)
    eb_hi = tau * float((fo.max(axis=1) - fo.min(axis=1)).max())
    if eb_hi <= 0:
        return eb_hi, True, []
    res = fo - rec.reshape(n, -1)
    probes = []

    def ok(eb):
        corr = rec + (np.rint(res / (2.0 * eb)) * (2.0 * eb)).reshape(rec.shape)
        good = bool(np.all(nrmse_rows(orig, corr) <= tau))
        probes.append((float(eb), good))
        return good

    if ok(eb_hi):
        return eb_hi, False, probes
    lo, hi = np.log(eb_hi * SPAN), np.log(eb_hi)
    best = None
    for _ in range(STEPS):
        mid = 0.5 * (lo + hi)
        if ok(np.exp(mid)):
            best, lo = np.exp(mid), mid
        else:
            hi = mid
    if best is not None:
        return float(best), False, probes
    low = eb_hi * SPAN
    return float(low), not ok(low), probes


# ---------------------------------------------------------------------------
# Lagrange projection (lagrange.py:68-253)

def apply_multipliers(imgs, lams, grid: Grid, qois, floor=FLOOR):
    """lagrange.py:152-185."""
    n = imgs.shape[0]
    flat = imgs.reshape(n, -1)
    vol, vpar, vperp = grid.cells()
    hm = 0.5 * grid.mass
    rows = [vol, vol * vpar, hm * vol * vperp ** 2]
    shared = [r / np.max(np.abs(r)) for r in rows]
    a3 = hm * vol[None, :] * (vpar[None, :] - qois[:, 1:2]) ** 2
    s3 = np.max(np.abs(a3), axis=1)
    a3 = a3 / np.where(s3 > 0, s3, 1.0)[:, None]
    t = (lams[:, 0:1] * shared[0][None, :] + lams[:, 1:2] * shared[1][None, :]
         + lams[:, 2:3] * shared[2][None, :] + lams[:, 3:4] * a3)
    top = flat.max(axis=1)
    out = np.maximum(flat, floor * top[:, None]) * np.exp(-np.clip(t, -700.0, 700.0))
    flat_img = ~(top > 0)
    out[flat_img] = flat[flat_img]
    return out.reshape(imgs.shape)


def narrow(lam, precision):
    """lagrange.py:239-253."""
    if precision == "f64":
        return lam.copy(), False
    with np.errstate(over="ignore"):
        n32 = lam.astype(np.float32)
    return n32.astype(np.float64), bool(np.any(~np.isfinite(n32)))


# ---------------------------------------------------------------------------
# container (container.py:30-216)

_HDR = struct.Struct("<4sHBB6IIHHBBH")
_PRE = struct.Struct("<4sHBxIIIHHqdQ32s")


def shard_blob(lam_bytes, n_img, rows, cols, L, bits, sections):
    """container.py:90-95 with sections in _SECTIONS order."""
    return _HDR.pack(b"MLK1", 1, 0, lam_bytes, *[len(s) for s in sections], n_img, rows,
                     cols, L, bits, 0) + b"".join(sections)


def split_blob(blob):
    """container.py:98-109."""
    f = _HDR.unpack_from(blob, 0)
    if f[0] != b"MLK1":
        raise ValueError("bad shard magic")
    lens = f[4:10]
    secs, off = [], _HDR.size
    for ln in lens:
        secs.append(blob[off:off + ln])
        off += ln
    if off != len(blob):
        raise ValueError("shard length mismatch")
    return dict(lam_bytes=f[3], n_img=f[10], rows=f[11], cols=f[12], L=f[13],
                bits=f[14]), secs


def archive(grid: Grid, cfg: Cfg, n_planes, n_nodes, timestep, blobs):
    """container.py:118-195."""
    head = _PRE.pack(b"MLKA", 1, {"row": 0, "col": 1}[cfg.mode], len(blobs), n_planes,
                     n_nodes, grid.vol.shape[0], grid.vol.shape[1], timestep, cfg.tau,
                     cfg.seed, cfg.digest)
    head += (struct.pack("<d", grid.mass) + grid.v_perp.astype("<f8").tobytes()
             + grid.v_par.astype("<f8").tobytes() + grid.vol.astype("<f8").tobytes())
    pos = len(head) + 8 * len(blobs)
    offs = []
    for b in blobs:
        offs.append(pos)
        pos += len(b)
    return head + struct.pack(f"<{len(offs)}Q", *offs) + b"".join(blobs)


def unarchive(raw):
    """container.py:198-216 (+ preamble unpack 146-179)."""
    (magic, ver, mode, n_sh, n_pl, n_no, rows, cols, ts, tau, seed,
     dig) = _PRE.unpack_from(raw, 0)
    if magic != b"MLKA":
        raise ValueError("bad archive magic")
    off = _PRE.size
    mass = struct.unpack_from("<d", raw, off)[0]
    off += 8
    vperp = np.frombuffer(raw, "<f8", rows, off).copy()
    off += 8 * rows
    vpar = np.frombuffer(raw, "<f8", cols, off).copy()
    off += 8 * cols
    vol = np.frombuffer(raw, "<f8", rows * cols, off).reshape(rows, cols).copy()
    off += 8 * rows * cols
    offs = list(struct.unpack_from(f"<{n_sh}Q", raw, off)) + [len(raw)]
    blobs = [raw[offs[i]:offs[i + 1]] for i in range(n_sh)]
    meta = dict(mode="row" if mode == 0 else "col", n_planes=n_pl, n_nodes=n_no,
                timestep=ts, tau=tau, seed=seed)
    return Grid(vperp, vpar, vol, mass), meta, blobs


# ---------------------------------------------------------------------------
# per-shard compress (pipeline.py:196-320)

@dataclass
class ShardOut:
    blob: bytes
    final: np.ndarray
    ae_err: np.ndarray
    stage4_err: np.ndarray
    latents: np.ndarray
    cents: np.ndarray
    idx: np.ndarray
    selected: np.ndarray
    eb: float
    lossless: bool
    probes: list
    payloads: list
    qoi_stored: np.ndarray
    raw_lams: np.ndarray
    lams: np.ndarray
    status: np.ndarray
    iters: np.ndarray
    final_err: np.ndarray
    exceptions: list
    n_converged: int


def compress_shard(images, grid: Grid, cfg: Cfg, model, wid: int) -> ShardOut:
    w32, mean, std = model
    n, rows, cols = images.shape
    flat = images.reshape(n, -1)
    seed = mix_seed(cfg.seed, wid)
    lat = ae_encode(w32, mean, std, flat)
    cents = pq_codebook(lat, 2 ** cfg.pq_bits, seed)
    idx = pq_indices(cents, lat)
    codes = native.pack_indices(idx.reshape(-1), cfg.pq_bits)
    rec = ae_decode(w32, mean, std, pq_lookup(cents, idx)).reshape(images.shape)

    ae_err = nrmse_rows(images, rec)
    bad = ~np.isfinite(ae_err)
    exc = set(np.flatnonzero(bad).tolist())
    sel = np.flatnonzero(~bad & (ae_err > cfg.tau))
    eb, lossless, probes, payloads = 0.0, False, [], []
    corrected = rec.copy()
    if sel.size:
        eb, lossless, probes = search_bound(images[sel], rec[sel], cfg.tau)
        for i in sel:
            r = images[i] - rec[i]
            p = payload_lossless(r) if lossless else payload_quantized(r, eb)
            payloads.append(p)
            corrected[i] = corrected[i] + payload_decode(p)
    stage4 = nrmse_rows(images, corrected)

    q = moments(images, grid)
    qst = q.astype(np.float32).astype(np.float64) if cfg.lambda_precision == "f32" else q.copy()
    vol, vpar, vperp = grid.cells()
    nw = cfg.newton
    raw, status, iters = native.project_batch(corrected.reshape(n, -1), vol, vpar, vperp,
                                              grid.mass, qst, nw.floor, nw.step, nw.max_iter,
                                              nw.tol, nw.retry, nw.retry_step,
                                              nw.retry_max_iter)
    lams = np.zeros((n, 4))
    n_conv = 0
    for i in range(n):
        if i in exc:
            continue
        if status[i] != CONVERGED:
            exc.add(i)
            continue
        lc, over = narrow(raw[i], cfg.lambda_precision)
        if over:
            exc.add(i)
            continue
        lams[i] = lc
        n_conv += 1
    final = apply_multipliers(corrected, lams, grid, qst, floor=nw.floor)
    ferr = nrmse_rows(images, final)
    exc.update(np.flatnonzero(~(ferr <= cfg.tau)).tolist())
    exc = sorted(exc)
    if exc:
        lams[exc] = 0.0
        qst[exc] = 0.0
        final[exc] = images[exc]

    dt = "<f4" if cfg.lambda_precision == "f32" else "<f8"
    res_sec = struct.pack("<dI", eb, len(sel)) + b"".join(
        struct.pack("<II", int(i), len(p)) + p for i, p in zip(sel, payloads))
    lam_sec = np.concatenate([lams, qst], axis=1).astype(dt).tobytes()
    exc_sec = struct.pack("<I", len(exc)) + b"".join(
        struct.pack("<I", i) + np.ascontiguousarray(images[i], dtype="<f8").tobytes()
        for i in exc)
    weights = struct.pack("<dd", mean, std) + np.asarray(w32, dtype="<f4").tobytes()
    blob = shard_blob(4 if cfg.lambda_precision == "f32" else 8, n, rows, cols,
                      cfg.latent_dim, cfg.pq_bits,
                      [weights, codes, cents.astype("<f4").tobytes(), res_sec, lam_sec,
                       exc_sec])
    return ShardOut(blob=blob, final=final, ae_err=ae_err, stage4_err=stage4, latents=lat,
                    cents=cents, idx=idx, selected=sel, eb=eb, lossless=lossless,
                    probes=probes, payloads=payloads, qoi_stored=qst, raw_lams=raw,
                    lams=lams, status=status, iters=iters, final_err=ferr,
                    exceptions=exc, n_converged=n_conv)


def manifest_nbytes(data, grid: Grid, timestep=0) -> int:
    """fdata.py:399-409 (ratio numerator)."""
    p, n, r, c = data.shape
    man = {"n_planes": p, "n_nodes": n, "rows": r, "cols": c, "timestep": timestep,
           "endianness": "little", "payload": "payload.f64", "mass": grid.mass,
           "v_perp": grid.v_perp.tolist(), "v_par": grid.v_par.tolist(),
           "vol": grid.vol.tolist()}
    return data.size * 8 + len(json.dumps(man, indent=1))


def compress(data, grid: Grid, cfg: Cfg, models, timestep=0, threads=1):
    """pipeline.py:323-391: shards on a thread pool like the reference's
    workers (pipeline.py:338-342; results do not depend on the worker count,
    pipeline.py:4-7), then the archive and the report.  Returns (archive,
    report, shards)."""
    P, N = data.shape[:2]
    members = shard_members(P, N, cfg.shards, cfg.mode)

    def job(wid):
        pl, no = members[wid]
        return compress_shard(data[pl, no], grid, cfg, models[wid], wid)

    if threads > 1:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=threads) as ex:
            outs = list(ex.map(job, range(len(members))))
    else:
        outs = [job(w) for w in range(len(members))]
    arc = archive(grid, cfg, P, N, timestep, [o.blob for o in outs])
    recon = np.empty_like(data)
    for (pl, no), o in zip(members, outs):
        recon[pl, no] = o.final
    report = make_report(data, recon, grid, arc, outs, cfg.tau)
    return arc, report, outs


def make_report(data, recon, grid, arc, outs, tau):
    """pipeline.py:367-391 (timings omitted)."""
    P, N, r, c = data.shape
    oi = data.reshape(P * N, r, c)
    ri = recon.reshape(P * N, r, c)
    qo, qr = moments(oi, grid), moments(ri, grid)
    ok = qo[:, 0] > 0
    names = ("n", "u_par", "t_perp", "t_par")
    qerr = {nm: nrmse_flat(qo[ok, k], qr[ok, k]) for k, nm in enumerate(names)}
    n_tot = sum(o.final.shape[0] for o in outs)
    ae = np.concatenate([o.ae_err for o in outs])
    return dict(
        pd_nrmse=nrmse_flat(oi.reshape(-1), ri.reshape(-1)),
        per_image_nrmse=nrmse_rows(oi, ri),
        qoi_nrmse=qerr,
        max_qoi_nrmse=max(qerr.values()),
        compression_ratio=manifest_nbytes(data, grid) / len(arc),
        ae_accuracy=float(np.mean(np.where(np.isfinite(ae), ae, np.inf) <= tau)),
        residual_fraction=sum(o.selected.size for o in outs) / n_tot,
        convergence_fraction=sum(o.n_converged for o in outs) / n_tot,
        exception_count=sum(len(o.exceptions) for o in outs),
    )


# ---------------------------------------------------------------------------
# decompress (pipeline.py:397-440)

def decode_shard(blob, grid: Grid):
    h, (wsec, codes, ptab, rsec, lsec, esec) = split_blob(blob)
    n, rows, cols, L, bits = h["n_img"], h["rows"], h["cols"], h["L"], h["bits"]
    d = rows * cols
    mean, std = struct.unpack_from("<dd", wsec, 0)
    w32 = np.frombuffer(wsec, "<f4", offset=16).reshape(L, d)
    cents = np.frombuffer(ptab, "<f4").reshape(L, 1 << bits)
    idx = native.unpack_indices(codes, n * L, bits).reshape(n, L).astype(np.int64)
    rec = ae_decode(w32, mean, std, pq_lookup(cents, idx)).reshape(n, rows, cols)
    corrected = rec.copy()
    _, count = struct.unpack_from("<dI", rsec, 0)
    off = 12
    for _ in range(count):
        i, ln = struct.unpack_from("<II", rsec, off)
        off += 8
        corrected[i] = corrected[i] + payload_decode(rsec[off:off + ln])
        off += ln
    dt = "<f4" if h["lam_bytes"] == 4 else "<f8"
    lq = np.frombuffer(lsec, dt).reshape(n, 8).astype(np.float64)
    final = apply_multipliers(corrected, lq[:, :4], grid, lq[:, 4:])
    cnt = struct.unpack_from("<I", esec, 0)[0]
    off = 4
    for _ in range(cnt):
        i = struct.unpack_from("<I", esec, off)[0]
        off += 4
        final[i] = np.frombuffer(esec, "<f8", d, off).reshape(rows, cols)
        off += 8 * d
    return rec, corrected, final


def decompress(arc, threads=1):
    """pipeline.py:430-440 (shards decoded independently, on a thread pool)."""
    grid, meta, blobs = unarchive(arc)
    P, N = meta["n_planes"], meta["n_nodes"]
    r, c = grid.vol.shape
    out = np.empty((P, N, r, c))
    members = shard_members(P, N, len(blobs), meta["mode"])

    def job(k):
        pl, no = members[k]
        out[pl, no] = decode_shard(blobs[k], grid)[2]

    if threads > 1:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=threads) as ex:
            list(ex.map(job, range(len(blobs))))
    else:
        for k in range(len(blobs)):
            job(k)
    return out, grid, meta


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()
