"""Tied-weight linear autoencoder (reference autoencoder.py:26-177).

The per-histogram path consumes trained weights: the contraction runs on
device in ``csrc/stage1.cu`` (encode) and every kernel that needs a
reconstruction (decode).  Training also runs on the
device: :func:`train` / :func:`train_jobs` drive ``csrc/train.cu``
(``mlk_ae_train``, one CTA per job for every epoch); the host only draws the
reference's PCG64 stream (Glorot init, per-epoch permutations) and the Adam
bias-correction table.
"""

from __future__ import annotations

import functools
import struct
from dataclasses import dataclass

import numpy as np

from .errors import ConfigError, DimensionError, TrainingDivergedError

__all__ = ["AEModel", "TrainConfig", "train", "train_jobs", "STD_FLOOR"]

STD_FLOOR = 1e-30


@dataclass(frozen=True)
class AEModel:
    weights: np.ndarray   # (latent_dim, D) float32
    norm_mean: float
    norm_std: float

    def __post_init__(self):
        w = np.asarray(self.weights, dtype=np.float32)
        if w.ndim != 2:
            raise ConfigError("weights must be a (latent_dim, D) matrix")
        if not self.norm_std > 0:
            raise ConfigError("normalizer std must be positive")
        object.__setattr__(self, "weights", w)

    @property
    def latent_dim(self) -> int:
        return self.weights.shape[0]

    @property
    def input_dim(self) -> int:
        return self.weights.shape[1]

    def to_bytes(self) -> bytes:
        """Weights section payload: ``<dd`` normaliser + f32 weights (autoencoder.py:44-46)."""
        return struct.pack("<dd", self.norm_mean, self.norm_std) + \
            self.weights.astype("<f4").tobytes()

    @classmethod
    def from_bytes(cls, raw: bytes, latent_dim: int, input_dim: int):
        mean, std = struct.unpack_from("<dd", raw, 0)
        w = np.frombuffer(raw, dtype="<f4", offset=16, count=latent_dim * input_dim)
        return cls(weights=w.reshape(latent_dim, input_dim).copy(), norm_mean=mean,
                   norm_std=std)


@dataclass(frozen=True)
class TrainConfig:
    """Adam settings (autoencoder.py:60-75)."""

    learning_rate: float = 0.001
    batch_size: int = 128
    epochs: int = 100
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    seed: int = 0

    def __post_init__(self):
        if self.learning_rate <= 0:
            raise ConfigError("learning rate must be positive")
        if self.batch_size < 1 or self.epochs < 1:
            raise ConfigError("batch size and epochs must be >= 1")


@dataclass
class TrainJob:
    """One independent training run: images base[row_off[i] : row_off[i] + D]."""

    base: object            # device float64 tensor (flat)
    row_off: np.ndarray     # (n,) int64 element offsets into base
    epochs: int
    seed: int
    init: AEModel | None = None


def _host_draws(n, d, latent_dim, epochs, seed, init):
    """Glorot init + per-epoch permutations from PCG64(seed) (autoencoder.py:150-163)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    if init is not None:
        w = init.weights.astype(np.float64)
    else:
        bound = np.sqrt(6.0 / (latent_dim + d))
        w = rng.uniform(-bound, bound, size=(latent_dim, d))
    order = np.empty((epochs, n), dtype=np.int32)
    for e in range(epochs):
        order[e] = rng.permutation(n)
    return np.ascontiguousarray(w, dtype=np.float64), order


PW_BLOCK = 128  # numpy PW_BLOCKSIZE


@functools.lru_cache(maxsize=32)
def pairwise_tree(n: int):
    """numpy's pairwise_sum recursion over n entries as a tree (the layout
    MlkPwTree describes): leaves (start, len) in entry order, each <= 128
    entries; internal nodes grouped by depth, deepest first, with the ids of
    their two children (leaf l has id l, internal node k has id n_leaves + k).
    Split rule: n2 = n // 2 rounded down to a multiple of 8 (loops_utils.h.src)."""
    levels = []                         # per depth: (lo, n) of every node
    lo, ln = np.array([0], np.int64), np.array([n], np.int64)
    while lo.size:
        levels.append((lo, ln))
        inner = ln > PW_BLOCK
        h = ln[inner] // 2
        n2 = h - h % 8
        lo = np.stack([lo[inner], lo[inner] + n2], 1).reshape(-1)
        ln = np.stack([n2, ln[inner] - n2], 1).reshape(-1)
    leaf_lo = np.concatenate([l[n_ <= PW_BLOCK] for l, n_ in levels])
    leaf_ln = np.concatenate([n_[n_ <= PW_BLOCK] for _, n_ in levels])
    order = np.argsort(leaf_lo, kind="stable")
    leaf_lo, leaf_ln = leaf_lo[order], leaf_ln[order]
    n_leaves = leaf_lo.size
    ids = [None] * len(levels)
    child, level_off, nxt = [], [0], n_leaves
    for dpt in range(len(levels) - 1, -1, -1):
        l, n_ = levels[dpt]
        idv = np.empty(l.size, np.int64)
        leaf = n_ <= PW_BLOCK
        idv[leaf] = np.searchsorted(leaf_lo, l[leaf])
        k = int((~leaf).sum())
        if k:
            idv[~leaf] = nxt + np.arange(k)
            nxt += k
            child.append(ids[dpt + 1].reshape(-1, 2))
            level_off.append(level_off[-1] + k)
        ids[dpt] = idv
    child = np.concatenate(child).reshape(-1) if child else np.zeros(0, np.int64)
    return (leaf_lo.astype(np.int64), leaf_ln.astype(np.int32), child.astype(np.int32),
            np.array(level_off, np.int32))


def train_jobs(jobs, config: TrainConfig, latent_dim: int, d: int):
    """Train every job in one launch; returns one AEModel per job.

    ``config.epochs`` and ``config.seed`` are taken per job from TrainJob."""
    import torch

    from . import _lib

    if not jobs:
        return []
    L = jobs[0].init.latent_dim if jobs[0].init is not None else latent_dim
    for jb in jobs:
        if jb.init is not None and (jb.init.input_dim != d or jb.init.latent_dim != L):
            raise DimensionError("warm-start model does not match image size")
        if len(jb.row_off) == 0:
            raise ConfigError("need at least one training image")
    dev = jobs[0].base.device
    B = config.batch_size
    T = max(jb.epochs * -(-len(jb.row_off) // B) for jb in jobs)
    # Python-float bias corrections, exactly as autoencoder.py:171-172 evaluates them
    bias = np.array([[1 - config.beta1 ** t, 1 - config.beta2 ** t] for t in range(1, T + 1)],
                    dtype=np.float64)
    ws, keep, recs, trees = [], [], [], []
    for jb in jobs:
        n = len(jb.row_off)
        w, order = _host_draws(n, d, L, jb.epochs, jb.seed, jb.init)
        wd = torch.from_numpy(w).to(dev)
        offs = torch.from_numpy(np.ascontiguousarray(jb.row_off, dtype=np.int64)).to(dev)
        od = torch.from_numpy(order).to(dev)
        xn = torch.empty(n * d, dtype=torch.float64, device=dev)
        # fit_normalizer's pairwise tree over the n*d entries
        t_lo, t_ln, t_ch, t_lv = (torch.from_numpy(a).to(dev) for a in pairwise_tree(n * d))
        nodes = torch.empty(t_lo.numel() + int(t_lv[-1].item() if t_lv.numel() else 0),
                            dtype=torch.float64, device=dev)
        keep += [offs, od, xn, jb.base, t_lo, t_ln, t_ch, t_lv, nodes]
        ws.append(wd)
        recs.append((jb.base.data_ptr(), offs.data_ptr(), od.data_ptr(), wd.data_ptr(),
                     0, xn.data_ptr(), n, jb.epochs))
        trees.append((t_lo.data_ptr(), t_ln.data_ptr(), t_ch.data_ptr(), t_lv.data_ptr(),
                      nodes.data_ptr(), n * d, t_lo.numel(), t_lv.numel() - 1))
    rec_t = np.dtype([("base", "<u8"), ("row_off", "<u8"), ("order", "<u8"), ("w", "<u8"),
                      ("mv", "<u8"), ("xn", "<u8"), ("n", "<i4"), ("epochs", "<i4")])
    tree_t = np.dtype([("leaf_start", "<u8"), ("leaf_len", "<u8"), ("child", "<u8"),
                       ("level_off", "<u8"), ("nodes", "<u8"), ("n_total", "<i8"),
                       ("n_leaves", "<i4"), ("n_levels", "<i4")])
    table_h = np.array(recs, dtype=rec_t)
    table_d = torch.from_numpy(table_h.view(np.uint8).copy()).to(dev)
    trees_h = np.array(trees, dtype=tree_t)
    trees_d = torch.from_numpy(trees_h.view(np.uint8).copy()).to(dev)
    bias_d = torch.from_numpy(bias.reshape(-1)).to(dev)
    norm = torch.empty(2 * len(jobs), dtype=torch.float64, device=dev)
    diag = torch.empty(2 * len(jobs), dtype=torch.float64, device=dev)
    _lib.call("mlk_ae_train", table_d, table_h.ctypes.data, trees_d, trees_h.ctypes.data,
              len(jobs), L, d, B,
              float(config.learning_rate), float(config.beta1), float(1 - config.beta1),
              float(config.beta2), float(1 - config.beta2), float(config.eps), bias_d, T,
              norm, diag, msg="(AE training)")
    norm_h, diag_h = norm.cpu().numpy(), diag.cpu().numpy()
    out = []
    for j, wd in enumerate(ws):
        if diag_h[2 * j] >= 0:
            raise TrainingDivergedError(int(diag_h[2 * j]), float(diag_h[2 * j + 1]))
        out.append(AEModel(weights=wd.cpu().numpy().astype(np.float32),
                           norm_mean=float(norm_h[2 * j]), norm_std=float(norm_h[2 * j + 1])))
    del keep
    return out


def train(images, config: TrainConfig, init: AEModel | None = None,
          latent_dim: int = 4) -> AEModel:
    """Adam-train a model on the device (autoencoder.py:137-177).

    ``images``: (N, rows, cols) / (N, D) host array or CUDA tensor.  Fresh
    Glorot init unless warm-started via ``init``; the normaliser is always
    refit on the supplied images."""
    import torch

    from .pipeline import _device

    if isinstance(images, torch.Tensor):
        if images.ndim < 2 or images.shape[0] == 0:
            raise ConfigError("need at least one training image")
        x = images.to(dtype=torch.float64).reshape(images.shape[0], -1).contiguous()
        if not x.is_cuda:
            x = x.to(_device())
    else:
        arr = np.asarray(images, dtype=np.float64)
        if arr.ndim < 2 or len(arr) == 0:
            raise ConfigError("need at least one training image")
        x = torch.from_numpy(np.ascontiguousarray(arr.reshape(len(arr), -1))).to(_device())
    n, d = x.shape
    if init is not None and init.input_dim != d:
        raise DimensionError("warm-start model does not match image size")
    job = TrainJob(base=x.reshape(-1), row_off=np.arange(n, dtype=np.int64) * d,
                   epochs=config.epochs, seed=config.seed, init=init)
    return train_jobs([job], config, latent_dim, d)[0]


def ae_accuracy(images, model: AEModel, tau: float) -> float:
    """Fraction of images whose AE-only reconstruction meets the bound
    (autoencoder.py:180-188): encode (OpenBLAS order, mlk_stage1), decode
    (mlk_ae_decode) and the exact per-image NRMSE (mlk_compare) on the
    device."""
    import torch

    from . import _ops
    from ._lib import call
    if tau <= 0:
        raise ConfigError("tau must be positive")
    images = np.asarray(images, dtype=np.float64)
    n = images.shape[0]
    flat = images.reshape(n, -1)
    d = flat.shape[1]
    if d != model.input_dim:
        raise DimensionError(f"images have {d} entries, model expects {model.input_dim}")
    if n == 0:
        return float(np.mean(np.zeros(0) <= tau))
    lat, imgs, W, grid = _ops.ae_encode(flat, model)
    recon = torch.empty(n * d, dtype=torch.float64, device=lat.device)
    # OpenBLAS's small-matrix kernel sums every column sequentially
    tree = grid.t["tree"] if n * model.latent_dim * d > 1e6 else None
    call("mlk_ae_decode", lat, n, model.latent_dim, W, d, float(model.norm_mean),
         float(model.norm_std), tree, recon)
    err, _ = _ops.image_nrmse(imgs, recon, n, d)
    return float(np.mean(err.cpu().numpy() <= tau))
