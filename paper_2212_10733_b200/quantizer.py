"""Product quantisation (reference quantizer.py): the codebook container and
the per-call functions kmeans_1d / pq_train / pq_encode / pq_decode.

Training (k-means++ + Lloyd, csrc/kmeans.cu), nearest-centroid encoding and
decoding (csrc/ops.cu, csrc/capi.cu) run on the device; the pipeline uses
the batched forms inside engine.compress_device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigError

__all__ = ["PQCodebook", "ALLOWED_K", "kmeans_1d", "pq_train", "pq_encode", "pq_decode"]

ALLOWED_K = (16, 64, 256)


@dataclass(frozen=True)
class PQCodebook:
    centroids: np.ndarray  # (latent_dim, k) float32, each row sorted

    def __post_init__(self):
        c = np.asarray(self.centroids, dtype=np.float32)
        if c.ndim != 2:
            raise ConfigError("centroids must be (latent_dim, k)")
        object.__setattr__(self, "centroids", c)

    @property
    def latent_dim(self) -> int:
        return self.centroids.shape[0]

    @property
    def k(self) -> int:
        return self.centroids.shape[1]

    @property
    def bits(self) -> int:
        return int(self.k - 1).bit_length()

    def to_bytes(self) -> bytes:
        return self.centroids.astype("<f4").tobytes()

    @classmethod
    def from_bytes(cls, raw: bytes, latent_dim: int, k: int):
        return cls(centroids=np.frombuffer(raw, dtype="<f4").reshape(latent_dim, k).copy())


# ---------------------------------------------------------------------------
# the reference's per-call functions (quantizer.py:53-138) on the device

KMEANS_MAX_N = 1 << 18  # members per (shard, dim) the device k-means holds


def _kmeans_device(lat, k: int, seed: int):
    """mlk_kmeans over the columns of lat (n, L): column d is clustered as
    kmeans_1d(lat[:, d], k, seed + d) (the PCG64 draws it consumes are a pure
    function of (n, k, seed) and are computed on the host)."""
    import ctypes

    import torch

    from . import _ops
    from ._lib import MlkShard, call
    from .engine import kmeans_draws
    n, L = lat.shape
    if n > KMEANS_MAX_N:
        raise ConfigError(f"the device k-means holds at most {KMEANS_MAX_N} values per column")
    table = (MlkShard * 1)()
    table[0] = MlkShard(base=0, plane_stride=0, block=max(n, 1), n_img=n, img_off=0,
                        small_blas=0, mean=0.0, std=1.0, eb=0.0, lossless=0, w_off=0, j0=0,
                        pad=0)
    first, draws = [], []
    for d in range(L):
        f, u = kmeans_draws(n, k, seed + d)
        first.append(f)
        draws.extend(u)
    d_ = _ops.dev()
    sh_d = torch.from_numpy(np.frombuffer(bytes(table), np.uint8).copy()).to(d_)
    cents = torch.empty((1, L, k), dtype=torch.float32, device=d_)
    c64 = torch.empty((1, L, k), dtype=torch.float64, device=d_)
    info = torch.empty((1, L, 4), dtype=torch.int32, device=d_)
    scratch = torch.empty(4 * L * n, dtype=torch.float64, device=d_)
    call("mlk_kmeans", _ops.to_dev(lat), sh_d, ctypes.addressof(table), 1, L, k,
         _ops.to_dev(np.asarray(first, np.int64), torch.int64),
         _ops.to_dev(np.asarray(draws if draws else [0.0], np.float64)), scratch, cents, c64, info)
    return cents[0], c64[0]


def kmeans_1d(values, k: int, seed: int) -> np.ndarray:
    """1D k-means with k-means++ seeding; returns the sorted float64
    centroids (quantizer.py:53-88), computed by csrc/kmeans.cu."""
    values = np.asarray(values, dtype=np.float64).ravel()
    if values.size == 0:
        raise ConfigError("cannot cluster an empty value list")
    if k < 1:
        raise ConfigError("k must be >= 1")
    return _kmeans_device(values.reshape(-1, 1), k, seed)[1][0].cpu().numpy()


def pq_train(latents, k: int, seed: int) -> PQCodebook:
    """Independent 1D codebook per latent dimension (quantizer.py:99-108)."""
    latents = np.asarray(latents, dtype=np.float64)
    if latents.ndim != 2 or latents.shape[0] == 0:
        raise ConfigError("latents must be a non-empty (N, latent_dim) array")
    if k not in ALLOWED_K:
        raise ConfigError(f"k must be one of {ALLOWED_K}, got {k}")
    return PQCodebook(centroids=_kmeans_device(latents, k, seed)[0].cpu().numpy())


def pq_encode(codebook: PQCodebook, latents) -> bytes:
    """Nearest-centroid indices packed little-endian (quantizer.py:111-120)."""
    import torch

    from . import _ops
    from ._lib import call
    from .errors import DimensionError
    latents = np.asarray(latents, dtype=np.float64)
    if latents.ndim != 2 or latents.shape[1] != codebook.latent_dim:
        raise DimensionError("latent dimension does not match the codebook")
    n, L = latents.shape
    if n == 0:
        return b""
    d = _ops.dev()
    idx = torch.empty(n * L, dtype=torch.int16, device=d)
    call("mlk_pq_nearest", _ops.to_dev(latents), n, L,
         _ops.to_dev(codebook.centroids, torch.float32), codebook.k, idx)
    bits = codebook.bits
    out = torch.empty((n * L * bits + 7) // 8, dtype=torch.uint8, device=d)
    bad = torch.zeros(1, dtype=torch.int32, device=d)
    call("mlk_pack_indices", idx, n * L, bits, out, bad)
    return out.cpu().numpy().tobytes()


def pq_decode(codebook: PQCodebook, packed: bytes, n_latents: int) -> np.ndarray:
    """Exact centroid lookup for packed codes (quantizer.py:123-138)."""
    import torch

    from . import _ops
    from ._lib import call
    from .errors import SizeMismatchError
    L = codebook.latent_dim
    total = n_latents * L
    expected = (total * codebook.bits + 7) // 8
    if len(packed) != expected:
        raise SizeMismatchError(f"code stream is {len(packed)} bytes, expected {expected}")
    if total == 0:
        return np.empty((n_latents, L), dtype=np.float64)
    d = _ops.dev()
    idx = torch.empty(total, dtype=torch.int16, device=d)
    call("mlk_unpack_indices", _ops.to_dev(np.frombuffer(bytes(packed), np.uint8), torch.uint8),
         total, codebook.bits, idx)
    out = torch.empty(total, dtype=torch.float64, device=d)
    bad = torch.zeros(1, dtype=torch.int32, device=d)
    call("mlk_pq_lookup", idx, n_latents, L, _ops.to_dev(codebook.centroids, torch.float32),
         codebook.k, out, bad)
    if int(bad.item()):
        raise SizeMismatchError("code index out of codebook range")
    return out.cpu().numpy().reshape(n_latents, L)
