"""Device plumbing shared by the per-call public operators (quantizer,
residual, lagrange, qoi, autoencoder): host arrays in, one stream of C-ABI
launches (include/mlk_b200.h), host arrays out.  No host fallback."""

from __future__ import annotations

import ctypes
import functools

import numpy as np
import torch

from ._lib import MlkGrid, call, lib


def dev() -> torch.device:
    lib()  # BackendError without the library / a CUDA device
    return torch.device("cuda", torch.cuda.current_device())


def to_dev(a, dtype=torch.float64) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev(), dtype=dtype)


@functools.lru_cache(maxsize=64)
def _pw_grid_cached(d: int):
    return MlkGrid(rows=1, cols=d, D=d, pad=0, mass=1.0, sep=0)


def flat_grid(d: int) -> int:
    """Address of an MlkGrid describing only D (what the NRMSE-only calls of
    mlk_compare read; no moments are requested through it)."""
    return ctypes.addressof(_pw_grid_cached(int(d)))


def image_nrmse(orig: torch.Tensor, other: torch.Tensor, n: int, d: int):
    """qoi.image_nrmse_batch (qoi.py:107-119) on the device, exact numpy
    pairwise order (mlk_compare); returns (err, ext) device tensors."""
    f64 = dict(dtype=torch.float64, device=orig.device)
    err = torch.empty(n, **f64)
    sse = torch.empty(n, **f64)
    ext = torch.empty((n, 2), **f64)
    call("mlk_compare", orig, other, n, flat_grid(d), err, sse, None, None, ext)
    return err, ext


class PlainGrid:
    """Device tables of a D-cell image with no velocity grid (rows 1 x D,
    not separable): what mlk_stage1 needs to encode flat images (its
    moments output is then meaningless and ignored)."""

    def __init__(self, d: int, latent_dim: int):
        from .engine import decode_tree_cols
        dv = dev()
        self.t = dict(one=torch.ones(d, dtype=torch.float64, device=dv),
                      zero=torch.zeros(3 * d, dtype=torch.float64, device=dv),
                      tree=torch.from_numpy(np.frombuffer(decode_tree_cols(d, latent_dim),
                                                          np.uint8).copy()).to(dv))
        z = self.t["zero"].data_ptr()
        self.struct = MlkGrid(rows=1, cols=d, D=d, pad=0, mass=1.0,
                              vol=self.t["one"].data_ptr(), vpar=z, vperp2=z, hmvol=z, ash=z,
                              tree_cols=self.t["tree"].data_ptr(), s0=1.0, s1=1.0, s2=1.0,
                              sep=0, pad2=0)

    @property
    def addr(self) -> int:
        return ctypes.addressof(self.struct)


def ae_encode(flat: np.ndarray, model):
    """autoencoder.encode_batch (autoencoder.py:99-103) in the OpenBLAS order
    (mlk_stage1 over one contiguous shard); returns (latents device tensor,
    the device copy of the images, the plain grid)."""
    from ._lib import MlkShard
    n, d = flat.shape
    L = model.latent_dim
    dv = dev()
    imgs = torch.zeros(n * d + 2, dtype=torch.float64, device=dv)  # + TMA tail pad
    imgs[:n * d].copy_(torch.from_numpy(np.ascontiguousarray(flat, dtype=np.float64))
                       .reshape(-1))
    table = (MlkShard * 1)()
    table[0] = MlkShard(base=0, plane_stride=n * d, block=n, n_img=n, img_off=0,
                        small_blas=int(n * L * d <= 1e6), mean=float(model.norm_mean),
                        std=float(model.norm_std), eb=0.0, lossless=0, w_off=0, j0=0, pad=0)
    sh_d = torch.from_numpy(np.frombuffer(bytes(table), np.uint8).copy()).to(dv)
    W = to_dev(model.weights, torch.float32)
    grid = PlainGrid(d, L)
    f64 = dict(dtype=torch.float64, device=dv)
    lat = torch.empty((n, L), **f64)
    stats = torch.empty((n, 4), **f64)
    qoi = torch.empty((n, 4), **f64)
    call("mlk_stage1", imgs, sh_d, 1, n, grid.addr, W, L, lat, stats, qoi)
    return lat, imgs, W, grid
