"""Moments, error metrics and the report type (reference qoi.py).

compute_qoi / compute_qoi_batch run on the device (mlk_compare); the
pipeline computes the moments inside its stage kernels.
"""

from __future__ import annotations

from dataclasses import asdict, dataclass, field

import numpy as np

from .errors import DegenerateRangeError, DimensionError

__all__ = ["ErrorReport", "QoISet", "compute_qoi", "compute_qoi_batch", "nrmse",
           "compression_ratio", "qoi_nrmse_from_moments"]


@dataclass(frozen=True)
class QoISet:
    """Per-(plane, node) moments; ratio entries are NaN where n == 0 (qoi.py:30-40)."""

    n: np.ndarray
    u_par: np.ndarray
    t_perp: np.ndarray
    t_par: np.ndarray

    def defined_mask(self) -> np.ndarray:
        return self.n > 0


def _moments_device(images: np.ndarray, grid) -> np.ndarray:
    """(N, 4) moments of a (N, rows, cols) stack on the device (mlk_compare's
    moment pass, the compute_qoi_batch formulas of qoi.py:60-76)."""
    import torch

    from . import _ops
    from ._lib import call
    from .pipeline import _device_grid
    n = images.shape[0]
    d = grid.rows * grid.cols
    dv = _ops.dev()
    x = _ops.to_dev(images.reshape(n, d))
    f64 = dict(dtype=torch.float64, device=dv)
    err, sse, q, ext = (torch.empty(n, **f64), torch.empty(n, **f64),
                        torch.empty((n, 4), **f64), torch.empty((n, 2), **f64))
    call("mlk_compare", x, x, n, _device_grid(grid, dv, 4).addr, err, sse, q, None, ext)
    return q.cpu().numpy()


def compute_qoi(image: np.ndarray, grid):
    """Moments of one histogram: (n, u_par, t_perp, t_par), NaN ratios where
    n <= 0 (qoi.py:42-57); computed on the device."""
    image = np.asarray(image, dtype=np.float64)
    if image.shape != (grid.rows, grid.cols):
        raise DimensionError(f"image shape {image.shape} does not match grid "
                             f"({grid.rows}, {grid.cols})")
    q = _moments_device(image[None], grid)[0]
    n = float(q[0])
    if n <= 0.0:
        return n, float("nan"), float("nan"), float("nan")
    return n, float(q[1]), float(q[2]), float(q[3])


def compute_qoi_batch(images: np.ndarray, grid) -> QoISet:
    """Moments of a (N, rows, cols) stack (qoi.py:60-76), on the device."""
    images = np.asarray(images, dtype=np.float64)
    if images.shape[1:] != (grid.rows, grid.cols):
        raise DimensionError("image stack does not match the grid")
    if images.shape[0] == 0:
        z = np.zeros(0)
        return QoISet(n=z, u_par=z.copy(), t_perp=z.copy(), t_par=z.copy())
    q = _moments_device(images, grid)
    return QoISet(n=q[:, 0].copy(), u_par=q[:, 1].copy(), t_perp=q[:, 2].copy(),
                  t_par=q[:, 3].copy())


def nrmse(u, f) -> float:
    """RMS error over the reference's range (qoi.py:79-90); host-side, for reports."""
    u = np.asarray(u, dtype=np.float64).ravel()
    f = np.asarray(f, dtype=np.float64).ravel()
    if u.size != f.size or u.size == 0:
        raise DimensionError("nrmse needs two equal-length, non-empty arrays")
    span = float(np.max(u) - np.min(u))
    if span == 0.0:
        if np.array_equal(u, f):
            return 0.0
        raise DegenerateRangeError("reference range is zero but arrays differ")
    return float(np.sqrt(np.mean((u - f) ** 2)) / span)


def compression_ratio(original_bytes: int, archive_bytes: int) -> float:
    if archive_bytes <= 0:
        raise ZeroDivisionError("archive size must be positive")
    return original_bytes / archive_bytes


def qoi_nrmse_from_moments(q_orig: np.ndarray, q_rec: np.ndarray):
    """qoi.qoi_error_report (qoi.py:122-133) from (N, 4) moment tables."""
    mask = q_orig[:, 0] > 0
    names = ("n", "u_par", "t_perp", "t_par")
    qo = np.ascontiguousarray(q_orig[mask].T)  # one gather, then contiguous columns
    qr = np.ascontiguousarray(q_rec[mask].T)
    errs = {nm: nrmse(qo[k], qr[k]) for k, nm in enumerate(names)}
    return errs, max(errs.values())


@dataclass
class ErrorReport:
    pd_nrmse: float = 0.0
    per_image_nrmse: list = field(default_factory=list)
    qoi_nrmse: dict = field(default_factory=dict)
    max_qoi_nrmse: float = 0.0
    compression_ratio: float = 0.0
    ae_accuracy: float = 0.0
    residual_fraction: float = 0.0
    convergence_fraction: float = 1.0
    exception_count: int = 0
    stage_timings: dict = field(default_factory=dict)
    gates: dict = field(default_factory=dict)

    def max_per_image_nrmse(self) -> float:
        return max(self.per_image_nrmse) if len(self.per_image_nrmse) else 0.0

    def to_dict(self) -> dict:
        return asdict(self)
