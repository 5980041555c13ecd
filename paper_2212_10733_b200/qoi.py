"""Error metrics and the report type (reference qoi.py:79-162)."""

from __future__ import annotations

from dataclasses import asdict, dataclass, field

import numpy as np

from .errors import DegenerateRangeError, DimensionError

__all__ = ["ErrorReport", "nrmse", "compression_ratio", "qoi_nrmse_from_moments"]


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
