"""Moment-preserving projection: options, statuses and the reference's
per-call API (lagrange.py:33-253).

The compress pipeline runs the projection batched in ``csrc/project.cu``
(one warp per histogram).  The per-image functions here --
``newton_project`` and ``apply_lambda`` -- run the same dual Newton
(kernels.newton_solve -> mlk_newton_solve_batch) and the same elementwise
correction (mlk_apply_lambda_rows) on the device; ``build_constraints`` is
the reference's definition of the scaled 4 x D system.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigError, DimensionError

__all__ = ["NewtonOptions", "NewtonStatus", "POSITIVITY_FLOOR", "ConstraintSystem",
           "constraint_features", "build_constraints", "newton_project", "apply_lambda",
           "cast_lambda"]

POSITIVITY_FLOOR = 1e-12


class NewtonStatus:
    CONVERGED = 0
    MAX_ITER = 1
    DEGENERATE = 2


@dataclass(frozen=True)
class NewtonOptions:
    step: float = 1.0
    max_iter: int = 50
    tol: float = 1e-13
    floor: float = POSITIVITY_FLOOR
    retry: bool = False
    retry_step: float = 0.01
    retry_max_iter: int = 400

    def __post_init__(self):
        if not 0 < self.step <= 1:
            raise ConfigError("step size must be in (0, 1]")
        if self.max_iter < 1:
            raise ConfigError("max_iter must be >= 1")


@dataclass(frozen=True)
class ConstraintSystem:
    """Scaled 4 x D moment constraints for one image (lagrange.py:60-65)."""

    a: np.ndarray            # (4, D) rows scaled to unit max magnitude
    b: np.ndarray            # (4,) targets in scaled space
    row_scales: np.ndarray   # (4,) positive scale factors that were divided out


def constraint_features(grid, u_par: float) -> np.ndarray:
    """Unscaled (4, D) rows: the integrands of n, n u, n T_perp, n T_par
    (lagrange.py:68-80) -- the same expressions engine.DeviceGrid tabulates."""
    r, c = grid.rows, grid.cols
    vol = grid.vol.reshape(-1)
    v_par = np.broadcast_to(grid.v_par, (r, c)).reshape(-1)
    v_perp = np.broadcast_to(grid.v_perp[:, None], (r, c)).reshape(-1)
    hm = 0.5 * grid.mass
    return np.stack([vol, vol * v_par, hm * vol * v_perp ** 2, hm * vol * (v_par - u_par) ** 2])


def build_constraints(grid, qoi_true) -> ConstraintSystem:
    """System for the true moments (n, u_par, t_perp, t_par) (lagrange.py:83-100):
    rows and targets divided by each row's max |entry|."""
    n, u_par, t_perp, t_par = (float(q) for q in qoi_true)
    if not n > 0:
        raise ConfigError("cannot build constraints for zero density")
    a = constraint_features(grid, u_par)
    b = np.array([n, n * u_par, n * t_perp, n * t_par])
    scales = np.max(np.abs(a), axis=1)
    if np.any(scales <= 0):
        raise ConfigError("degenerate constraint row")
    return ConstraintSystem(a=a / scales[:, None], b=b / scales, row_scales=scales)


def apply_lambda(f_hat: np.ndarray, lam: np.ndarray, cs: ConstraintSystem,
                 floor: float = POSITIVITY_FLOOR) -> np.ndarray:
    """f_plus * exp(-clip(lam . a, +-700)) with f_plus = max(f_hat, floor *
    max f_hat), or a copy when max f_hat <= 0 (lagrange.py:136-149), on the
    device (mlk_apply_lambda_rows; the reference's elementwise order)."""
    import torch

    from . import _ops
    from ._lib import call
    lam = np.asarray(lam, dtype=np.float64)
    if not np.all(np.isfinite(lam)):
        raise ConfigError("lambda values must be finite")
    shape = np.shape(f_hat)
    flat = np.ascontiguousarray(f_hat, dtype=np.float64).reshape(-1)
    d = flat.size
    if cs.a.shape[1] != d:
        raise DimensionError("image size does not match the constraint system")
    f = _ops.to_dev(flat)
    out = torch.empty_like(f)
    call("mlk_apply_lambda_rows", f, 1, d, _ops.to_dev(lam.reshape(4)),
         _ops.to_dev(np.ascontiguousarray(cs.a, dtype=np.float64)), 0, float(floor), out)
    return out.cpu().numpy().reshape(shape)


def newton_project(f_hat: np.ndarray, cs: ConstraintSystem,
                   opts: NewtonOptions = NewtonOptions()):
    """Project f_hat onto the constraint manifold (lagrange.py:110-133):
    returns (lam, f_corrected, status, iterations).  The dual Newton is
    kernels.newton_solve on the device; the correction is apply_lambda."""
    from . import kernels
    flat = np.asarray(f_hat, dtype=np.float64).reshape(-1)
    if flat.size != cs.a.shape[1]:
        raise DimensionError("image size does not match the constraint system")
    top = float(np.max(flat))
    if top <= 0:
        return np.zeros(4), np.asarray(f_hat, dtype=np.float64).copy(), \
            NewtonStatus.DEGENERATE, 0
    f_plus = np.maximum(flat, opts.floor * top)
    lam, status, iters = kernels.newton_solve(f_plus, cs.a, cs.b, opts.step, opts.max_iter,
                                              opts.tol)
    if status == NewtonStatus.MAX_ITER and opts.retry:
        lam2, st2, it2 = kernels.newton_solve(f_plus, cs.a, cs.b, opts.retry_step,
                                              opts.retry_max_iter, opts.tol)
        if st2 == NewtonStatus.CONVERGED:
            lam, status, iters = lam2, st2, iters + it2
    f_corr = apply_lambda(f_hat, lam, cs, floor=opts.floor)
    return lam, f_corr.reshape(np.shape(f_hat)), status, iters


def cast_lambda(lam: np.ndarray, precision: str):
    """Storage cast of the multipliers (lagrange.py:239-253): (values, overflow)."""
    lam = np.asarray(lam, dtype=np.float64)
    if precision == "f64":
        return lam.copy(), False
    if precision != "f32":
        raise ConfigError(f"unknown lambda precision {precision!r}")
    with np.errstate(over="ignore"):
        out = lam.astype(np.float32)
    overflow = not np.all(np.isfinite(out))
    return out.astype(np.float64), overflow
