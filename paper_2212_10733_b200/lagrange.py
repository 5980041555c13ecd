"""Newton options and statuses for the QoI projection (reference lagrange.py:33-56).

The projection itself is ``csrc/project.cu`` (batched per image, one CTA
each); these are the configuration objects the public API carries.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import ConfigError

__all__ = ["NewtonOptions", "NewtonStatus", "POSITIVITY_FLOOR"]

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
