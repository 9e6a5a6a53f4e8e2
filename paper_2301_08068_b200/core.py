"""Policy algebra types on the hot path (mirror of rmpnav/core.py).

``Policy`` (core.py:36-67) and ``RobotState`` (core.py:70-83) keep the
reference's construction rules: the metric is symmetrised, non-finite
values raise ValueError.  ``pinv_psd`` (core.py:103-115: eigen-decompose,
drop eigenvalues <= 1e-8 * max(lambda_max, 0), invert the rest) runs on the
B200 (3x3 Jacobi in fp64, librmpb ``rmpb_pinv_psd``).  ``combine`` and
``soft_normalize`` serve the rollout loop, which is outside the hot path
(SURVEY.md §2), and are not provided.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["Policy", "RobotState", "pinv_psd", "PINV_RCOND"]

PINV_RCOND = 1e-8  # core.py:26 -- fixed in the device solver

_PSD_TOL = 1e-9


def _vec3(v) -> np.ndarray:
    return np.asarray(v, dtype=float).reshape(3)


@dataclass(frozen=True)
class Policy:
    """(acceleration, metric) pair; the metric is stored symmetrised."""

    accel: np.ndarray
    metric: np.ndarray

    def __post_init__(self):
        f = _vec3(self.accel)
        m = np.asarray(self.metric, dtype=float).reshape(3, 3)
        m = 0.5 * (m + m.T)
        if not np.isfinite(f).all():
            raise ValueError("policy acceleration must be finite")
        if not np.isfinite(m).all():
            raise ValueError("policy metric must be finite")
        object.__setattr__(self, "accel", f)
        object.__setattr__(self, "metric", m)

    @classmethod
    def _trusted(cls, accel: np.ndarray, metric: np.ndarray) -> "Policy":
        """Construct without re-checking: the caller guarantees a finite
        (3,) accel and a finite, exactly symmetric (3, 3) metric (what
        __post_init__ would produce unchanged)."""
        p = object.__new__(cls)
        d = p.__dict__  # (frozen dataclass: bypass __setattr__)
        d["accel"] = accel
        d["metric"] = metric
        return p

    def is_psd(self, tol: float = _PSD_TOL) -> bool:
        return bool(np.linalg.eigvalsh(self.metric).min() >= -tol)

    @staticmethod
    def zero() -> "Policy":
        return Policy(np.zeros(3), np.zeros((3, 3)))

    @staticmethod
    def identity_metric(accel) -> "Policy":
        return Policy(accel, np.eye(3))


@dataclass(frozen=True)
class RobotState:
    """Point-robot position and velocity (finite)."""

    position: np.ndarray
    velocity: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def __post_init__(self):
        x, v = _vec3(self.position), _vec3(self.velocity)
        if not (np.isfinite(x).all() and np.isfinite(v).all()):
            raise ValueError("robot state must be finite")
        object.__setattr__(self, "position", x)
        object.__setattr__(self, "velocity", v)


def pinv_psd(a, rcond: float = PINV_RCOND) -> np.ndarray:
    """PSD pseudo-inverse of a symmetric 3x3 (or a stack of them), on device."""
    from ._kernels import get_backend

    return get_backend().pinv_psd(np.asarray(a, dtype=float), float(rcond))
