"""The policy-evaluation API (mirror of rmpnav/policies.py) over the B200.

Drop-in entry points (same signatures, argument meaning, return type and
error behaviour as the reference):

* ``ray_policy(state, field, bundle, p, max_range=20, t=0, workers=1,
  backend=None)`` (policies.py:182-192) -- on an ``EsdfGrid`` this is ONE
  fused launch (sphere trace + per-ray policy + fixed-order reduction + 3x3
  pinv) returning 16 doubles; on an analytic ``Scene`` it traces the scene
  on device, then reduces on device.
* ``lidar_policy(velocity, scan, p, min_range=0.3, workers=1, backend=None)``
  (policies.py:195-205) -- one launch; the sensor-to-world rotation of the
  beam lattice happens in the kernel.

Beyond the reference: ``ray_policy_batch`` (many poses per launch, config
C4), ``lidar_policy_points`` (raw sensor-frame points, no lattice) and
``lidar_policy_batch`` (many scans per launch).

Every policy evaluation returns ``Policy(pinv(sum A) @ sum A f, sum A)`` with
misses / invalid beams contributing nothing and zero hits giving the zero
policy.
"""

from __future__ import annotations

import json
from dataclasses import asdict, dataclass

import math

import numpy as np

from ._kernels import get_backend
from .core import Policy, RobotState
from .geometry import EsdfGrid
from .rays import (DEFAULT_MAX_RANGE, GRID_STEP_SCALE, RangeScan, RayBundle, policy_range,
                   raycast_many)

__all__ = ["AttractorParams", "ObstacleParams", "PolicyParams", "PRESETS", "preset", "esdf_policy",
           "ray_policy", "ray_policy_batch", "lidar_policy", "lidar_policy_points",
           "lidar_policy_batch", "obstacle_ray_policy", "activation_weight", "save_params",
           "load_params", "DEFAULT_LIDAR_MIN_RANGE"]

DEFAULT_LIDAR_MIN_RANGE = 0.3  # policies.py:39


@dataclass(frozen=True)
class AttractorParams:
    alpha: float
    beta: float
    c: float

    def __post_init__(self):
        if min(self.alpha, self.beta, self.c) <= 0:
            raise ValueError("attractor parameters must be positive")


@dataclass(frozen=True)
class ObstacleParams:
    """Obstacle policy tuning (Table I).  ``as_tuple`` is the kernel order."""

    eta_rep: float
    nu_rep: float
    eta_damp: float
    nu_damp: float
    radius: float
    c: float
    epsilon: float = 1e-6

    def __post_init__(self):
        if min(self.eta_rep, self.nu_rep, self.eta_damp, self.nu_damp, self.radius, self.c,
               self.epsilon) <= 0:
            raise ValueError("obstacle parameters must be positive")

    def as_tuple(self) -> tuple:
        return (self.eta_rep, self.nu_rep, self.eta_damp, self.nu_damp, self.epsilon,
                self.radius, self.c)


@dataclass(frozen=True)
class PolicyParams:
    attractor: AttractorParams
    obstacle: ObstacleParams


# Table I of the paper (policies.py:92-103).
PRESETS: dict[str, PolicyParams] = {
    "static_map": PolicyParams(AttractorParams(10.0, 15.0, 0.2),
                               ObstacleParams(88.0, 1.4, 140.0, 1.2, 2.4, 0.2)),
    "lidar": PolicyParams(AttractorParams(0.8, 1.6, 1.0),
                          ObstacleParams(1.2, 1.5, 3.0, 1.0, 1.3, 1.0)),
}


def preset(name: str) -> PolicyParams:
    if name not in PRESETS:
        raise ValueError(f"unknown preset {name!r}; available: {sorted(PRESETS)}")
    return PRESETS[name]


def save_params(params: PolicyParams, path) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        json.dump({"attractor": asdict(params.attractor), "obstacle": asdict(params.obstacle)},
                  fh, indent=2, sort_keys=True)
        fh.write("\n")


def load_params(path) -> PolicyParams:
    with open(path, "r", encoding="utf-8") as fh:
        doc = json.load(fh)
    return PolicyParams(AttractorParams(**doc["attractor"]), ObstacleParams(**doc["obstacle"]))


def activation_weight(d: float, radius: float) -> float:
    """w_r(d) = d^2/r^2 - 2d/r + 1 below the radius, 0 at and beyond it."""
    if d >= radius:
        return 0.0
    return d * d / (radius * radius) - 2.0 * d / radius + 1.0


def obstacle_ray_policy(velocity, away_dir, distance: float, p: ObstacleParams) -> Policy:
    """Single surface-point policy, Eqs. 5-9 (policies.py:143-163).  A scalar
    helper (one 3-vector), not part of the data-parallel path."""
    v = np.asarray(velocity, dtype=float).reshape(3)
    r = np.asarray(away_dir, dtype=float).reshape(3)
    d = float(distance)
    f_rep = p.eta_rep * np.exp(-d / p.nu_rep) * r
    closing = max(0.0, -float(v @ r))
    f_damp = p.eta_damp / (d / p.nu_damp + p.epsilon) * (closing * closing * r)
    n = float(np.linalg.norm(f_damp))
    s = f_damp / (n + p.c * np.log1p(np.exp(-2.0 * p.c * n)))
    return Policy(f_rep + f_damp, activation_weight(d, p.radius) * np.outer(s, s))


def esdf_policy(state: RobotState, grid: EsdfGrid, p: ObstacleParams) -> Policy:
    """Single-lookup obstacle policy (policies.py:166-172, row f4): one
    distance / gradient query on the device, one obstacle policy; a
    degenerate (zero) gradient gives the zero policy."""
    from .geometry import esdf_lookup

    sample = esdf_lookup(grid, state.position)
    if sample.degenerate:
        return Policy.zero()
    return obstacle_ray_policy(state.velocity, sample.gradient, sample.distance, p)


_SYM_SAFE = 8.98e307  # 0.5 * (m + m.T) overflows above DBL_MAX / 2
_F64 = np.dtype(np.float64)


def _policy_from_slot(slot, accel) -> Policy:
    """Policy from a device slot.  The device writes the metric exactly
    symmetric (a01 duplicated), so Policy's symmetrisation 0.5 * (m + m.T)
    returns it unchanged whenever it cannot overflow: such slots take a
    check-only path (~2 us instead of ~15 us of small NumPy ops); anything
    else goes through Policy's own construction (and its ValueError)."""
    if type(slot) is np.ndarray and type(accel) is np.ndarray and slot.dtype is _F64 \
            and accel.dtype is _F64 and slot.ndim == 1 and accel.shape == (3,):
        lm = slot.tolist()
        m9 = lm[:9]
        tot = sum(m9) + sum(accel.tolist())  # NaN / inf (or an overflowing sum) -> not finite
        if (len(lm) >= 9 and tot - tot == 0.0 and lm[1] == lm[3] and lm[2] == lm[6]
                and lm[5] == lm[7] and max(m9) < _SYM_SAFE and min(m9) > -_SYM_SAFE):
            return Policy._trusted(accel, slot[0:9].reshape(3, 3))
    return Policy(np.asarray(accel, dtype=float), np.asarray(slot[0:9], dtype=float).reshape(3, 3))


def _reduced_policy(be, dirs, dists, velocity, p: ObstacleParams, min_range: float,
                    workers: int) -> Policy:
    """Generic two-call path (policies.py:175-179) for non-grid fields."""
    metric, weighted, _n = be.policy_reduce(dirs, dists, velocity, p.as_tuple(), min_range,
                                            workers)
    return Policy(be.pinv_psd(metric) @ weighted, metric)


def ray_policy(state: RobotState, field, bundle: RayBundle, p: ObstacleParams,
               max_range: float = DEFAULT_MAX_RANGE, t: float = 0.0, workers: int = 1,
               backend: str | None = None, policy_only: bool = False) -> Policy:
    """Cast the bundle from the robot; one obstacle policy per hit ray with
    away direction = -cast direction; metric-weighted combination.

    ``policy_only=True`` (beyond the reference) stops each ray at the
    activation radius ``p.radius`` (``policy_range``): the returned Policy
    sums exactly the same hits, for less marching (C1: 12.2 -> 7.9 ms per
    4096 poses, single pose ~30 -> ~18 us of kernel)."""
    be = get_backend(backend)
    if policy_only:
        max_range = policy_range(max_range, p.radius)
    if isinstance(field, EsdfGrid) and hasattr(be, "ray_policy_fused"):
        slot, accel = be.ray_policy_fused(field.values, field.origin, field.resolution,
                                          state.position, state.velocity, bundle.directions,
                                          p.as_tuple(), max_range, 0.5 * field.resolution,
                                          GRID_STEP_SCALE)
        return _policy_from_slot(slot, accel)
    dists = raycast_many(field, state.position, bundle.directions, max_range, t,
                         workers=workers, backend=backend)
    return _reduced_policy(be, bundle.directions, dists, state.velocity, p, 0.0, workers)


def ray_policy_batch(states, field: EsdfGrid, bundle: RayBundle, p: ObstacleParams,
                     max_range: float = DEFAULT_MAX_RANGE, backend: str | None = None,
                     policy_only: bool = False):
    """``ray_policy`` for many robot states in one launch.  ``states`` is a
    sequence of RobotState or a (positions P x 3, velocities P x 3) pair.
    Returns (accels P x 3, metrics P x 3 x 3, n_hits P); with
    ``policy_only`` (see ``ray_policy``) n_hits counts hits within the
    activation radius only."""
    if policy_only:
        max_range = policy_range(max_range, p.radius)
    if not isinstance(field, EsdfGrid):
        raise TypeError("ray_policy_batch needs an EsdfGrid")
    if isinstance(states, tuple) and len(states) == 2 and not isinstance(states[0], RobotState):
        x, v = states
    else:
        x = np.array([s.position for s in states], dtype=np.float64).reshape(-1, 3)
        v = np.array([s.velocity for s in states], dtype=np.float64).reshape(-1, 3)
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, 3)
    v = np.ascontiguousarray(v, dtype=np.float64).reshape(-1, 3)
    if not (np.isfinite(x).all() and np.isfinite(v).all()):
        raise ValueError("robot state must be finite")
    be = get_backend(backend)
    slots, accels = be.ray_policy_batch(field.values, field.origin, field.resolution, x, v,
                                        bundle.directions, p.as_tuple(), max_range,
                                        0.5 * field.resolution, GRID_STEP_SCALE)
    metrics = slots[:, 0:9].reshape(-1, 3, 3)
    if not (np.isfinite(accels).all() and np.isfinite(metrics).all()):
        raise ValueError("policy acceleration / metric must be finite")
    return accels, metrics, slots[:, 12].astype(np.int64)


def lidar_policy(velocity, scan: RangeScan, p: ObstacleParams,
                 min_range: float = DEFAULT_LIDAR_MIN_RANGE, workers: int = 1,
                 backend: str | None = None) -> Policy:
    """Reduction over a scan's valid beams taken verbatim (world frame)."""
    be = get_backend(backend)
    v = np.asarray(velocity, dtype=float)
    if hasattr(be, "lidar_policy_fused"):
        slot, accel = be.lidar_policy_fused(scan.directions, scan.orientation, scan.ranges,
                                            scan.valid, v, p.as_tuple(), min_range)
        return _policy_from_slot(slot, accel)
    dirs = np.ascontiguousarray(scan.world_directions())
    dists = np.where(scan.valid, scan.ranges, np.inf)
    return _reduced_policy(be, dirs, dists, v, p, min_range, workers)


def lidar_policy_points(velocity, points, p: ObstacleParams, orientation=None,
                        min_range: float = DEFAULT_LIDAR_MIN_RANGE,
                        backend: str | None = None) -> Policy:
    """LiDAR-direct policy from raw sensor-frame points (N x 3): beam
    direction p * (1/|p|) (within 1 ulp of p/|p|), range |p|; zero / non-finite points
    are invalid."""
    be = get_backend(backend)
    slot, accel = be.lidar_points_fused(points, orientation, np.asarray(velocity, dtype=float),
                                        p.as_tuple(), min_range)
    return _policy_from_slot(slot, accel)


def lidar_policy_batch(velocities, scans, p: ObstacleParams,
                       min_range: float = DEFAULT_LIDAR_MIN_RANGE):
    """Many scans sharing one beam lattice, one launch (device-resident).
    Returns (accels S x 3, metrics S x 3 x 3, n_hits S)."""
    from . import device as D

    return D.lidar_policy_batch_host(velocities, scans, p, min_range)
