"""Batched closed-loop rollouts on the B200.

The reference steps ONE robot per Python loop iteration
(rmpnav/sim.py:196-306: checks -> ray_policy -> combine with the attractor
-> clamp -> semi-implicit Euler) and parallelises only across rollouts with
a thread pool (sim.py:398-403).  ``rollout_batch`` advances many robots in
lockstep entirely on the GPU: per control tick one check kernel, the fused
ray-policy kernel (masked to running robots) and one update kernel, with no
host round trip.  Outcomes follow sim.Outcome; trajectories can be recorded
for the first ``record_ticks`` ticks in the reference's TrajectoryRecord
layout (state and command per tick, terminal sample with zero command).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from ._kernels import b200
from .geometry import EsdfGrid, Scene
from .policies import PolicyParams
from .rays import DEFAULT_MAX_RANGE, RayBundle, policy_range

OUTCOMES = {0: "RUNNING", 1: "SUCCESS", 2: "COLLISION", 3: "TIMEOUT", 4: "STUCK"}


@dataclass(frozen=True)
class BatchRolloutConfig:
    """The ray-planner subset of rmpnav's RolloutConfig (sim.py:102-134)."""

    params: PolicyParams
    dt: float = 0.01
    max_time: float = 60.0
    robot_radius: float = 0.3
    goal_tolerance: float = 0.3
    max_accel: float = 40.0
    stuck_window: float = 2.0
    stuck_speed: float = 0.01
    max_range: float = DEFAULT_MAX_RANGE
    hold_mode: bool = False
    # beyond the reference: rays stop at the activation radius (the same
    # obstacle policy up to the summation order; rays.policy_range)
    policy_only: bool = False

    def __post_init__(self):
        if self.dt <= 0:
            raise ValueError("dt must be positive")
        if self.robot_radius < 0:
            raise ValueError("robot_radius must be >= 0")


@dataclass
class BatchRolloutResult:
    outcome: list          # per robot: "SUCCESS" | "COLLISION" | "TIMEOUT" | "STUCK" | "RUNNING"
    steps: np.ndarray      # ticks taken
    n_clamped: np.ndarray
    positions: np.ndarray  # final
    velocities: np.ndarray
    trajectory: np.ndarray | None = None  # (P, record_ticks + 1, 9): x, v, accel


class RolloutBatch:
    """Device-resident batch of rollouts on one map / bundle / scene."""

    def __init__(self, scene: Scene, grid: EsdfGrid, bundle: RayBundle, starts, goals,
                 cfg: BatchRolloutConfig, record_ticks: int = 0):
        self.grid = b200.device_grid(grid.values, grid.origin, grid.resolution)
        self.bundle = b200.device_bundle(bundle.directions)
        self.scene = b200.device_scene(scene.packed())
        x = np.ascontiguousarray(starts, dtype=np.float64).reshape(-1, 3)
        g = np.ascontiguousarray(goals, dtype=np.float64).reshape(-1, 3)
        if x.shape != g.shape:
            raise ValueError("starts and goals must have the same shape")
        if not (np.isfinite(x).all() and np.isfinite(g).all()):
            raise ValueError("robot state must be finite")
        self.P = x.shape[0]
        self.record = int(record_ticks)
        ap = cfg.params.attractor
        att = np.array([ap.alpha, ap.beta, ap.c], dtype=np.float64)
        prm = np.ascontiguousarray(cfg.params.obstacle.as_tuple(), dtype=np.float64)
        mr = policy_range(cfg.max_range, cfg.params.obstacle.radius) if cfg.policy_only \
            else cfg.max_range
        c = np.array([cfg.dt, cfg.max_time, cfg.robot_radius, cfg.goal_tolerance, cfg.max_accel,
                      cfg.stuck_window, cfg.stuck_speed, mr,
                      1.0 if cfg.hold_mode else 0.0], dtype=np.float64)
        h = ctypes.c_void_p()
        L.call("rmpb_rollout_create", self.grid.handle, self.bundle.handle, self.scene.handle,
               self.P, x.ctypes.data, g.ctypes.data, att.ctypes.data, prm.ctypes.data,
               c.ctypes.data, self.record, ctypes.byref(h))
        self.handle = h
        self.max_steps = int(round(cfg.max_time / cfg.dt))

    def run(self, max_ticks: int | None = None) -> int:
        """Advance up to ``max_ticks`` ticks (default: to completion)."""
        left = ctypes.c_int64(0)
        ticks = self.max_steps + 1 if max_ticks is None else int(max_ticks)
        L.call("rmpb_rollout_run", self.handle, ticks, ctypes.byref(left), None)
        return int(left.value)

    def result(self) -> BatchRolloutResult:
        P = self.P
        out = np.empty(P, np.int32)
        steps = np.empty(P, np.int64)
        ncl = np.empty(P, np.int64)
        x = np.empty((P, 3))
        v = np.empty((P, 3))
        L.call("rmpb_rollout_result", self.handle, out.ctypes.data, steps.ctypes.data,
               ncl.ctypes.data, x.ctypes.data, v.ctypes.data)
        traj = None
        if self.record:
            traj = np.empty((P, self.record + 1, 9))
            L.call("rmpb_rollout_trajectory", self.handle, traj.ctypes.data)
        return BatchRolloutResult([OUTCOMES[int(o)] for o in out], steps, ncl, x, v, traj)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                L.load().rmpb_rollout_destroy(h)
            except Exception:
                pass
            self.handle = None


def rollout_batch(scene: Scene, grid: EsdfGrid, bundle: RayBundle, starts, goals,
                  cfg: BatchRolloutConfig, record_ticks: int = 0) -> BatchRolloutResult:
    """Run every robot to its outcome (SUCCESS / COLLISION / TIMEOUT / STUCK)."""
    rb = RolloutBatch(scene, grid, bundle, starts, goals, cfg, record_ticks)
    rb.run()
    return rb.result()
