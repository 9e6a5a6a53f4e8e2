"""Synthetic workloads of BASELINE.json's configs.

* C1 world: 200 axis-aligned boxes from ``default_rng(0)`` (per box: centre
  U[lo, hi]^3 then half-extents U[0.3, 1.5]^3) in bounds
  [0, 19.9] x [0, 19.9] x [0, 9.9] m; node grid origin 0, res 0.1 m,
  dims (200, 200, 100); values baked then rounded once to f32 (the
  reference's ESDF file precision, geometry.py:466).  f32 sha256 prefix
  3d7616953ef3751e, occupancy 0.2233.
* robot states: ``bench_states`` (rmpnav/bench.py:60-72): free-space
  rejection sampling with clearance 0.4, unit-speed Gaussian directions.
* C3 scans: 128 x 1024 lattice, vfov +-45 deg, synthesized at the states.

The scene distance / bake callables are injected so CPU-only tests can build
the same inputs with the oracle; the product default is the b200 backend.
"""

from __future__ import annotations

import hashlib

import numpy as np

from .core import RobotState
from .geometry import Aabb, EsdfGrid, Primitive, Scene

C1_LO = np.zeros(3)
C1_HI = np.array([19.9, 19.9, 9.9])
C1_RES = 0.1
C1_DIMS = (200, 200, 100)
C1_SHA_PREFIX = "3d7616953ef3751e"


def c1_scene(n_boxes: int = 200, seed: int = 0, lo=C1_LO, hi=C1_HI) -> Scene:
    rng = np.random.default_rng(seed)
    prims = []
    for _ in range(n_boxes):
        c = rng.uniform(lo, hi)
        h = rng.uniform(0.3, 1.5, size=3)
        prims.append(Primitive.box(c, h))
    return Scene(Aabb(lo, hi), prims, seed=seed)


def c1_grid(scene: Scene | None = None, bake=None) -> EsdfGrid:
    """The f32-rounded C1 grid as an EsdfGrid (f64 values, f32-exact)."""
    scene = c1_scene() if scene is None else scene
    if bake is None:
        from ._kernels import get_backend

        bake = get_backend().bake_values
    vals = bake(scene.packed(), np.zeros(3), C1_RES, C1_DIMS)
    vals = np.asarray(vals, dtype=np.float32).astype(np.float64)
    return EsdfGrid(np.zeros(3), C1_RES, C1_DIMS, vals)


# C5: 50 x 50 x 10 m @ 0.05 m (1000 x 1000 x 200 nodes), random boxes at the
# C1 density (200 boxes per 19.9 x 19.9 x 9.9 m), TSDF truncation 4 voxels.
C5_RES = 0.05
C5_DIMS = (1000, 1000, 200)
C5_ORIGIN = np.zeros(3)
C5_HI = np.array([49.95, 49.95, 9.95])
C5_TAU = 0.2


def c5_scene(seed: int = 1) -> Scene:
    ratio = float(np.prod(C5_HI) / np.prod(C1_HI))
    return c1_scene(n_boxes=int(round(200 * ratio)), seed=seed, lo=C5_ORIGIN, hi=C5_HI)


def c5_grids(scene: Scene):
    """(dense QUAD grid, block-hashed BRICK grid, info) of the f32 TSDF,
    baked on the device (clamp(sd, -tau, tau), rounded once to f32)."""
    from . import _lib as L
    from ._kernels import b200

    ds = b200.device_scene(scene.packed())
    brick = b200.DeviceGrid.bake_tsdf(ds, C5_ORIGIN, C5_RES, C5_DIMS, C5_TAU,
                                      storage=L.STORE_F32, layout=L.LAYOUT_BRICK)
    dense = b200.DeviceGrid.bake_tsdf(ds, C5_ORIGIN, C5_RES, C5_DIMS, C5_TAU,
                                      storage=L.STORE_F32, layout=L.LAYOUT_QUAD)
    nb = int(np.prod([(d + 7) // 8 for d in C5_DIMS]))
    info = {"bricks_allocated": brick.bricks, "bricks_total": nb,
            "brick_bytes": brick.device_bytes, "dense_quad_bytes": dense.device_bytes}
    return dense, brick, info


def c5_values_host(scene: Scene, grid=None) -> np.ndarray:
    """The exact C5 node values (f64, f32-exact) for the CPU oracle."""
    if grid is None:
        grid = c5_grids(scene)[1]
    return grid.values()


def grid_sha_prefix(grid: EsdfGrid) -> str:
    return hashlib.sha256(grid.values.astype(np.float32).tobytes()).hexdigest()[:16]


def bench_states(scene: Scene, count: int = 10, seed: int = 123, clearance: float = 0.4,
                 speed: float = 1.0, distance=None) -> list[RobotState]:
    """Deterministic free-space states (rmpnav/bench.py:60-72 sampling order)."""
    if distance is None:
        from ._kernels import get_backend

        be = get_backend()

        def distance(x):
            return float(be.scene_distance_many(scene.packed(), x.reshape(1, 3), 0.0)[0])

    rng = np.random.default_rng(seed)
    out: list[RobotState] = []
    while len(out) < count:
        x = rng.uniform(scene.bounds.lo, scene.bounds.hi)
        if distance(x) <= clearance:
            continue
        v = rng.normal(size=3)
        v *= speed / np.linalg.norm(v)
        out.append(RobotState(x, v))
    return out


def host_box_distance(scene: Scene):
    """Scene distance for BENCH INPUT GENERATION ONLY (rejection sampling of
    start states, never on the evaluated path): a NumPy restatement of the
    union-of-boxes case of _ckern.pyx:21-56 with the same operation order,
    so the accept / reject decisions equal the reference's.  Avoids one GPU
    launch per candidate while synthesising thousands of poses."""
    pk = scene.packed()
    if (pk["kinds"] != 1).any() or (pk["ops"] != 0).any() or (pk["velocities"] != 0).any():
        raise ValueError("host_box_distance handles static union-of-boxes scenes only")
    c, h, empty = pk["centers"], pk["sizes"], float(pk["empty_dist"])

    def distance(x):
        x = np.asarray(x, dtype=np.float64).reshape(3)
        q = np.abs(x - c) - h
        e = np.maximum(q, 0.0)
        mx = np.maximum(np.maximum(q[:, 0], q[:, 1]), q[:, 2])
        dp = np.sqrt(e[:, 0] * e[:, 0] + e[:, 1] * e[:, 1] + e[:, 2] * e[:, 2]) + np.minimum(mx, 0.0)
        return float(min(empty, dp.min())) if dp.size else empty

    return distance


def states_arrays(states) -> tuple[np.ndarray, np.ndarray]:
    x = np.ascontiguousarray([s.position for s in states], dtype=np.float64).reshape(-1, 3)
    v = np.ascontiguousarray([s.velocity for s in states], dtype=np.float64).reshape(-1, 3)
    return x, v


def lidar_scans(scene: Scene, states, rows: int = 128, cols: int = 1024,
                max_range: float = 20.0):
    """C3: synthetic OS0-style scans at the given states (identity pose)."""
    from .rays import synthesize_scan

    return [synthesize_scan(scene, s.position, rows, cols, max_range) for s in states]
