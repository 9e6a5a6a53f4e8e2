"""Maps the hot path traverses (mirror of the parts of rmpnav/geometry.py the
path and its input side need).

* ``EsdfGrid`` (geometry.py:215-255): node-sampled signed distances,
  positive = free; node (i,j,k) at origin + (i,j,k)*resolution; values f64
  C-order, shape == dims >= 2 per axis.
* ``Aabb`` / ``Primitive`` / ``Scene`` and the flat pack (geometry.py:65-197)
  -- the analytic world the bench and the LiDAR scan synthesis use.
* ``bake_esdf`` (geometry.py:271-289) runs on the B200 (row f2), including
  the reference's 512^3-node bound; ``bake_esdf_device`` skips the host copy
  and the bound (the 1000x1000x200 config needs 2e8 nodes).
* ``esdf_lookup`` (geometry.py:292-309, row f4) and the ESDF binary file
  (geometry.py:455-488: documented header, f32 x-fastest payload).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

from ._kernels import get_backend

__all__ = ["Aabb", "Primitive", "Scene", "EsdfGrid", "EsdfSample", "SceneFormatError",
           "scene_distance", "scene_distance_many", "bake_esdf", "bake_esdf_device",
           "esdf_lookup", "esdf_lookup_many", "occupied_fraction", "save_esdf", "load_esdf",
           "DEFAULT_RESOLUTION", "DEFAULT_MAX_VOXELS"]

DEFAULT_RESOLUTION = 0.2
DEFAULT_MAX_VOXELS = 512 ** 3
KIND_SPHERE, KIND_BOX = 0, 1
OP_UNION, OP_SUBTRACT = 0, 1
ESDF_MAGIC = b"ESDF"
ESDF_VERSION = 1
# The reference's format string "<4sI3ddd3I" (geometry.py:458) has one 'd'
# too many for the fields it documents and packs (magic, version, origin
# 3xf64, resolution f64, dims 3xu32), so its save_esdf / load_esdf raise
# struct.error.  This mirror implements the documented 52-byte header.
_ESDF_HEADER = struct.Struct("<4sI3dd3I")


class SceneFormatError(ValueError):
    """Malformed or unsupported map / scan file."""


@dataclass(frozen=True)
class Aabb:
    lo: np.ndarray
    hi: np.ndarray

    def __post_init__(self):
        lo = np.asarray(self.lo, dtype=float).reshape(3)
        hi = np.asarray(self.hi, dtype=float).reshape(3)
        if not (hi > lo).all():
            raise ValueError("degenerate bounds: hi must exceed lo on every axis")
        object.__setattr__(self, "lo", lo)
        object.__setattr__(self, "hi", hi)

    @property
    def diagonal(self) -> float:
        return float(np.linalg.norm(self.hi - self.lo))

    @property
    def center(self) -> np.ndarray:
        return 0.5 * (self.lo + self.hi)

    def contains(self, p) -> bool:
        p = np.asarray(p, dtype=float)
        return bool((p >= self.lo).all() and (p <= self.hi).all())


@dataclass(frozen=True)
class Primitive:
    """Sphere (size = radius) or axis-aligned box (size = half extents)."""

    kind: str
    center: np.ndarray
    size: np.ndarray
    op: str = "union"
    velocity: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def __post_init__(self):
        if self.kind not in ("sphere", "box"):
            raise ValueError(f"unknown primitive kind {self.kind!r}")
        if self.op not in ("union", "subtract"):
            raise ValueError(f"unknown boolean op {self.op!r}")
        size = np.asarray(self.size, dtype=float)
        size = np.full(3, float(size)) if size.ndim == 0 else size.reshape(3)
        if (size <= 0).any():
            raise ValueError("primitive size must be positive")
        if self.kind == "sphere" and not (size == size[0]).all():
            raise ValueError("sphere size entries must be equal (the radius)")
        object.__setattr__(self, "center", np.asarray(self.center, dtype=float).reshape(3))
        object.__setattr__(self, "size", size)
        object.__setattr__(self, "velocity", np.asarray(self.velocity, dtype=float).reshape(3))

    @staticmethod
    def sphere(center, radius: float, op: str = "union", velocity=(0, 0, 0)) -> "Primitive":
        return Primitive("sphere", center, float(radius), op, velocity)

    @staticmethod
    def box(center, half_extents, op: str = "union", velocity=(0, 0, 0)) -> "Primitive":
        return Primitive("box", center, half_extents, op, velocity)


class Scene:
    """Ordered primitives inside bounds; immutable, with a cached flat pack."""

    def __init__(self, bounds: Aabb, primitives=(), seed=None, start=None, goal=None):
        self.bounds = bounds
        self.primitives = tuple(primitives)
        self.seed = seed
        self.start = None if start is None else np.asarray(start, dtype=float).reshape(3)
        self.goal = None if goal is None else np.asarray(goal, dtype=float).reshape(3)
        n = len(self.primitives)
        pack = {
            "kinds": np.array([KIND_SPHERE if p.kind == "sphere" else KIND_BOX
                               for p in self.primitives], dtype=np.int8).reshape(n),
            "ops": np.array([OP_UNION if p.op == "union" else OP_SUBTRACT
                             for p in self.primitives], dtype=np.int8).reshape(n),
            "centers": np.array([p.center for p in self.primitives], dtype=np.float64).reshape(n, 3),
            "sizes": np.array([p.size for p in self.primitives], dtype=np.float64).reshape(n, 3),
            "velocities": np.array([p.velocity for p in self.primitives],
                                   dtype=np.float64).reshape(n, 3),
            "empty_dist": bounds.diagonal,
        }
        self._pack = pack

    @property
    def is_dynamic(self) -> bool:
        return any(bool((p.velocity != 0).any()) for p in self.primitives)

    @property
    def empty_distance(self) -> float:
        return self.bounds.diagonal

    def packed(self) -> dict:
        return self._pack


def scene_distance_many(scene: Scene, pts, t: float = 0.0) -> np.ndarray:
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
    return get_backend().scene_distance_many(scene.packed(), pts, float(t))


def scene_distance(scene: Scene, x, t: float = 0.0) -> float:
    return float(scene_distance_many(scene, np.asarray(x, dtype=float).reshape(1, 3), t)[0])


def deeply_frozen(a) -> bool:
    """True when neither ``a`` nor any array it views is writable: its content
    cannot change through NumPy without re-enabling a flag by hand."""
    while isinstance(a, np.ndarray):
        if a.flags.writeable:
            return False
        a = a.base
    return True


def immutable_f64(a, shape=None) -> np.ndarray:
    """A read-only f64 C-contiguous array with the content of ``a``: ``a``
    itself when it is already that and deeply frozen, else a private copy
    whose buffer is read-only (device caches key on identity, so the content
    behind a cached array must not change without them seeing it)."""
    arr = np.asarray(a)
    if (arr.dtype == np.float64 and arr.flags.c_contiguous and deeply_frozen(arr)
            and (shape is None or arr.shape == tuple(shape))):
        return arr
    out = np.array(arr, dtype=np.float64, order="C", copy=True)
    if shape is not None:
        out = out.reshape(shape)
    out.setflags(write=False)
    return out


@dataclass(frozen=True)
class EsdfGrid:
    """Regular node grid of signed distances (positive = free).

    Deviation from the reference (geometry.py:215-240, whose ``values`` may
    alias the caller's array and stay writable): ``values`` is a read-only
    private copy, so a device-resident copy of the map can never be served
    stale.  Edit the map through :meth:`update`, which also patches every
    cached device copy (only the touched nodes move over PCIe)."""

    origin: np.ndarray
    resolution: float
    dims: tuple
    values: np.ndarray

    def __post_init__(self):
        if self.resolution <= 0:
            raise ValueError("resolution must be positive")
        dims = tuple(int(d) for d in self.dims)
        if len(dims) != 3 or min(dims) < 2:
            raise ValueError("grid needs at least 2 nodes per axis")
        vals = np.asarray(self.values)
        if vals.shape != dims:
            raise ValueError(f"values shape {vals.shape} != dims {dims}")
        object.__setattr__(self, "origin", np.asarray(self.origin, dtype=float).reshape(3))
        object.__setattr__(self, "dims", dims)
        frozen = immutable_f64(vals)
        object.__setattr__(self, "values", frozen)
        object.__setattr__(self, "_owned", frozen is not vals)

    def update(self, index, values) -> None:
        """Write ``values`` into ``self.values[index]`` (``index``: a tuple of
        three ints / unit-step slices) and bring every cached device copy of
        this map up to date before returning."""
        if not isinstance(index, tuple) or len(index) != 3:
            raise ValueError("index must be a tuple of 3 ints / slices")
        box = []
        for ax, ix in enumerate(index):
            n = self.dims[ax]
            if isinstance(ix, slice):
                a, b, st = ix.indices(n)
                if st != 1:
                    raise ValueError("update slices must have unit step")
            else:
                a = int(ix)
                if a < 0:
                    a += n
                if not 0 <= a < n:
                    raise IndexError(f"index {ix} out of range for axis {ax} of size {n}")
                b = a + 1
            if b <= a:
                return
            box.append((a, b))
        sl = tuple(slice(a, b) for a, b in box)
        new = np.broadcast_to(np.asarray(values, dtype=np.float64),
                              tuple(b - a for a, b in box))
        if not getattr(self, "_owned", False):
            # shared with another owner (a frozen input array): copy first, so
            # the edit stays private to this grid (a new array = new cache key)
            own = np.array(self.values, dtype=np.float64, order="C", copy=True)
            own.setflags(write=False)
            object.__setattr__(self, "values", own)
            object.__setattr__(self, "_owned", True)
        buf = self.values
        buf.setflags(write=True)
        try:
            buf[sl] = new
        finally:
            buf.setflags(write=False)
        hook = getattr(get_backend(), "grid_updated", None)
        if hook is not None:
            hook(buf, tuple(a for a, _ in box), np.ascontiguousarray(buf[sl]))

    @property
    def domain(self) -> Aabb:
        return Aabb(self.origin, self.origin + (np.array(self.dims) - 1) * self.resolution)

    def node_position(self, i: int, j: int, k: int) -> np.ndarray:
        return self.origin + np.array([i, j, k], dtype=float) * self.resolution


@dataclass(frozen=True)
class EsdfSample:
    distance: float
    gradient: np.ndarray
    extrapolated: bool = False

    @property
    def degenerate(self) -> bool:
        return not bool((self.gradient != 0.0).any())


def _bake_dims(scene: Scene, resolution: float, pad: float):
    lo = scene.bounds.lo - pad
    hi = scene.bounds.hi + pad
    dims = tuple(int(np.ceil((hi[a] - lo[a]) / resolution)) + 1 for a in range(3))
    return lo, dims


def bake_esdf(scene: Scene, resolution: float = DEFAULT_RESOLUTION, pad: float = 0.0,
              max_voxels: int = DEFAULT_MAX_VOXELS) -> EsdfGrid:
    """Sample the scene at t = 0 on the grid covering its (padded) bounds."""
    if resolution <= 0:
        raise ValueError("resolution must be positive")
    lo, dims = _bake_dims(scene, resolution, pad)
    n = dims[0] * dims[1] * dims[2]
    if n > max_voxels:
        raise ValueError(f"grid of {dims} = {n} voxels exceeds the {max_voxels} voxel bound")
    values = get_backend().bake_values(scene.packed(), lo, float(resolution), dims)
    return EsdfGrid(lo, float(resolution), dims, values)


def bake_esdf_device(scene: Scene, origin, resolution: float, dims, storage: str = "f32",
                     layout: str = "quad"):
    """Bake straight into a device map (no host copy, no node bound).
    ``storage='f32'`` rounds once to f32, the reference ESDF file precision."""
    from . import _lib as L
    from ._kernels import b200

    st = {"f32": L.STORE_F32, "f64": L.STORE_F64, "auto": L.STORE_AUTO}[storage]
    lay = {"linear": L.LAYOUT_LINEAR, "quad": L.LAYOUT_QUAD}[layout]
    return b200.DeviceGrid.bake(b200.device_scene(scene.packed()), origin, resolution, dims,
                                storage=st, layout=lay)


def esdf_lookup_many(grid: EsdfGrid, pts):
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
    return get_backend().esdf_sample_many(grid.values, grid.origin, grid.resolution, pts)


def esdf_lookup(grid: EsdfGrid, x) -> EsdfSample:
    d, g, flag = esdf_lookup_many(grid, np.asarray(x, dtype=float).reshape(1, 3))
    return EsdfSample(float(d[0]), g[0], bool(flag[0]))


def occupied_fraction(scene: Scene, resolution: float = DEFAULT_RESOLUTION) -> float:
    """Fraction of grid nodes inside solid geometry (values <= 0)."""
    return float(np.mean(bake_esdf(scene, resolution).values <= 0.0))


def save_esdf(grid: EsdfGrid, path) -> None:
    head = _ESDF_HEADER.pack(ESDF_MAGIC, ESDF_VERSION, *map(float, grid.origin),
                             float(grid.resolution), *grid.dims)
    with open(path, "wb") as fh:
        fh.write(head)
        fh.write(np.asarray(grid.values, dtype=np.float32).tobytes(order="F"))


def load_esdf(path) -> EsdfGrid:
    with open(path, "rb") as fh:
        raw = fh.read(_ESDF_HEADER.size)
        if len(raw) != _ESDF_HEADER.size:
            raise SceneFormatError(f"{path}: truncated ESDF header")
        magic, version, ox, oy, oz, res, nx, ny, nz = _ESDF_HEADER.unpack(raw)
        if magic != ESDF_MAGIC:
            raise SceneFormatError(f"{path}: bad magic {magic!r}")
        if version != ESDF_VERSION:
            raise SceneFormatError(f"{path}: unsupported ESDF version {version}")
        payload = fh.read(4 * nx * ny * nz)
    if len(payload) != 4 * nx * ny * nz:
        raise SceneFormatError(f"{path}: truncated ESDF payload")
    vals = np.frombuffer(payload, dtype="<f4").reshape((nx, ny, nz), order="F")
    return EsdfGrid(np.array([ox, oy, oz]), res, (nx, ny, nz),
                    np.ascontiguousarray(vals, dtype=np.float64))
