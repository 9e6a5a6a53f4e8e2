"""The ``"b200"`` kernel backend: the reference's backend protocol
(rmpnav/_kernels/ckern.py:19-93, npkern.py:21-221) served by librmpb.so on a
B200, plus fused / batched entries the reference does not have.

Protocol functions (same names, argument meaning and return shapes as the
reference's ``compiled`` backend):

    scene_distance_many(pack, pts, t)                         ckern.py:19-23
    bake_values(pack, origin, res, dims)                      ckern.py:25-35
    esdf_sample_many(values, origin, res, pts)                ckern.py:38-46
    grid_trace(values, origin, res, start, dirs, max_range,
               eps, step_scale, workers=1)                    ckern.py:49-62
    scene_trace(pack, start, dirs, max_range, eps, t,
                workers=1, step_scale=1.0)                    ckern.py:65-77
    policy_reduce(dirs, dists, v, params, min_range=0.0,
                  workers=1)                                  ckern.py:80-93

``workers`` is accepted for signature compatibility; the reference
guarantees results independent of it (_pool.py:1-7) and so does this
backend (fixed reduction order on device).

The reference passes the grid / directions on every call and retains
nothing.  This backend keeps device copies in small caches:
deeply read-only arrays (``EsdfGrid.values``, ``RayBundle.directions``) by
identity -- their content cannot change, and ``EsdfGrid.update`` patches the
device copies itself; writable arrays by address, re-validated bit for bit
against a private snapshot on every hit, so an in-place edit is always
seen.
"""

from __future__ import annotations

import ctypes
import os
import threading
from collections import OrderedDict

import numpy as np

from .. import _lib as L

name = "b200"
compiled = True

_lock = threading.RLock()


def _default_device() -> int:
    for k in ("RMPNAV_DEVICE", "LOCAL_RANK"):
        v = os.environ.get(k, "").strip()
        if v.isdigit():
            return int(v)
    return 0


_device = _default_device()


def set_device(dev: int) -> None:
    """Select the CUDA device new device objects are created on."""
    global _device
    _device = int(dev)
    invalidate_caches()


def get_device() -> int:
    return _device


def _ptr(a) -> int | None:
    return None if a is None else a.ctypes.data


def _f64(a, shape=None):
    """C-contiguous f64 view / copy; the SAME object when ``a`` already is
    that with the wanted shape (the device caches compare identities)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is None:
        return a
    if a.ndim == len(shape) and all(w in (-1, n) for w, n in zip(shape, a.shape)):
        return a
    return a.reshape(shape)


def _vec3(v):
    a = np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(3))
    return a


def _params(params):
    p = np.ascontiguousarray(np.asarray(params, dtype=np.float64).reshape(7))
    return p


# --------------------------------------------------------------------------
# device objects

class DeviceGrid:
    """A map on device (EsdfGrid values in LINEAR / QUAD / BRICK layout)."""

    def __init__(self, values, origin, res, storage=L.STORE_AUTO, layout=L.LAYOUT_AUTO,
                 device=None, brick_fill=None, _handle=None):
        self.device = _device if device is None else int(device)
        self.origin = np.asarray(origin, dtype=np.float64).reshape(3).copy()
        self.res = float(res)
        h = ctypes.c_void_p()
        if _handle is not None:
            h = _handle
            self.dims = tuple(values)
        else:
            v = np.asarray(values)
            if v.ndim != 3:
                raise ValueError(f"grid values must be 3-D, got shape {v.shape}")
            if v.dtype == np.float32:
                v = np.ascontiguousarray(v)
                dt = L.RMPB_F32
            else:
                v = np.ascontiguousarray(v, dtype=np.float64)
                dt = L.RMPB_F64
            self.dims = tuple(int(d) for d in v.shape)
            o = self.origin
            if brick_fill is None:
                L.call("rmpb_grid_create", v.ctypes.data, dt, *self.dims, o[0], o[1], o[2],
                       self.res, int(storage), int(layout), self.device, ctypes.byref(h))
            else:
                L.call("rmpb_grid_create_brick", v.ctypes.data, dt, *self.dims, o[0], o[1], o[2],
                       self.res, float(brick_fill), int(storage), self.device, ctypes.byref(h))
        self.handle = h
        self.refresh_info()

    def refresh_info(self) -> None:
        """Storage / layout / sizes from the handle (they change when a map
        update has to switch the layout)."""
        st, lay, nb, nbr = ctypes.c_int(), ctypes.c_int(), ctypes.c_int64(), ctypes.c_int64()
        L.call("rmpb_grid_info", self.handle, ctypes.byref(st), ctypes.byref(lay),
               ctypes.byref(nb), ctypes.byref(nbr))
        self.storage = {L.STORE_F32: "f32", L.STORE_F64: "f64"}[st.value]
        self.layout = {L.LAYOUT_LINEAR: "linear", L.LAYOUT_QUAD: "quad",
                       L.LAYOUT_BRICK: "brick", L.LAYOUT_PAIR64: "pair64"}[lay.value]
        self.device_bytes = int(nb.value)
        self.bricks = int(nbr.value)

    @classmethod
    def from_device(cls, d_ptr: int, dtype_f32: bool, dims, origin, res, storage=L.STORE_AUTO,
                    layout=L.LAYOUT_AUTO, device=None):
        """Wrap values already resident in device memory (e.g. a torch tensor)."""
        dev = _device if device is None else int(device)
        h = ctypes.c_void_p()
        o = np.asarray(origin, dtype=np.float64).reshape(3)
        L.call("rmpb_grid_create_device", int(d_ptr), L.RMPB_F32 if dtype_f32 else L.RMPB_F64,
               *[int(d) for d in dims], o[0], o[1], o[2], float(res), int(storage), int(layout),
               dev, ctypes.byref(h))
        return cls(tuple(int(d) for d in dims), o, res, device=dev, _handle=h)

    @classmethod
    def bake(cls, scene: "DeviceScene", origin, res, dims, storage=L.STORE_F64,
             layout=L.LAYOUT_AUTO):
        """GPU bake (row f2) straight into a device grid."""
        h = ctypes.c_void_p()
        o = np.asarray(origin, dtype=np.float64).reshape(3)
        L.call("rmpb_bake_grid", scene.handle, o[0], o[1], o[2], float(res),
               *[int(d) for d in dims], int(storage), int(layout), scene.device, ctypes.byref(h))
        return cls(tuple(int(d) for d in dims), o, res, device=scene.device, _handle=h)

    @classmethod
    def bake_tsdf(cls, scene: "DeviceScene", origin, res, dims, tau, storage=L.STORE_F32,
                  layout=L.LAYOUT_BRICK):
        """Truncated GPU bake (clamp(sd, -tau, tau)) into a device grid."""
        h = ctypes.c_void_p()
        o = np.asarray(origin, dtype=np.float64).reshape(3)
        L.call("rmpb_bake_grid_tsdf", scene.handle, o[0], o[1], o[2], float(res),
               *[int(d) for d in dims], float(tau), int(storage), int(layout), scene.device,
               ctypes.byref(h))
        return cls(tuple(int(d) for d in dims), o, res, device=scene.device, _handle=h)

    def values(self) -> np.ndarray:
        """Node values back on the host (f64, C-order), from any layout."""
        out = np.empty(self.dims, dtype=np.float64)
        L.call("rmpb_grid_values", self.handle, out.ctypes.data)
        return out

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                L.load().rmpb_grid_destroy(h)
            except Exception:
                pass
            self.handle = None


class DeviceBundle:
    """Ray directions on device, evaluated in Morton(polar, azimuth) order."""

    def __init__(self, dirs=None, order=L.ORDER_MORTON, device=None, halton_n=None,
                 lattice=None):
        """``halton_n``: the reference's Halton bundle of that size generated
        on device (rays.py:78-86); ``lattice=(rows, cols, vfov_deg)``: the
        spherical-grid scan pattern generated on device (rays.py:176-199)."""
        self.device = _device if device is None else int(device)
        h = ctypes.c_void_p()
        if halton_n is not None:
            L.call("rmpb_bundle_halton", int(halton_n), int(order), self.device, ctypes.byref(h))
            self.n = int(halton_n)
        elif lattice is not None:
            rows, cols, vfov = lattice
            L.call("rmpb_bundle_lattice", int(rows), int(cols), float(vfov), int(order),
                   self.device, ctypes.byref(h))
            self.n = int(rows) * int(cols)
        else:
            d = _f64(dirs, (-1, 3))
            self.n = d.shape[0]
            L.call("rmpb_bundle_create", d.ctypes.data, self.n, int(order), self.device,
                   ctypes.byref(h))
        self.handle = h
        self.order = order

    def directions(self) -> np.ndarray:
        out = np.empty((self.n, 3))
        L.call("rmpb_bundle_directions", self.handle, out.ctypes.data)
        return out

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                L.load().rmpb_bundle_destroy(h)
            except Exception:
                pass
            self.handle = None


class DeviceOccupancy:
    """K5: bit-packed occupancy (node value <= 0) of a device grid, for the
    Amanatides-Woo DDA traversal (not the reference's sphere trace)."""

    def __init__(self, grid: "DeviceGrid"):
        self.grid = grid
        self.device = grid.device
        self.dims = grid.dims
        h = ctypes.c_void_p()
        L.call("rmpb_occupancy_create", grid.handle, ctypes.byref(h))
        self.handle = h

    def bits(self) -> np.ndarray:
        nx, ny, nz = self.dims
        out = np.empty(nx * ny * ((nz + 31) // 32), dtype=np.uint32)
        L.call("rmpb_occupancy_bits", self.handle, out.ctypes.data)
        return out

    def trace(self, start, dirs, max_range):
        """(t float32 (+inf = miss), voxel (N,3) int32 (-1 = miss), visited)."""
        d = _f64(dirs, (-1, 3))
        n = d.shape[0]
        t = np.empty(n, np.float32)
        vox = np.empty((n, 3), np.int32)
        steps = np.empty(n, np.int32)
        s = _vec3(start)  # named: a temporary's buffer would be freed before the call
        L.call("rmpb_dda_trace", self.handle, d.ctypes.data, n, s.ctypes.data,
               float(max_range), t.ctypes.data, vox.ctypes.data, steps.ctypes.data, None)
        return t, vox, steps

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                L.load().rmpb_occupancy_destroy(h)
            except Exception:
                pass
            self.handle = None


class DeviceScene:
    """Analytic primitive scene on device (pack of geometry.py:177-197)."""

    def __init__(self, pack: dict, device=None):
        self.device = _device if device is None else int(device)
        k = np.ascontiguousarray(pack["kinds"], dtype=np.int8)
        o = np.ascontiguousarray(pack["ops"], dtype=np.int8)
        c = _f64(pack["centers"], (-1, 3))
        s = _f64(pack["sizes"], (-1, 3))
        v = _f64(pack["velocities"], (-1, 3))
        n = int(k.shape[0])
        if not (o.shape[0] == c.shape[0] == s.shape[0] == v.shape[0] == n):
            raise ValueError("scene pack arrays must have equal length")
        h = ctypes.c_void_p()
        L.call("rmpb_scene_create", k.ctypes.data, o.ctypes.data, c.ctypes.data, s.ctypes.data,
               v.ctypes.data, n, float(pack["empty_dist"]), self.device, ctypes.byref(h))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                L.load().rmpb_scene_destroy(h)
            except Exception:
                pass
            self.handle = None


# --------------------------------------------------------------------------
# caches (the reference re-passes inputs on every call)

_MAX_GRIDS = 4
_MAX_BUNDLES = 16
_grids: "OrderedDict[tuple, tuple]" = OrderedDict()
_bundles: "OrderedDict[tuple, tuple]" = OrderedDict()
_scenes: "OrderedDict[int, tuple]" = OrderedDict()


def _frozen(a: np.ndarray) -> bool:
    """True when neither the array nor any base it views is writable (e.g.
    EsdfGrid.values, RayBundle.directions): its content cannot change through
    NumPy, so a cache hit needs no content check."""
    while isinstance(a, np.ndarray):
        if a.flags.writeable:
            return False
        a = a.base
    return True


def _bits(a: np.ndarray) -> np.ndarray:
    """Unsigned-integer view of a contiguous array (bitwise compare, NaN-safe)."""
    return a.reshape(-1).view({8: np.uint64, 4: np.uint32, 2: np.uint16, 1: np.uint8}[a.itemsize])


def _same_content(a: np.ndarray, snap) -> bool:
    """Writable arrays are re-validated on every cache hit against a private
    snapshot, bit for bit (one pass over the array: ~3 ms for the 32 MB C1
    map -- the reference re-reads the whole map on every call too,
    ckern.py:49-62).  Frozen arrays carry no snapshot."""
    return snap is None or (a.shape == snap.shape and np.array_equal(_bits(a), _bits(snap)))


def _snapshot(a: np.ndarray, frozen: bool):
    return None if frozen else a.copy()


def _entry_valid(a: np.ndarray, snap) -> bool:
    """A keyed entry (same address, shape, dtype) serves ``a`` when it was
    stored for a deeply frozen array and ``a`` is frozen too (the entry keeps
    that buffer alive, so the address cannot belong to another allocation,
    and its content cannot change), or when ``a`` equals its snapshot."""
    if snap is None:
        return _frozen(a)
    return _same_content(a, snap)


def invalidate_caches() -> None:
    """Drop every cached device grid / bundle / scene."""
    with _lock:
        _grids.clear()
        _bundles.clear()
        _scenes.clear()
        _fast.clear()
        _patterns.clear()


# Identity fast path for the control-loop pattern (the same EsdfGrid.values /
# RayBundle.directions objects passed on every call): id(array) -> entry,
# valid while the entry holds the array (so the id cannot be reused).  Only
# deeply frozen arrays take it (their content cannot change behind the cache;
# EsdfGrid.update patches the device copies itself): ~2 us instead of the
# keyed lookup.
_fast: "OrderedDict[int, tuple]" = OrderedDict()
_FAST_MAX = 16


def _fast_get(obj, extra):
    e = _fast.get(id(obj))
    if e is None or e[0] is not obj or e[1] != extra:
        return None
    return e[2]


def _fast_put(obj, extra, dev_obj) -> None:
    with _lock:
        if len(_fast) >= _FAST_MAX:
            _fast.popitem(last=False)
        _fast[id(obj)] = (obj, extra, dev_obj)


def device_grid(values, origin, res) -> DeviceGrid:
    """Device copy of an EsdfGrid's values (cached)."""
    if isinstance(values, DeviceGrid):
        return values
    o_l = origin.tolist() if type(origin) is np.ndarray else [float(x) for x in origin]
    extra = (o_l, res, _device)
    hit = _fast_get(values, extra)
    if hit is not None:
        return hit
    g = _device_grid_keyed(values, origin, res)
    if (type(values) is np.ndarray and values.flags.c_contiguous and values.dtype in
            (np.float64, np.float32) and _frozen(values)):
        _fast_put(values, extra, g)
    return g


def _device_grid_keyed(values, origin, res) -> DeviceGrid:
    v = np.asarray(values)
    if v.dtype != np.float32:
        v = np.ascontiguousarray(v, dtype=np.float64)
    else:
        v = np.ascontiguousarray(v)
    o = tuple(float(x) for x in np.asarray(origin, dtype=np.float64).reshape(3))
    key = (v.ctypes.data, v.shape, v.dtype.str, o, float(res), _device)
    with _lock:
        hit = _grids.get(key)
        if hit is not None and _entry_valid(v, hit[2]):
            _grids.move_to_end(key)
            return hit[0]
        frozen = _frozen(v)
        g = DeviceGrid(v, o, res)
        _grids[key] = (g, v, _snapshot(v, frozen))  # `v` alive: the address stays unique
        while len(_grids) > _MAX_GRIDS:
            _grids.popitem(last=False)
        return g


def grid_updated(values: np.ndarray, corner, sub: np.ndarray) -> None:
    """EsdfGrid.update hook: ``values[corner : corner + sub.shape] = sub`` has
    just been written on the host.  Every cached device copy of ``values`` is
    patched in place (only the touched nodes cross PCIe; QUAD / LINEAR /
    PAIR64 layouts).  A copy that cannot take the patch (f32 storage and
    values that are not f32-exact) is re-uploaded whole into the SAME handle
    (rmpb_grid_update: holders such as a LatencyServer see the new map); one
    that cannot be updated at all is dropped from the cache."""
    sub = np.ascontiguousarray(sub, dtype=np.float64)
    i0, j0, k0 = (int(c) for c in corner)
    ni, nj, nk = sub.shape
    with _lock:
        targets = []
        for k, e in list(_fast.items()):
            if e[0] is values:
                targets.append(("fast", k, e[2]))
        ptr = values.ctypes.data
        for k, e in list(_grids.items()):
            if k[0] == ptr and k[1] == values.shape:  # this buffer, any view of it
                targets.append(("keyed", k, e[0]))
        done = {}
        for kind, k, g in targets:
            ok = done.get(id(g))
            if ok is None:
                lib = L.load()
                st = lib.rmpb_grid_update_region(g.handle, sub.ctypes.data, L.RMPB_F64,
                                                 i0, j0, k0, ni, nj, nk)
                if st != 0:  # whole re-upload into the same handle
                    full = np.ascontiguousarray(values, dtype=np.float64)
                    st = lib.rmpb_grid_update(g.handle, full.ctypes.data, L.RMPB_F64)
                    if st == 0:
                        g.refresh_info()
                ok = done[id(g)] = st == 0
            if not ok:
                (_fast if kind == "fast" else _grids).pop(k, None)


def device_bundle(dirs) -> DeviceBundle:
    if isinstance(dirs, DeviceBundle):
        return dirs
    hit = _fast_get(dirs, _device)
    if hit is not None:
        return hit
    b = _device_bundle_keyed(dirs)
    if (type(dirs) is np.ndarray and dirs.flags.c_contiguous and dirs.dtype == np.float64 and
            dirs.ndim == 2 and dirs.shape[1] == 3 and _frozen(dirs)):
        _fast_put(dirs, _device, b)
    return b


def _device_bundle_keyed(dirs) -> DeviceBundle:
    d = _f64(dirs, (-1, 3))
    key = (d.ctypes.data, d.shape[0], _device)
    with _lock:
        hit = _bundles.get(key)
        if hit is not None and _entry_valid(d, hit[2]):
            _bundles.move_to_end(key)
            return hit[0]
        b = DeviceBundle(d)
        _bundles[key] = (b, d, _snapshot(d, _frozen(d)))
        while len(_bundles) > _MAX_BUNDLES:
            _bundles.popitem(last=False)
        return b


def register_bundle(dirs: np.ndarray, dev: DeviceBundle) -> None:
    """Associate a host direction array with an existing device bundle (e.g.
    one generated on device) so later calls do not re-upload it."""
    d = _f64(dirs, (-1, 3))
    key = (d.ctypes.data, d.shape[0], dev.device)
    with _lock:
        _bundles[key] = (dev, d, _snapshot(d, _frozen(d)))
        while len(_bundles) > _MAX_BUNDLES:
            _bundles.popitem(last=False)


def device_scene(pack: dict) -> DeviceScene:
    key = id(pack)
    with _lock:
        hit = _scenes.get(key)
        if hit is not None and hit[1] is pack:
            return hit[0]
        s = DeviceScene(pack)
        _scenes[key] = (s, pack)
        while len(_scenes) > 16:
            _scenes.popitem(last=False)
        return s


# --------------------------------------------------------------------------
# the reference protocol

def scene_distance_many(pack: dict, pts: np.ndarray, t: float) -> np.ndarray:
    pts = _f64(pts, (-1, 3))
    out = np.empty(pts.shape[0])
    L.call("rmpb_scene_distance", device_scene(pack).handle, pts.ctypes.data, pts.shape[0],
           float(t), out.ctypes.data, None)
    return out


def bake_values(pack: dict, origin, res: float, dims) -> np.ndarray:
    nx, ny, nz = (int(d) for d in dims)
    o = np.asarray(origin, dtype=np.float64).reshape(3)
    out = np.empty((nx, ny, nz), dtype=np.float64)
    L.call("rmpb_bake", device_scene(pack).handle, o[0], o[1], o[2], float(res), nx, ny, nz,
           out.ctypes.data, None)
    return out


def esdf_sample_many(values, origin, res: float, pts: np.ndarray):
    g = device_grid(values, origin, res)
    pts = _f64(pts, (-1, 3))
    n = pts.shape[0]
    d = np.empty(n)
    gr = np.empty((n, 3))
    fl = np.empty(n, dtype=np.uint8)
    L.call("rmpb_esdf_sample", g.handle, pts.ctypes.data, n, d.ctypes.data, gr.ctypes.data,
           fl.ctypes.data, None)
    return d, gr, fl.astype(bool)


def grid_trace(values, origin, res: float, start, dirs: np.ndarray, max_range: float,
               eps: float, step_scale: float, workers: int = 1) -> np.ndarray:
    return grid_trace_ex(values, origin, res, start, dirs, max_range, eps, step_scale)[0]


def grid_trace_ex(values, origin, res, start, dirs, max_range, eps, step_scale,
                  with_cells=False, with_steps=False):
    """grid_trace plus optional hit cells (N,3 int32; -1 on miss) and steps."""
    g = device_grid(values, origin, res)
    d = _f64(dirs, (-1, 3))
    s = _vec3(start)
    n = d.shape[0]
    t = np.empty(n)
    cells = np.empty((n, 3), np.int32) if with_cells else None
    steps = np.empty(n, np.int32) if with_steps else None
    L.call("rmpb_grid_trace", g.handle, d.ctypes.data, n, s.ctypes.data, float(max_range),
           float(eps), float(step_scale), t.ctypes.data, _ptr(cells), _ptr(steps), None)
    return t, cells, steps


def scene_trace(pack: dict, start, dirs: np.ndarray, max_range: float, eps: float, t: float,
                workers: int = 1, step_scale: float = 1.0) -> np.ndarray:
    d = _f64(dirs, (-1, 3))
    s = _vec3(start)
    out = np.empty(d.shape[0])
    L.call("rmpb_scene_trace", device_scene(pack).handle, s.ctypes.data, d.ctypes.data,
           d.shape[0], float(max_range), float(eps), float(t), float(step_scale), out.ctypes.data,
           None)
    return out


def policy_reduce(dirs: np.ndarray, dists: np.ndarray, v, params: tuple, min_range: float = 0.0,
                  workers: int = 1):
    d = _f64(dirs, (-1, 3))
    r = _f64(dists, (-1,))
    if r.shape[0] != d.shape[0]:
        raise ValueError(f"dirs ({d.shape[0]}) and dists ({r.shape[0]}) lengths differ")
    slot = np.empty(13)
    va, pa = _vec3(v), _params(params)  # named: kept alive across the call
    L.call("rmpb_policy_reduce", d.ctypes.data, r.ctypes.data, d.shape[0], va.ctypes.data,
           pa.ctypes.data, float(min_range), slot.ctypes.data, None)
    return slot[0:9].reshape(3, 3).copy(), slot[9:12].copy(), int(slot[12])


# --------------------------------------------------------------------------
# fused / batched entries (beyond the reference protocol)

_param_cache: "OrderedDict[tuple, tuple]" = OrderedDict()


def _params_cached(params):
    """(array, pointer) of the 7 params; LRU-cached for hashable params.
    The CALLER must keep the returned array alive until the C call returns
    (the pointer alone does not own the buffer)."""
    key = (params if type(params) is tuple else tuple(params)) \
        if not isinstance(params, np.ndarray) else None
    if key is not None:
        hit = _param_cache.get(key)  # (a dict lookup is atomic: no lock on a hit)
        if hit is not None:
            return hit
        with _lock:
            hit = _param_cache.get(key)
            if hit is None:
                a = _params(params)
                hit = (a, a.ctypes.data)
                _param_cache[key] = hit
                while len(_param_cache) > 64:
                    _param_cache.popitem(last=False)
        return hit
    a = _params(params)
    return a, a.ctypes.data


_tls = threading.local()


def _scratch():
    """Per-thread pinned-free scratch (pose in, 16 doubles out) with cached
    addresses: ndarray.ctypes costs ~2 us per access."""
    s = getattr(_tls, "s", None)
    if s is None:
        xv = np.empty(6)
        out = np.empty(16)
        s = (xv, xv.ctypes.data, out, out.ctypes.data)
        _tls.s = s
    return s


def ray_policy_fused(values, origin, res, start, velocity, dirs, params, max_range, eps,
                     step_scale, with_rays=False):
    """Fused ray_policy (policies.py:182-192): returns (slot13, accel3) and,
    with ``with_rays``, per-ray (t, cells, steps) in original ray order."""
    g = device_grid(values, origin, res)
    b = device_bundle(dirs)
    xv, base, out, optr = _scratch()
    xv[0:3] = start
    xv[3:6] = velocity
    t = cells = steps = None
    if with_rays:
        t = np.empty(b.n)
        cells = np.empty((b.n, 3), np.int32)
        steps = np.empty(b.n, np.int32)
    pa, pptr = _params_cached(params)  # `pa` keeps the buffer alive across the call
    L.check(L.load().rmpb_ray_policy(
        g.handle, b.handle, base, base + 24, pptr,
        float(max_range), float(eps), float(step_scale), optr, optr + 104,
        _ptr(t), _ptr(cells), _ptr(steps), None), "rmpb_ray_policy")
    del pa
    out = out.copy()
    slot, acc = out[:13], out[13:]
    if with_rays:
        return slot, acc, t, cells, steps
    return slot, acc


def ray_policy_batch(values, origin, res, positions, velocities, dirs, params, max_range, eps,
                     step_scale):
    """P poses in one launch (config C4): returns (slots P x 13, accels P x 3)."""
    g = device_grid(values, origin, res)
    b = device_bundle(dirs)
    x = _f64(positions, (-1, 3))
    v = _f64(velocities, (-1, 3))
    if x.shape != v.shape:
        raise ValueError("positions and velocities must have the same shape")
    P = x.shape[0]
    slots = np.empty((P, 13))
    acc = np.empty((P, 3))
    if P == 0:
        return slots, acc
    pa = _params(params)
    L.call("rmpb_ray_policy_batch", g.handle, b.handle, x.ctypes.data, v.ctypes.data, P,
           pa.ctypes.data, float(max_range), float(eps), float(step_scale),
           slots.ctypes.data, acc.ctypes.data, None)
    return slots, acc


def lidar_policy_fused(dirs, R, ranges, valid, velocity, params, min_range):
    """LiDAR-direct (policies.py:195-205) in one launch.  ``dirs`` are the
    sensor-frame beam directions and ``R`` the orientation (world = dirs @ R.T);
    pass R=None for world-frame directions."""
    d = _f64(dirs, (-1, 3))
    r = _f64(ranges, (-1,))
    n = d.shape[0]
    if r.shape[0] != n:
        raise ValueError("directions and ranges must have equal length")
    vl = None
    if valid is not None:
        vl = np.ascontiguousarray(np.asarray(valid, dtype=bool).reshape(-1)).view(np.uint8)
        if vl.shape[0] != n:
            raise ValueError("valid must have the same length as ranges")
    Rm = None if R is None else _f64(R, (3, 3))
    slot = np.empty(13)
    acc = np.empty(3)
    va, pa = _vec3(velocity), _params(params)
    if _frozen(d) and n >= 4096:
        pat = device_bundle_identity(d)
        L.call("rmpb_lidar_policy_bundle", pat.handle, _ptr(Rm), r.ctypes.data, _ptr(vl),
               va.ctypes.data, pa.ctypes.data, float(min_range),
               slot.ctypes.data, acc.ctypes.data, None)
    else:
        L.call("rmpb_lidar_policy", d.ctypes.data, _ptr(Rm), r.ctypes.data, _ptr(vl), n,
               va.ctypes.data, pa.ctypes.data, float(min_range),
               slot.ctypes.data, acc.ctypes.data, None)
    return slot, acc


_patterns: "OrderedDict[tuple, tuple]" = OrderedDict()


def device_bundle_identity(d: np.ndarray) -> DeviceBundle:
    """Read-only sensor lattices (rays.py:176-191 caches them read-only) are
    kept on device so a scan call only moves ranges + validity."""
    key = (d.ctypes.data, d.shape[0], _device)
    with _lock:
        hit = _patterns.get(key)
        if hit is not None and _entry_valid(d, hit[2]):
            return hit[0]
        b = DeviceBundle(d, order=L.ORDER_IDENTITY)
        _patterns[key] = (b, d, _snapshot(d, _frozen(d)))
        while len(_patterns) > 8:
            _patterns.popitem(last=False)
        return b


def lidar_points_fused(xyz, R, velocity, params, min_range):
    """LiDAR-direct policy from raw sensor-frame points (f32 xyz)."""
    p = np.ascontiguousarray(np.asarray(xyz, dtype=np.float32).reshape(-1, 3))
    Rm = None if R is None else _f64(R, (3, 3))
    slot = np.empty(13)
    acc = np.empty(3)
    if p.shape[0] == 0:
        slot[:] = 0.0
        acc[:] = 0.0
        return slot, acc
    va, pa = _vec3(velocity), _params(params)
    L.call("rmpb_lidar_points", p.ctypes.data, _ptr(Rm), p.shape[0], va.ctypes.data,
           pa.ctypes.data, float(min_range), slot.ctypes.data, acc.ctypes.data, None)
    return slot, acc


def pinv_psd(a, rcond: float = 1e-8) -> np.ndarray:
    """Batch of symmetric 3x3 -> PSD pseudo-inverse on device (core.py:103-115)."""
    m = _f64(a)
    single = m.shape == (3, 3)
    m = m.reshape(-1, 9)
    out = np.empty_like(m)
    L.call("rmpb_pinv_psd_rcond", m.ctypes.data, m.shape[0], float(rcond), out.ctypes.data, None)
    return out.reshape(3, 3) if single else out.reshape(-1, 3, 3)
