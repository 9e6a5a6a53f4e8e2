"""ctypes binding of ``librmpb.so`` (the C ABI declared in include/rmpb.h).

The library is built in-tree (``paper_2301_08068_b200/librmpb.so``) by
``__graft_entry__.build()`` / ``make -C paper_2301_08068_b200/csrc``.  There
is no fallback: if the library is missing or cannot be loaded, importing the
backend raises ImportError, and calls fail with RuntimeError when no CUDA
device is present.

Status mapping mirrors the reference's error behaviour (ValueError for bad
arguments, rmpnav/_kernels/__init__.py:45-48; Cython buffer checks):
RMPB_ERR_INVALID -> ValueError, RMPB_ERR_NOMEM -> MemoryError, everything
else -> RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RMPB_LIBRARY") or os.path.join(HERE, "librmpb.so")

RMPB_OK = 0
RMPB_ERR_INVALID = -1
RMPB_ERR_CUDA = -2
RMPB_ERR_NOMEM = -3
RMPB_ERR_UNSUPPORTED = -4

RMPB_F32, RMPB_F64 = 0, 1
STORE_AUTO, STORE_F32, STORE_F64 = 0, 1, 2
LAYOUT_LINEAR, LAYOUT_QUAD, LAYOUT_BRICK, LAYOUT_PAIR64, LAYOUT_AUTO = 0, 1, 2, 4, -1
ORDER_IDENTITY, ORDER_MORTON = 0, 1
MODE_EXACT, MODE_FAST = 0, 1

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_d = ctypes.c_double
_i = ctypes.c_int

# name -> (restype, argtypes); every pointer is passed as c_void_p.
_SIGS = {
    "rmpb_last_error": (ctypes.c_char_p, []),
    "rmpb_api_version": (_i, []),
    "rmpb_device_count": (_i, [_vp]),
    "rmpb_launch_count": (ctypes.c_uint64, []),
    "rmpb_set_option": (_i, [ctypes.c_char_p, _i64]),
    "rmpb_grid_create": (_i, [_vp, _i, _i64, _i64, _i64, _d, _d, _d, _d, _i, _i, _i, _vp]),
    "rmpb_grid_create_device": (_i, [_vp, _i, _i64, _i64, _i64, _d, _d, _d, _d, _i, _i, _i, _vp]),
    "rmpb_grid_create_brick": (_i, [_vp, _i, _i64, _i64, _i64, _d, _d, _d, _d, _d, _i, _i, _vp]),
    "rmpb_grid_update": (_i, [_vp, _vp, _i]),
    "rmpb_grid_update_region": (_i, [_vp, _vp, _i, _i64, _i64, _i64, _i64, _i64, _i64]),
    "rmpb_grid_info": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "rmpb_div2_exact": (_i, [_d, _vp]),
    "rmpb_grid_destroy": (_i, [_vp]),
    "rmpb_bundle_create": (_i, [_vp, _i64, _i, _i, _vp]),
    "rmpb_bundle_halton": (_i, [_i64, _i, _i, _vp]),
    "rmpb_bundle_lattice": (_i, [_i64, _i64, _d, _i, _i, _vp]),
    "rmpb_bundle_size": (_i64, [_vp]),
    "rmpb_bundle_directions": (_i, [_vp, _vp]),
    "rmpb_bundle_destroy": (_i, [_vp]),
    "rmpb_ray_policy": (_i, [_vp, _vp, _vp, _vp, _vp, _d, _d, _d, _vp, _vp, _vp, _vp, _vp, _vp]),
    "rmpb_ray_policy_batch": (_i, [_vp, _vp, _vp, _vp, _i64, _vp, _d, _d, _d, _vp, _vp, _vp]),
    "rmpb_ray_policy_batch_device": (_i, [_vp, _vp, _vp, _vp, _i64, _vp, _d, _d, _d, _vp, _vp,
                                          _vp, _vp]),
    "rmpb_ray_policy_batch_device_mode": (_i, [_vp, _vp, _vp, _vp, _i64, _vp, _d, _d, _d, _i,
                                               _vp, _vp, _vp, _vp]),
    "rmpb_ray_policy_range_device": (_i, [_vp, _vp, _vp, _vp, _i64, _i64, _vp, _d, _d, _d, _vp,
                                          _vp]),
    "rmpb_fold_resolve_device": (_i, [_vp, _i64, _vp, _vp, _vp]),
    "rmpb_server_start": (_i, [_vp, _vp, _vp, _d, _d, _d, _d, _vp]),
    "rmpb_server_eval": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "rmpb_server_stop": (_i, [_vp]),
    "rmpb_peer_create": (_i, [_i, _i, _i, _vp, _vp]),
    "rmpb_peer_open_ipc": (_i, [_vp, _i, _vp]),
    "rmpb_peer_attach": (_i, [_vp, _i, _vp]),
    "rmpb_peer_error": (_i, [_vp, _vp]),
    "rmpb_peer_destroy": (_i, [_vp]),
    "rmpb_ray_policy_range_exchange": (_i, [_vp, _vp, _vp, _vp, _i64, _i64, _vp, _d, _d, _d, _vp,
                                            ctypes.c_uint64, _i, _vp, _vp, _vp]),
    "rmpb_lidar_policy": (_i, [_vp, _vp, _vp, _vp, _i64, _vp, _vp, _d, _vp, _vp, _vp]),
    "rmpb_lidar_policy_bundle": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _d, _vp, _vp, _vp]),
    "rmpb_lidar_policy_batch_device": (_i, [_vp, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _d, _vp,
                                            _vp, _vp]),
    "rmpb_lidar_points": (_i, [_vp, _vp, _i64, _vp, _vp, _d, _vp, _vp, _vp]),
    "rmpb_lidar_points_batch_device": (_i, [_vp, _vp, _i64, _i64, _vp, _vp, _d, _vp, _vp, _vp]),
    "rmpb_lidar_policy_batch_device_mode": (_i, [_vp, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _d,
                                                 _vp, _vp, _vp, _i]),
    "rmpb_lidar_points_batch_device_mode": (_i, [_vp, _vp, _i64, _i64, _vp, _vp, _d, _vp, _vp,
                                                 _vp, _i]),
    "rmpb_grid_trace": (_i, [_vp, _vp, _i64, _vp, _d, _d, _d, _vp, _vp, _vp, _vp]),
    "rmpb_policy_reduce": (_i, [_vp, _vp, _i64, _vp, _vp, _d, _vp, _vp]),
    "rmpb_pinv_psd": (_i, [_vp, _i64, _vp, _vp]),
    "rmpb_pinv_psd_rcond": (_i, [_vp, _i64, _d, _vp, _vp]),
    "rmpb_scene_create": (_i, [_vp, _vp, _vp, _vp, _vp, _i64, _d, _i, _vp]),
    "rmpb_scene_destroy": (_i, [_vp]),
    "rmpb_scene_distance": (_i, [_vp, _vp, _i64, _d, _vp, _vp]),
    "rmpb_scene_trace": (_i, [_vp, _vp, _vp, _i64, _d, _d, _d, _d, _vp, _vp]),
    "rmpb_bake": (_i, [_vp, _d, _d, _d, _d, _i64, _i64, _i64, _vp, _vp]),
    "rmpb_bake_grid": (_i, [_vp, _d, _d, _d, _d, _i64, _i64, _i64, _i, _i, _i, _vp]),
    "rmpb_bake_grid_tsdf": (_i, [_vp, _d, _d, _d, _d, _i64, _i64, _i64, _d, _i, _i, _i, _vp]),
    "rmpb_grid_values": (_i, [_vp, _vp]),
    "rmpb_esdf_sample": (_i, [_vp, _vp, _i64, _vp, _vp, _vp, _vp]),
    "rmpb_l2_probe": (_i, [_vp, _i64, _i, _i, _vp, _vp]),
    "rmpb_rollout_create": (_i, [_vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _i64, _vp]),
    "rmpb_rollout_run": (_i, [_vp, _i64, _vp, _vp]),
    "rmpb_rollout_result": (_i, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "rmpb_rollout_trajectory": (_i, [_vp, _vp]),
    "rmpb_rollout_destroy": (_i, [_vp]),
    "rmpb_occupancy_create": (_i, [_vp, _vp]),
    "rmpb_occupancy_destroy": (_i, [_vp]),
    "rmpb_occupancy_bits": (_i, [_vp, _vp]),
    "rmpb_dda_trace": (_i, [_vp, _vp, _i64, _vp, _d, _vp, _vp, _vp, _vp]),
    "rmpb_ray_policy_dda_batch_device": (_i, [_vp, _vp, _vp, _vp, _i64, _vp, _d, _vp, _vp, _vp]),
}

EXPORTED = tuple(_SIGS)

_lock = threading.Lock()
_lib = None


def load(path: str | None = None):
    """Load librmpb.so (once).  Raises ImportError when it is not built."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise ImportError(
                f"librmpb.so not found at {p}: build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` or "
                "`make -C paper_2301_08068_b200/csrc` (there is no CPU fallback)")
        lib = ctypes.CDLL(p)
        # experiment builds (RMPB_LIBRARY) may predate newer entry points
        lenient = bool(os.environ.get("RMPB_LIBRARY"))
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name, None) if lenient else getattr(lib, name)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        if lib.rmpb_api_version() != 1:
            raise ImportError("librmpb API version mismatch")
        if path is None:
            _lib = lib
        return lib


def last_error() -> str:
    msg = load().rmpb_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str = "") -> None:
    if status == RMPB_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if status == RMPB_ERR_INVALID:
        raise ValueError(msg)
    if status == RMPB_ERR_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"librmpb error {status}: {msg}")


def call(name: str, *args):
    check(getattr(load(), name)(*args), name)


def device_count() -> int:
    n = ctypes.c_int(0)
    st = load().rmpb_device_count(ctypes.byref(n))
    if st != RMPB_OK:
        return 0
    return int(n.value)


def launch_count() -> int:
    return int(load().rmpb_launch_count())


def set_option(name: str, value: int) -> None:
    call("rmpb_set_option", name.encode(), int(value))
