"""Latency mode for the single-pose call (SURVEY.md §8d "latency-Hz").

``ray_policy`` (rmpnav/policies.py:182-192) called once per control tick
pays a kernel launch and a stream synchronisation per call (~10 us on the
B200 box, measured: scripts/lat_c.cu) on top of the trace.
``LatencyServer`` keeps ONE cooperative kernel resident (librmpb
``rmpb_server_*``) that takes requests from pinned, mapped host memory and
writes the slot + acceleration back there: same kernel body and ray
segmentation as ``ray_policy``, so the results are bitwise identical.

The resident kernel holds its CTAs' SM resources while it runs; it exits by
itself after ``idle_timeout_s`` (default 1 s) without a request (the next
call relaunches it) and on ``close()``.  Calls of librmpb that must
synchronise the device (freeing a workspace / map / bundle, peer setup) first
park the running servers of that device (stop + wait) instead of blocking
behind them; the next ``evaluate`` relaunches transparently.  Requests of one
server are serialised (a per-server lock).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib as L
from ._kernels import b200
from .core import Policy, RobotState
from .geometry import EsdfGrid
from .policies import GRID_STEP_SCALE, ObstacleParams, _policy_from_slot
from .rays import DEFAULT_MAX_RANGE, RayBundle, policy_range


class LatencyServer:
    def __init__(self, field: EsdfGrid, bundle: RayBundle, p: ObstacleParams,
                 max_range: float = DEFAULT_MAX_RANGE, idle_timeout_s: float = 1.0,
                 storage: int | None = None, layout: int | None = None,
                 policy_only: bool = False):
        """``storage`` / ``layout`` (librmpb STORE_* / LAYOUT_*) give the
        server its own device copy of the map in that layout; default: the
        map shared with ``ray_policy``.  ``policy_only`` as in
        ``ray_policy``: rays stop at the activation radius, same Policy."""
        if not isinstance(field, EsdfGrid):
            raise TypeError("LatencyServer needs an EsdfGrid")
        if storage is None and layout is None:
            self._grid = b200.device_grid(field.values, field.origin, field.resolution)
        else:
            self._grid = b200.DeviceGrid(field.values, field.origin, field.resolution,
                                         storage=L.STORE_AUTO if storage is None else storage,
                                         layout=L.LAYOUT_AUTO if layout is None else layout)
        self._bundle = b200.device_bundle(getattr(bundle, "directions", bundle))
        self._params = np.ascontiguousarray(np.asarray(p.as_tuple(), dtype=np.float64))
        if policy_only:
            max_range = policy_range(max_range, p.radius)
        self.max_range = float(max_range)
        h = ctypes.c_void_p()
        L.call("rmpb_server_start", self._grid.handle, self._bundle.handle,
               self._params.ctypes.data, float(max_range), 0.5 * float(field.resolution),
               GRID_STEP_SCALE, float(idle_timeout_s), ctypes.byref(h))
        self.handle = h
        self._xv = np.empty(6)
        self._xv_p = self._xv.ctypes.data
        self._out = np.empty(16)
        self._out_p = self._out.ctypes.data
        self._eval = L.load().rmpb_server_eval

    def evaluate(self, position, velocity):
        """(slot13, accel3) of one pose, as ``ray_policy_fused`` returns."""
        if self.handle is None:
            raise RuntimeError("LatencyServer is closed")
        self._xv[0:3] = position
        self._xv[3:6] = velocity
        L.check(self._eval(self.handle, self._xv_p, self._xv_p + 24, self._out_p,
                           self._out_p + 104), "rmpb_server_eval")
        out = self._out.copy()
        return out[:13], out[13:]

    def policy(self, state: RobotState) -> Policy:
        """``ray_policy(state, field, bundle, p, max_range)`` through the
        resident kernel."""
        slot, acc = self.evaluate(state.position, state.velocity)
        return _policy_from_slot(slot, acc)

    def close(self) -> None:
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            self.handle = None
            L.call("rmpb_server_stop", h)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
