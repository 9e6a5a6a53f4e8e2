"""Device-resident entry points for callers whose tensors already live on the
GPU (the "PyTorch extension" side of the north star).  PyTorch is only the
plumbing here: memory, the current stream, ``torch.distributed``; all
compute is librmpb's sm_100a kernels, called through the C ABI with raw
device pointers on ``torch.cuda.current_stream()``.

* ``RayPolicyEngine`` -- one map + one bundle + params; ``evaluate(x, v)``
  takes P x 3 f64 CUDA tensors and returns (slots P x 13, accels P x 3) CUDA
  tensors asynchronously (K3, config C4).  ``partial(x, v, begin, end)``
  returns the 13-slot of a ray range (config C5 ray split) and
  ``resolve(slots)`` folds slots in fixed order and solves on device.
* ``lidar_policy_batch_device`` / ``lidar_points_batch_device`` -- many scans
  per launch (K2).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib as L
from ._kernels import b200
from .rays import policy_range


def _torch():
    import torch

    return torch


def _stream_ptr(stream=None) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _check_tensor(t, shape_tail, dtype_name, name, rows=None, device=None, min_numel=None):
    """Validate a tensor handed to librmpb as a raw pointer: CUDA, dtype,
    contiguous, trailing shape, leading dimension ``rows``, same device as
    ``device``, at least ``min_numel`` elements.  A mismatch would be an
    out-of-bounds device access (a poisoned CUDA context), so it raises
    ValueError here instead."""
    torch = _torch()
    want = getattr(torch, dtype_name)
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != want:
        raise ValueError(f"{name} must be {dtype_name}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if shape_tail is not None and tuple(t.shape[1:]) != tuple(shape_tail):
        raise ValueError(f"{name} must have shape (P, {', '.join(map(str, shape_tail))})")
    if rows is not None and (t.dim() == 0 or t.shape[0] != rows):
        raise ValueError(f"{name} must have {rows} rows, got shape {tuple(t.shape)}")
    if device is not None and t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device}")
    if min_numel is not None and t.numel() < min_numel:
        raise ValueError(f"{name} needs at least {min_numel} elements, got {t.numel()}")


def _check_out(t, shape, name, device):
    torch = _torch()
    _check_tensor(t, shape[1:], "float64", name, rows=shape[0], device=device)
    return t


class RayPolicyEngine:
    """Fused map-based policy evaluation with device-resident inputs."""

    def __init__(self, grid, bundle, params, max_range: float = 20.0, device: int | None = None,
                 eps: float | None = None, step_scale: float = 0.9, mode: str = "exact",
                 policy_only: bool = False):
        """``mode="exact"`` (default) is bit-identical to the reference;
        ``mode="fast"`` marches in fp32 (opt-in, NOT reference-exact).
        ``policy_only=True`` stops rays at the activation radius
        (params[5]; ``rays.policy_range``): the same policy sums, slot[12]
        then counts hits within the radius only."""
        if mode not in ("exact", "fast"):
            raise ValueError("mode must be 'exact' or 'fast'")
        self.mode = L.MODE_FAST if mode == "fast" else L.MODE_EXACT
        dev = b200.get_device() if device is None else int(device)
        if isinstance(grid, b200.DeviceGrid):
            self.grid = grid
        else:  # EsdfGrid
            prev = b200.get_device()
            b200._device = dev
            try:
                self.grid = b200.DeviceGrid(grid.values, grid.origin, grid.resolution, device=dev)
            finally:
                b200._device = prev
        if isinstance(bundle, b200.DeviceBundle):
            self.bundle = bundle
        else:
            dirs = getattr(bundle, "directions", bundle)
            self.bundle = b200.DeviceBundle(dirs, device=dev)
        self.device = dev
        self.params = np.ascontiguousarray(np.asarray(params, dtype=np.float64).reshape(7))
        self.max_range = float(max_range)
        self.policy_only = bool(policy_only)
        if self.policy_only:
            self.max_range = policy_range(self.max_range, self.params[5])
        self.eps = 0.5 * self.grid.res if eps is None else float(eps)
        self.step_scale = float(step_scale)
        self.n_rays = self.bundle.n

    def evaluate(self, x, v, out_slot=None, out_accel=None, step_counter=None, stream=None):
        torch = _torch()
        _check_tensor(x, (3,), "float64", "x")
        P = x.shape[0]
        _check_tensor(v, (3,), "float64", "v", rows=P, device=x.device)
        if out_slot is None:
            out_slot = torch.empty((P, 13), dtype=torch.float64, device=x.device)
        _check_out(out_slot, (P, 13), "out_slot", x.device)
        if out_accel is None:
            out_accel = torch.empty((P, 3), dtype=torch.float64, device=x.device)
        _check_out(out_accel, (P, 3), "out_accel", x.device)
        if step_counter is not None:
            _check_tensor(step_counter, None, "int64", "step_counter", device=x.device,
                          min_numel=1)
        cnt = 0 if step_counter is None else step_counter.data_ptr()
        L.call("rmpb_ray_policy_batch_device_mode", self.grid.handle, self.bundle.handle,
               x.data_ptr(), v.data_ptr(), P, self.params.ctypes.data, self.max_range, self.eps,
               self.step_scale, self.mode, out_slot.data_ptr(), out_accel.data_ptr(),
               cnt or None, _stream_ptr(stream))
        return out_slot, out_accel

    def partial(self, x, v, ray_begin: int, ray_end: int, out_slot=None, stream=None):
        """13-slot of stored rays [ray_begin, ray_end) for one pose (no pinv)."""
        torch = _torch()
        _check_tensor(x, None, "float64", "x", min_numel=3)
        _check_tensor(v, None, "float64", "v", device=x.device, min_numel=3)
        if out_slot is None:
            out_slot = torch.empty(13, dtype=torch.float64, device=x.device)
        _check_tensor(out_slot, None, "float64", "out_slot", device=x.device, min_numel=13)
        L.call("rmpb_ray_policy_range_device", self.grid.handle, self.bundle.handle, x.data_ptr(),
               v.data_ptr(), int(ray_begin), int(ray_end), self.params.ctypes.data,
               self.max_range, self.eps, self.step_scale, out_slot.data_ptr(),
               _stream_ptr(stream))
        return out_slot

    @staticmethod
    def resolve(slots, stream=None):
        """Fixed-order pairwise fold of (n, 13) slots + pinv, on device."""
        torch = _torch()
        _check_tensor(slots, (13,), "float64", "slots")
        if slots.shape[0] < 1:
            raise ValueError("resolve needs at least one slot")
        out_slot = torch.empty(13, dtype=torch.float64, device=slots.device)
        out_accel = torch.empty(3, dtype=torch.float64, device=slots.device)
        L.call("rmpb_fold_resolve_device", slots.data_ptr(), slots.shape[0], out_slot.data_ptr(),
               out_accel.data_ptr(), _stream_ptr(stream))
        return out_slot, out_accel

    def exchange(self, x, v, mailbox: "PeerMailbox", epoch: int, ray_begin: int, ray_end: int,
                 mode: int = 3, out_slot=None, out_accel=None, stream=None):
        """K4 fused: this rank's rays [ray_begin, ray_end) of one pose, the
        partial slot stored into every rank's mailbox over peer memory, the
        wait, the fixed-order fold and the solve -- one launch.  Returns
        (slot13, accel3) device tensors, identical on every rank."""
        torch = _torch()
        _check_tensor(x, None, "float64", "x", min_numel=3)
        _check_tensor(v, None, "float64", "v", device=x.device, min_numel=3)
        if out_slot is None:
            out_slot = torch.empty(13, dtype=torch.float64, device=x.device)
        if out_accel is None:
            out_accel = torch.empty(3, dtype=torch.float64, device=x.device)
        _check_tensor(out_slot, None, "float64", "out_slot", device=x.device, min_numel=13)
        _check_tensor(out_accel, None, "float64", "out_accel", device=x.device, min_numel=3)
        L.call("rmpb_ray_policy_range_exchange", self.grid.handle, self.bundle.handle, x.data_ptr(),
               v.data_ptr(), int(ray_begin), int(ray_end), self.params.ctypes.data,
               self.max_range, self.eps, self.step_scale, mailbox.handle, int(epoch), int(mode),
               out_slot.data_ptr(), out_accel.data_ptr(), _stream_ptr(stream))
        return out_slot, out_accel


EX_POST, EX_WAIT = 1, 2


class PeerMailbox:
    """This rank's mailbox for the fused ray-split exchange (K4, config C5):
    [2][world] epoch flags + [2][world][16] slot doubles in device memory.
    ``ipc_handle`` (64 bytes) is what the other ranks open; ``attach`` links
    a same-process mailbox (one process driving several GPUs, or tests)."""

    def __init__(self, world: int, rank: int, device: int | None = None):
        self.world, self.rank = int(world), int(rank)
        self.device = b200.get_device() if device is None else int(device)
        buf = ctypes.create_string_buffer(64)
        h = ctypes.c_void_p()
        L.call("rmpb_peer_create", self.world, self.rank, self.device, buf, ctypes.byref(h))
        self.handle = h
        self.ipc_handle = buf.raw

    def open(self, handles) -> None:
        """Open every other rank's mailbox from its IPC handle (rank order)."""
        if len(handles) != self.world:
            raise ValueError(f"{len(handles)} handles for world {self.world}")
        for r, hb in enumerate(handles):
            if r != self.rank:
                L.call("rmpb_peer_open_ipc", self.handle, r, bytes(hb))

    def attach(self, other: "PeerMailbox") -> None:
        L.call("rmpb_peer_attach", self.handle, other.rank, other.handle)

    def timed_out(self) -> bool:
        e = ctypes.c_int(0)
        L.call("rmpb_peer_error", self.handle, ctypes.byref(e))
        return bool(e.value)

    def close(self) -> None:
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            L.load().rmpb_peer_destroy(h)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DdaPolicyEngine:
    """K5: fused Amanatides-Woo DDA over occupancy + per-ray policy +
    reduction for P poses (device tensors).  A different traversal from the
    reference's sphere trace: its results are not reference-parity results."""

    def __init__(self, grid, bundle, params, max_range: float = 20.0, device: int | None = None):
        base = RayPolicyEngine(grid, bundle, params, max_range, device=device)
        self.grid, self.bundle, self.params = base.grid, base.bundle, base.params
        self.max_range = float(max_range)
        self.occ = b200.DeviceOccupancy(self.grid)

    def evaluate(self, x, v, out_slot=None, out_accel=None, stream=None):
        torch = _torch()
        _check_tensor(x, (3,), "float64", "x")
        P = x.shape[0]
        _check_tensor(v, (3,), "float64", "v", rows=P, device=x.device)
        if out_slot is None:
            out_slot = torch.empty((P, 13), dtype=torch.float64, device=x.device)
        if out_accel is None:
            out_accel = torch.empty((P, 3), dtype=torch.float64, device=x.device)
        _check_out(out_slot, (P, 13), "out_slot", x.device)
        _check_out(out_accel, (P, 3), "out_accel", x.device)
        L.call("rmpb_ray_policy_dda_batch_device", self.occ.handle, self.bundle.handle,
               x.data_ptr(), v.data_ptr(), P, self.params.ctypes.data, self.max_range,
               out_slot.data_ptr(), out_accel.data_ptr(), _stream_ptr(stream))
        return out_slot, out_accel


def _lidar_mode(mode):
    if mode not in ("exact", "fast"):
        raise ValueError("mode must be 'exact' or 'fast'")
    return L.MODE_FAST if mode == "fast" else L.MODE_EXACT


def lidar_policy_batch_device(dirs, R, ranges, valid, v, params, min_range=0.3, stream=None,
                              mode: str = "exact"):
    """S scans sharing the lattice ``dirs`` (n x 3 f64, CUDA): R (S x 9 or
    None), ranges (S x n f64), valid (S x n uint8 / bool or None), v (S x 3).
    Returns (slots S x 13, accels S x 3) CUDA tensors.  ``mode="fast"``
    (opt-in, NOT reference-exact): the per-beam policy math in fp32, the
    same contributing beams, sums within ~1e-7 relative."""
    m = _lidar_mode(mode)
    torch = _torch()
    if not isinstance(ranges, torch.Tensor) or ranges.dim() != 2:
        raise ValueError("ranges must be a (S, n) float64 CUDA tensor")
    S, n = ranges.shape
    dev = ranges.device
    _check_tensor(ranges, (n,), "float64", "ranges")
    _check_tensor(dirs, (3,), "float64", "dirs", rows=n, device=dev)
    _check_tensor(v, (3,), "float64", "v", rows=S, device=dev)
    if R is not None:
        if R.numel() != 9 * S:
            raise ValueError(f"R must hold {S} row-major 3x3 matrices")
        R = R.reshape(S, 9).contiguous()
        _check_tensor(R, (9,), "float64", "R", rows=S, device=dev)
    if valid is not None:
        if tuple(valid.shape) != (S, n):
            raise ValueError(f"valid must have shape ({S}, {n}), got {tuple(valid.shape)}")
        valid = valid.to(torch.uint8).contiguous()
        _check_tensor(valid, (n,), "uint8", "valid", rows=S, device=dev)
    p = np.ascontiguousarray(np.asarray(params, dtype=np.float64).reshape(7))
    slots = torch.empty((S, 13), dtype=torch.float64, device=ranges.device)
    accels = torch.empty((S, 3), dtype=torch.float64, device=ranges.device)
    L.call("rmpb_lidar_policy_batch_device_mode", dirs.data_ptr(),
           None if R is None else R.data_ptr(), ranges.data_ptr(),
           None if valid is None else valid.data_ptr(), n, S, v.data_ptr(), p.ctypes.data,
           float(min_range), slots.data_ptr(), accels.data_ptr(), _stream_ptr(stream), m)
    return slots, accels


def lidar_points_batch_device(xyz, R, v, params, min_range=0.3, stream=None,
                              mode: str = "exact"):
    """Raw points: xyz (S x n x 3 f32 CUDA), R (S x 9 or None), v (S x 3);
    ``mode`` as lidar_policy_batch_device."""
    m = _lidar_mode(mode)
    torch = _torch()
    if xyz.dtype != torch.float32 or not xyz.is_cuda or xyz.dim() != 3:
        raise ValueError("xyz must be a (S, n, 3) float32 CUDA tensor")
    xyz = xyz.contiguous()
    S, n, three = xyz.shape
    if three != 3:
        raise ValueError("xyz must have shape (S, n, 3)")
    _check_tensor(v, (3,), "float64", "v", rows=S, device=xyz.device)
    if R is not None:
        if R.numel() != 9 * S:
            raise ValueError(f"R must hold {S} row-major 3x3 matrices")
        R = R.reshape(S, 9).contiguous()
        _check_tensor(R, (9,), "float64", "R", rows=S, device=xyz.device)
    p = np.ascontiguousarray(np.asarray(params, dtype=np.float64).reshape(7))
    slots = torch.empty((S, 13), dtype=torch.float64, device=xyz.device)
    accels = torch.empty((S, 3), dtype=torch.float64, device=xyz.device)
    L.call("rmpb_lidar_points_batch_device_mode", xyz.data_ptr(), None if R is None else R.data_ptr(),
           n, S, v.data_ptr(), p.ctypes.data, float(min_range), slots.data_ptr(),
           accels.data_ptr(), _stream_ptr(stream), m)
    return slots, accels


def lidar_policy_batch_host(velocities, scans, p, min_range=0.3):
    """Host-facing wrapper: scans share one lattice; uploads, runs, returns
    (accels S x 3, metrics S x 3 x 3, n_hits S)."""
    torch = _torch()
    if not scans:
        raise ValueError("need at least one scan")
    dirs0 = scans[0].directions
    for s in scans:
        if s.directions.shape != dirs0.shape or not np.array_equal(s.directions, dirs0):
            raise ValueError("lidar_policy_batch needs scans sharing one beam lattice")
    dev = torch.device("cuda", b200.get_device())
    d = torch.from_numpy(np.ascontiguousarray(dirs0)).to(dev)
    R = torch.from_numpy(np.stack([s.orientation for s in scans]).reshape(-1, 9).copy()).to(dev)
    rg = torch.from_numpy(np.stack([s.ranges for s in scans])).to(dev)
    vl = torch.from_numpy(np.stack([s.valid for s in scans]).astype(np.uint8)).to(dev)
    v = torch.from_numpy(np.asarray(velocities, dtype=np.float64).reshape(-1, 3).copy()).to(dev)
    slots, accels = lidar_policy_batch_device(d, R, rg, vl, v, p.as_tuple(), min_range)
    slots = slots.cpu().numpy()
    return accels.cpu().numpy(), slots[:, 0:9].reshape(-1, 3, 3), slots[:, 12].astype(np.int64)
