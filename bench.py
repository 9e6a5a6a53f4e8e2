#!/usr/bin/env python3
"""Benchmark of the raycasting-RMP hot path (BASELINE.json ``metric``).

Workload (one "step"): config C4's shape on the C1 headline map -- P = 4096
robot poses (bench_states, seed 123) x 65536 Halton rays each, 200x200x100
node map @0.1 m (200 random boxes, f32-exact values), 10 m range, preset
``static_map`` -- evaluated as ONE fused launch (trace + per-ray policy +
reduction + 3x3 pinv per pose).  ``value`` is whole-job rays/s with inputs
resident in HBM (CUDA events around each step, L2 flushed between steps);
``hz`` is the matching 65536-ray policy-evaluation rate.  Under torchrun
each rank evaluates its own block of P poses (weak scaling, no collective on
the data path).

``e2e`` is the same metric through the public host API
(``ray_policy_batch`` with host arrays: pose upload + result download inside
the timed region).  ``latency_hz`` is the single-pose ``ray_policy`` call
rate (the paper's load -> execute -> readback window).

``--impl reference`` times the reference's own compiled CPU kernels
(oracle/_ref, built from /root/reference) on the box's host cores on the
same workload, a bounded sample of poses per step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("rays/sec and RMP evaluation rate (Hz) at 65536 rays; "
          "voxel-steps/s vs L2/HBM BW")
N_RAYS = 65536
MAX_RANGE = 10.0
PARAMS = (88.0, 1.4, 140.0, 1.2, 1e-6, 2.4, 0.2)  # static_map, kernel order
BYTES_PER_STEP = 32  # 8 corner reads x f32 storage


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            import shutil

            pre = ["stdbuf", "-oL"] if shutil.which("stdbuf") else []  # line-buffered pipe
            self.proc = subprocess.Popen(
                pre + ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_first(self, timeout=5.0):
        """Block until nvidia-smi delivered its first sample (it takes ~0.5 s
        to start; the timed region is shorter than that)."""
        t0 = time.perf_counter()
        while self.proc is not None and not self.lines and time.perf_counter() - t0 < timeout:
            time.sleep(0.02)
        self.n0 = len(self.lines)

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        n0 = getattr(self, "n0", 0)
        lines = self.lines[n0:] if len(self.lines) > n0 else self.lines
        for ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def build_world(backend_bake=None, distance=None, total_poses=4096):
    from paper_2301_08068_b200 import synth

    scene = synth.c1_scene()
    grid = synth.c1_grid(scene, bake=backend_bake)
    if distance is None:
        distance = synth.host_box_distance(scene)  # input synthesis only
    states = synth.bench_states(scene, count=total_poses, seed=123, distance=distance)
    return scene, grid, states


def ncu_summary():
    """Latest committed ncu --set full summary of the hot kernel (profiles/)."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_summary.json")))
    if not files:
        return None
    try:
        with open(files[-1]) as fh:
            d = json.load(fh)
        d["file"] = os.path.relpath(files[-1], ROOT)
        return d
    except Exception:
        return None


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


# ----------------------------------------------------------------------------
# our arm

def run_b200(args):
    import torch
    import torch.distributed as dist

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    # (RMPB_BENCH_BACKEND=gloo: a code-path check of the N > 1 flow with
    # several ranks sharing the visible GPUs -- never a measurement)
    backend = os.environ.get("RMPB_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        # communicator-init lines on stderr (the driver's rank check reads them)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    os.environ["RMPNAV_DEVICE"] = str(local)

    from paper_2301_08068_b200 import _lib, synth
    from paper_2301_08068_b200._kernels import b200
    from paper_2301_08068_b200.device import RayPolicyEngine
    from paper_2301_08068_b200.policies import ObstacleParams, ray_policy, ray_policy_batch
    from paper_2301_08068_b200.rays import sample_directions

    b200.set_device(local)
    P = args.poses
    scene, grid, states_all = build_world(total_poses=P * world)
    states = states_all[rank * P:(rank + 1) * P]
    x_h, v_h = synth.states_arrays(states)
    bundle = sample_directions(N_RAYS)  # Halton bundle generated on device
    params = ObstacleParams(88.0, 1.4, 140.0, 1.2, 2.4, 0.2)
    eng = RayPolicyEngine(grid, bundle, params.as_tuple(), MAX_RANGE, device=local)
    dev = torch.device("cuda", local)
    x = torch.from_numpy(x_h).to(dev)
    v = torch.from_numpy(v_h).to(dev)
    slots = torch.empty((P, 13), dtype=torch.float64, device=dev)
    accels = torch.empty((P, 3), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    # calibration (untimed): voxel-steps per step, for the roofline numerator
    steps_ctr = torch.zeros(1, dtype=torch.int64, device=dev)
    eng.evaluate(x, v, slots, accels, step_counter=steps_ctr)
    torch.cuda.synchronize()
    vox_steps = int(steps_ctr.item())

    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        flush.zero_()
        eng.evaluate(x, v, slots, accels)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    clocks.wait_first()
    n0 = _lib.launch_count()
    total_ms = 0.0
    for _ in range(args.steps):
        flush.zero_()  # L2 flush between timed steps (256 MiB > 126 MB L2)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eng.evaluate(x, v, slots, accels)
        e1.record(stream)
        e1.synchronize()
        total_ms += e0.elapsed_time(e1)
    torch.cuda.synchronize()
    launches = _lib.launch_count() - n0
    if world > 1:
        dist.barrier()
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    rays_per_step = P * N_RAYS * world
    value = rays_per_step / (ms_per_step * 1e-3)
    hz = P * world / (ms_per_step * 1e-3)

    # e2e: public host API, host arrays in, host results out, every step
    for _ in range(2):
        ray_policy_batch((x_h, v_h), grid, bundle, params, MAX_RANGE)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e2e_s = 0.0
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        acc_h, met_h, nh = ray_policy_batch((x_h, v_h), grid, bundle, params, MAX_RANGE)
        e2e_s += time.perf_counter() - t0
    clk = clocks.stop()  # sampled over the device-timed and the e2e steps
    t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_s = float(t.item())
    e2e_value = rays_per_step * args.steps / e2e_s

    # single-pose latency through ray_policy (paper's window), rank-local
    lat = []
    for i in range(args.latency_calls + 20):
        st = states[i % len(states)]
        t0 = time.perf_counter()
        ray_policy(st, grid, bundle, params, MAX_RANGE)
        if i >= 20:
            lat.append(time.perf_counter() - t0)
    lat_med = statistics.median(lat)
    # the same call through the resident-kernel latency server (no launch /
    # stream sync per call; bitwise the same results)
    from paper_2301_08068_b200 import LatencyServer

    lat_s = []
    with LatencyServer(grid, bundle, params, MAX_RANGE) as srv:
        for i in range(args.latency_calls + 20):
            st = states[i % len(states)]
            t0 = time.perf_counter()
            srv.policy(st)
            if i >= 20:
                lat_s.append(time.perf_counter() - t0)
    lat_srv = statistics.median(lat_s)
    breakdown = latency_breakdown(grid, bundle, params, states, eng, dev, lat_med, lat_srv)
    # policy-only evaluation (opt-in, rays stop at the activation radius:
    # the same Policy; per-ray masks / n_hits then count hits within it)
    from paper_2301_08068_b200.device import RayPolicyEngine
    from paper_2301_08068_b200.rays import policy_range

    lat_po, lat_spo = [], []
    for i in range(args.latency_calls + 20):  # (no server resident meanwhile)
        st = states[i % len(states)]
        t0 = time.perf_counter()
        ray_policy(st, grid, bundle, params, MAX_RANGE, policy_only=True)
        if i >= 20:
            lat_po.append(time.perf_counter() - t0)
    with LatencyServer(grid, bundle, params, MAX_RANGE, policy_only=True) as srv:
        for i in range(args.latency_calls + 20):
            st = states[i % len(states)]
            t0 = time.perf_counter()
            srv.policy(st)
            if i >= 20:
                lat_spo.append(time.perf_counter() - t0)
    eng_po = RayPolicyEngine(grid, bundle, params.as_tuple(), MAX_RANGE, policy_only=True)
    breakdown["policy_only"] = latency_breakdown(
        grid, bundle, params, states, eng_po, dev, statistics.median(lat_po),
        statistics.median(lat_spo), max_range=policy_range(MAX_RANGE, params.radius))

    # measured L2 read ceiling (untimed), CUDA events
    l2 = l2_peaks(dev, stream)

    # live kernel duration = step time (one k_ray_policy launch per step)
    kern_ms = ms_per_step
    peaks, peak_src = measured_peaks()
    algo_bytes = vox_steps * BYTES_PER_STEP
    achieved = algo_bytes / (kern_ms * 1e-3) / 1e9
    ncu = ncu_summary()
    traffic = args.ncu_traffic
    if traffic is None and ncu is not None:
        traffic = ncu.get("dram_bytes_per_launch")
    limiter = ("latency: each sphere-trace step is a dependent chain of ~25 fp64 ops around "
               "one L2 gather (map L2-resident); not HBM bandwidth")
    if ncu is not None:
        limiter += (f" -- ncu: issue slots {ncu.get('issue_active_pct')} %, fp64 pipe "
                    f"{ncu.get('fp64_pipe_active_pct')} %, warps active "
                    f"{ncu.get('warps_active_pct')} %")
    roof = {"bound": "hbm", "limiter": limiter,
            "fp64_pipe_active_pct": (ncu or {}).get("fp64_pipe_active_pct"),
            "issue_active_pct": (ncu or {}).get("issue_active_pct"),
            "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"],
            "unit": "GB/s", "frac": round(achieved / peaks["hbm_gbs"], 4),
            "traffic": traffic, "peak_source": peak_src,
            "traffic_source": (ncu or {}).get("file"),
            "l2_read_GBps_ncu": (ncu or {}).get("l2_read_GBps"),
            "l2_stream_peak_GBps": l2.get("stream"),
            "frac_of_l2_stream_peak": (round(achieved / l2["stream"], 4)
                                       if l2.get("stream") else None),
            "kernel": "k_ray_policy2<QuadGridF32Div2O0>",
            "algorithmic_bytes_per_launch": algo_bytes,
            "voxel_steps_per_launch": vox_steps,
            "note": "bytes = voxel-steps x 8 corners x 4 B (f32 map); map is L2-resident"}

    configs = {}
    if rank == 0 and not args.no_configs:
        configs["C3_lidar_1024_scans"] = c3_config(dev, stream, peaks["hbm_gbs"], flush,
                                                   cpu=(world == 1 and not args.no_cpu_baseline))
        configs["C2_1M_rays_10m"] = c2_config(grid, dev, stream, flush, params)
        configs["C4_policy_only"] = c4_policy_only(eng_po, x, v, slots, accels, stream, flush)
        if world == 1:
            configs["C5_1M_rays_ray_split"] = c5_config(dev, stream)

    out = None
    if rank == 0:
        cpu = None
        parity = None
        if not args.no_parity:
            parity = parity_check(grid, x_h, v_h, bundle.directions, slots.cpu().numpy(),
                                  accels.cpu().numpy())
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(grid, states, args.cpu_seconds)
        out = {
            "metric": METRIC, "value": round(value, 1), "unit": "rays/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": "C4-shape batch on the C1 headline map: "
                                   f"{P} poses/rank x {N_RAYS} Halton rays, 200x200x100 "
                                   "@0.1 m (200 boxes), max range 10 m, static_map",
                       "poses_per_rank": P, "rays_per_pose": N_RAYS, "max_range_m": MAX_RANGE,
                       "map": "C1 200x200x100 @0.1m f32-exact, QUAD layout",
                       "l2": "flushed (256 MiB write) between timed steps",
                       "parallelism": f"pose-sharded x{world}"},
            "hz": round(hz, 1),
            "voxel_steps_per_s": round(vox_steps * world / (ms_per_step * 1e-3), 1),
            "latency_hz": round(1.0 / lat_med, 1),
            "latency_us_median": round(lat_med * 1e6, 2),
            "latency_server_hz": round(1.0 / lat_srv, 1),
            "latency_server_us_median": round(lat_srv * 1e6, 2),
            "latency_breakdown": breakdown,
            "roofline": roof,
            "parity": parity,
            "configs": configs,
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_value, 1), "unit": "rays/s",
                    "h2d_bytes_per_step": int(P * 6 * 8), "d2h_bytes_per_step": int(P * 16 * 8),
                    "api": "paper_2301_08068_b200.ray_policy_batch (host arrays)"},
            "gpu_launches": int(launches),
            "clocks": clk,
        }
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return out


def latency_breakdown(grid, bundle, params, states, eng, dev, lat_py, lat_srv, n=200,
                      max_range=None):
    """Where the single-pose call's time goes (C1, 65536 rays): the public
    Python call, the bare C-ABI call (ctypes, pre-staged pointers: host
    staging + launch + kernel + readback + sync), and the kernel alone on the
    device timeline (CUDA events around a device-resident P = 1 launch)."""
    import ctypes

    import numpy as np
    import torch

    from paper_2301_08068_b200 import _lib
    from paper_2301_08068_b200._kernels import b200

    g = b200.device_grid(grid.values, grid.origin, grid.resolution)
    b = b200.device_bundle(bundle.directions)
    xv = np.empty(6)
    out = np.empty(16)
    pa = np.ascontiguousarray(np.asarray(params.as_tuple(), dtype=np.float64))
    fn = _lib.load().rmpb_ray_policy
    eps = 0.5 * grid.resolution
    mr = MAX_RANGE if max_range is None else float(max_range)
    xvp, outp, pap = xv.ctypes.data, out.ctypes.data, pa.ctypes.data
    c_us = []
    for i in range(n + 20):
        st = states[i % len(states)]
        xv[0:3] = st.position
        xv[3:6] = st.velocity
        t0 = time.perf_counter()
        rc = fn(g.handle, b.handle, xvp, xvp + 24, pap, mr, eps, 0.9, outp, outp + 104,
                None, None, None, None)
        t1 = time.perf_counter()
        if rc != 0:
            raise RuntimeError(_lib.last_error())
        if i >= 20:
            c_us.append((t1 - t0) * 1e6)
    x_all = torch.from_numpy(np.stack([s.position for s in states[:64]])).to(dev)
    v_all = torch.from_numpy(np.stack([s.velocity for s in states[:64]])).to(dev)
    k_us = []
    for i in range(n + 20):
        x1 = x_all[i % 64:i % 64 + 1]
        v1 = v_all[i % 64:i % 64 + 1]
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200000)  # GPU busy while the host enqueues: e0 -> e1 is the kernel
        e0.record()
        eng.evaluate(x1, v1)
        e1.record()
        e1.synchronize()
        if i >= 20:
            k_us.append(e0.elapsed_time(e1) * 1e3)
    # the same launch with max range ~0: the fixed part (launch, ray prep,
    # first step, CTA reduce, ticket, fold, solve); the rest is the rays' tail
    from paper_2301_08068_b200.device import RayPolicyEngine

    eng0 = RayPolicyEngine(eng.grid, eng.bundle, eng.params, 1e-6)
    k0_us = []
    for i in range(n // 2 + 20):
        x1 = x_all[i % 64:i % 64 + 1]
        v1 = v_all[i % 64:i % 64 + 1]
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200000)
        e0.record()
        eng0.evaluate(x1, v1)
        e1.record()
        e1.synchronize()
        if i >= 20:
            k0_us.append(e0.elapsed_time(e1) * 1e3)
    # the platform floor: one empty-ish kernel launch + stream sync (host clock)
    z = torch.zeros(1, device=dev)
    f_us = []
    for i in range(n + 20):
        t0 = time.perf_counter()
        z.fill_(1.0)
        torch.cuda.current_stream().synchronize()
        if i >= 20:
            f_us.append((time.perf_counter() - t0) * 1e6)
    c_med = statistics.median(c_us)
    k_med = statistics.median(k_us)
    return {"python_ray_policy_us": round(lat_py * 1e6, 2),
            "c_abi_rmpb_ray_policy_us": round(c_med, 2),
            "device_kernel_us": round(k_med, 2),
            "device_kernel_fixed_us": round(statistics.median(k0_us), 2),
            "device_kernel_ray_tail_us": round(k_med - statistics.median(k0_us), 2),
            "python_overhead_us": round(lat_py * 1e6 - c_med, 2),
            "host_launch_sync_readback_us": round(c_med - k_med, 2),
            "latency_server_us": round(lat_srv * 1e6, 2), "max_range_m": mr,
            "empty_kernel_launch_sync_us": round(statistics.median(f_us), 2),
            "note": "medians of 200 calls; device_kernel_us = CUDA events around one "
                    "device-resident P=1 launch (segments of 256 rays: the pose's longest "
                    "ray is the floor); device_kernel_fixed_us = the same launch at max "
                    "range ~0 (launch, prep, CTA reduce, ticket, fold, solve; includes the "
                    "~6 us event-timing floor of any kernel); device timeline of the parts: "
                    "profiles/README.md (scripts/lat_tl.cu)"}


def parity_check(grid, x_h, v_h, dirs, slots, accels, poses=8):
    """Checker (outside every timed region): `poses` strided poses of the
    LAST timed launch against the reference's own compiled kernels
    (oracle/_ref, the C port if absent) on the same direction array."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    P = slots.shape[0]
    idx = list(range(0, P, max(1, P // poses)))[:poses]
    kind = "reference" if O.ref_available() else "port"
    pool = O.RefPool(_cpu_threads()) if kind == "reference" else None
    n_eq, rel_s, rel_a = True, 0.0, 0.0
    try:
        for k in idx:
            if kind == "reference":
                m, w, nh, acc, _ = O.ref_ray_policy(grid.values, grid.origin, grid.resolution,
                                                    x_h[k], v_h[k], dirs, PARAMS, MAX_RANGE, pool)
                ref = np.concatenate([np.asarray(m).reshape(9), np.asarray(w).reshape(3), [nh]])
            else:
                ref, acc, _ = O.ray_policy(grid.values, grid.origin, grid.resolution, x_h[k],
                                           v_h[k], dirs, PARAMS, MAX_RANGE, workers=_cpu_threads())
            n_eq &= bool(slots[k][12] == ref[12])
            sc = max(1e-300, float(np.abs(ref[:12]).max()))
            rel_s = max(rel_s, float(np.abs(slots[k][:12] - ref[:12]).max()) / sc)
            sa = max(1e-300, float(np.abs(acc).max()))
            rel_a = max(rel_a, float(np.abs(accels[k] - acc).max()) / sa)
    finally:
        if pool is not None:
            pool.close()
    return {"poses": len(idx), "pose_indices": idx, "checker": kind, "n_hits_equal": n_eq,
            "max_rel_sums": rel_s, "max_rel_accel": rel_a, "tolerance_sums": 1e-5,
            "pass": bool(n_eq and rel_s <= 1e-5 and rel_a <= 1e-5)}


def _ev_ms(fn, stream, flush, reps=5):
    import torch

    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts), statistics.median(ts)


def c3_config(dev, stream, hbm_peak, flush, cpu=True, S=1024):
    """Config C3 (LiDAR-direct, 128x1024 OS0 scans): 1024 scans per launch,
    device resident (K2 k_lidar_warp), HBM fraction of its 9 B/beam stream,
    and the single-scan public call; the reference's CPU lidar_policy on the
    box's cores beside it."""
    import torch

    from paper_2301_08068_b200 import synth
    from paper_2301_08068_b200.device import lidar_policy_batch_device
    from paper_2301_08068_b200.policies import lidar_policy, preset
    from paper_2301_08068_b200.rays import scan_pattern

    scene = synth.c1_scene()
    states = synth.bench_states(scene, count=10, seed=123, distance=synth.host_box_distance(scene))
    scans = synth.lidar_scans(scene, states, 128, 1024, 20.0)
    n = 128 * 1024
    lidar = preset("lidar").obstacle
    lp = lidar.as_tuple()
    dirs = torch.from_numpy(np.ascontiguousarray(scan_pattern(128, 1024)).copy()).to(dev)
    rg = torch.from_numpy(np.stack([scans[i % 10].ranges for i in range(S)])).to(dev)
    vl = torch.from_numpy(np.stack([scans[i % 10].valid for i in range(S)]).astype(np.uint8)).to(dev)
    R = torch.from_numpy(np.stack([scans[i % 10].orientation for i in range(S)])
                         .reshape(S, 9).copy()).to(dev)
    v = torch.from_numpy(np.stack([states[i % 10].velocity for i in range(S)])).to(dev)
    best, med = _ev_ms(lambda: lidar_policy_batch_device(dirs, R, rg, vl, v, lp, 0.3), stream,
                       flush)
    gbs = S * n * 9 / (best * 1e-3) / 1e9
    lat = []
    for i in range(120):
        t0 = time.perf_counter()
        lidar_policy(states[i % 10].velocity, scans[i % 10], lidar)
        if i >= 20:
            lat.append(time.perf_counter() - t0)
    rec = {"scans_per_launch": S, "beams_per_scan": n, "ms_per_launch_best": round(best, 4),
           "ms_per_launch_median": round(med, 4), "scans_per_s": round(S / (best * 1e-3), 1),
           "beams_per_s": round(S * n / (best * 1e-3), 1),
           "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm_peak,
                        "unit": "GB/s", "frac": round(gbs / hbm_peak, 4),
                        "bytes_per_beam": 9, "kernel": "k_lidar_warp<LatticeSrc>"},
           "single_scan_public_api_us_median": round(statistics.median(lat) * 1e6, 1)}
    # opt-in fast mode (fp32 per-beam policy math, the same contributing
    # beams; sums within ~1e-7 of the exact mode): not the headline
    bf, _mf = _ev_ms(lambda: lidar_policy_batch_device(dirs, R, rg, vl, v, lp, 0.3, mode="fast"),
                     stream, flush)
    s_ex, _ = lidar_policy_batch_device(dirs, R, rg, vl, v, lp, 0.3)
    s_fa, _ = lidar_policy_batch_device(dirs, R, rg, vl, v, lp, 0.3, mode="fast")
    s_ex, s_fa = s_ex.cpu().numpy(), s_fa.cpu().numpy()
    rec["fast_mode"] = {"ms_per_launch_best": round(bf, 4),
                        "hbm_frac": round(S * n * 9 / (bf * 1e-3) / 1e9 / hbm_peak, 4),
                        "max_rel_sums_vs_exact": float(np.abs(s_fa[:, :12] - s_ex[:, :12]).max()
                                                       / np.abs(s_ex[:, :12]).max()),
                        "n_hits_equal": bool(np.array_equal(s_fa[:, 12], s_ex[:, 12]))}
    if cpu:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O

        if O.ref_available():
            wd = [np.ascontiguousarray(s.world_directions()) for s in scans]
            out = {}
            for w in (_cpu_threads(), 1):
                pool = O.RefPool(w)
                ts = []
                for i in range(30):
                    t0 = time.perf_counter()
                    O.ref_lidar_policy(wd[i % 10], scans[i % 10].ranges, scans[i % 10].valid,
                                       states[i % 10].velocity, lp, 0.3, pool)
                    ts.append(time.perf_counter() - t0)
                pool.close()
                out[f"threads_{w}"] = {"ms_median": round(statistics.median(ts[5:]) * 1e3, 3),
                                       "ms_best": round(min(ts) * 1e3, 3),
                                       "scans_per_s": round(1.0 / statistics.median(ts[5:]), 1)}
            rec["cpu_reference"] = {**out, "kind": "reference",
                                    "sample": "30 scans per thread count (world directions "
                                              "precomputed, as rmpnav's lidar_policy passes them)"}
    return rec


def c4_policy_only(eng_po, x, v, slots, accels, stream, flush):
    """The bench step (same poses, bundle, map) through the policy-only
    engine: rays stop at the activation radius (rays.policy_range); the
    slots' policy sums are checked against the timed full-range step."""
    import numpy as np

    best, med = _ev_ms(lambda: eng_po.evaluate(x, v), stream, flush, reps=5)
    s_po, a_po = eng_po.evaluate(x, v)
    s_full = slots.cpu().numpy()
    s_po = s_po.cpu().numpy()
    scale = float(np.abs(s_full[:, :12]).max())
    P = x.shape[0]
    return {"max_range_m": eng_po.max_range, "ms_per_step_best": round(best, 3),
            "ms_per_step_median": round(med, 3),
            "evaluations_per_s": round(P / (best * 1e-3), 1),
            "max_rel_sum_vs_full_range": float(np.abs(s_po[:, :12] - s_full[:, :12]).max()) / scale,
            "n_hits_within_radius": int(s_po[:, 12].sum()), "n_hits_full": int(s_full[:, 12].sum()),
            "note": "opt-in policy_only=True: same Policy (hits at d >= radius have weight 0); "
                    "not the headline (the headline traces every ray to max range)"}


def c2_config(grid, dev, stream, flush, params, P=64):
    """Config C2 subset: 1 M Halton rays @ 10 m on the C1 map, P poses per
    launch (device resident)."""
    import torch

    from paper_2301_08068_b200 import synth
    from paper_2301_08068_b200.device import RayPolicyEngine
    from paper_2301_08068_b200.rays import sample_directions

    n = 1 << 20
    scene = synth.c1_scene()
    states = synth.bench_states(scene, count=P, seed=7, distance=synth.host_box_distance(scene))
    x_h, v_h = synth.states_arrays(states)
    eng = RayPolicyEngine(grid, sample_directions(n), params.as_tuple(), MAX_RANGE)
    x = torch.from_numpy(x_h).to(dev)
    v = torch.from_numpy(v_h).to(dev)
    best, med = _ev_ms(lambda: eng.evaluate(x, v), stream, flush, reps=3)
    return {"poses_per_launch": P, "rays_per_pose": n, "max_range_m": MAX_RANGE,
            "ms_per_launch_best": round(best, 3), "ms_per_launch_median": round(med, 3),
            "rays_per_s": round(P * n / (best * 1e-3), 1),
            "evaluations_per_s": round(P / (best * 1e-3), 1)}


def c5_config(dev, stream, steps=20):
    """Config C5 at N = 1 inside the default line: one 1 M-ray pose on the
    1000x1000x200 block-hashed TSDF through the K4 exchange kernel (world-1
    mailbox; `--workload c5` under torchrun splits it over GPUs)."""
    import torch

    from paper_2301_08068_b200 import synth
    from paper_2301_08068_b200._kernels import b200
    from paper_2301_08068_b200.device import PeerMailbox, RayPolicyEngine

    scene = synth.c5_scene()
    _dense, brick, info = synth.c5_grids(scene)
    del _dense
    states = synth.bench_states(scene, count=8, seed=123, distance=synth.host_box_distance(scene))
    n = 1 << 20
    eng = RayPolicyEngine(brick, b200.DeviceBundle(halton_n=n), PARAMS, MAX_RANGE)
    xs = [torch.tensor(s.position, dtype=torch.float64, device=dev) for s in states]
    vs = [torch.tensor(s.velocity, dtype=torch.float64, device=dev) for s in states]
    mb = PeerMailbox(1, 0)
    mb.open([mb.ipc_handle])
    ep = [0]

    def one(k):
        ep[0] += 1
        eng.exchange(xs[k % 8], vs[k % 8], mb, ep[0], 0, n)
    for k in range(5):
        one(k)
    torch.cuda.synchronize()
    ts = []
    for k in range(steps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        one(k)
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    # the same poses through a policy-only engine (rays stop at the 2.4 m
    # activation radius; the same sums -- the partial RMP sums are what the
    # ray split exchanges)
    eng_po = RayPolicyEngine(brick, eng.bundle, PARAMS, MAX_RANGE, policy_only=True)
    ts_po = []
    for k in range(steps):
        ep[0] += 1
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eng_po.exchange(xs[k % 8], vs[k % 8], mb, ep[0], 0, n)
        e1.record(stream)
        e1.synchronize()
        ts_po.append(e0.elapsed_time(e1))
    mb.close()
    ms = statistics.median(ts)
    return {"rays_per_pose": n,
            "map": "1000x1000x200 @0.05 m TSDF (tau 0.2 m), BRICK 8^3 f32 (apron-QUAD records)",
            "policy_only_ms_per_pose_median": round(statistics.median(ts_po), 4),
            "bricks_allocated": info["bricks_allocated"], "brick_bytes": info["brick_bytes"],
            "ms_per_pose_median": round(ms, 4), "ms_per_pose_best": round(min(ts), 4),
            "rays_per_s": round(n / (ms * 1e-3), 1), "hz": round(1e3 / ms, 1),
            "kernel": "k_ray_policy2<BrickQuadF32*, EX> (K4 exchange epilogue, world 1; the "
                      "kernel the batch path selects for 512-ray segments)"}


def run_c5(args):
    """`--workload c5`: config C5 -- ONE pose of 1 M Halton rays on the
    1000x1000x200 @0.05 m block-hashed TSDF (tau 0.2 m), its rays split over
    the WORLD_SIZE ranks (strong scaling: the work per step is fixed).  Each
    step is one K4 launch per rank (FusedRaySplit: trace the rank's ray range
    -> post the partial 13-slot into every rank's mailbox over peer memory ->
    wait -> fixed-order fold -> pinv, rmpnav/_kernels/_pool.py:61-72); the
    all_gather path (partial kernel, NCCL all_gather of the 13-slots, fold
    kernel) is timed alongside.  Device time, max over ranks."""
    import torch
    import torch.distributed as dist

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    os.environ["RMPNAV_DEVICE"] = str(local)
    from paper_2301_08068_b200 import _lib, synth
    from paper_2301_08068_b200._kernels import b200
    from paper_2301_08068_b200.device import PeerMailbox, RayPolicyEngine
    from paper_2301_08068_b200.parallel import FusedRaySplit, balanced_range, split_ray_policy

    b200.set_device(local)
    dev = torch.device("cuda", local)
    t0 = time.perf_counter()
    scene = synth.c5_scene()
    _dense, brick, info = synth.c5_grids(scene)
    del _dense
    build_s = time.perf_counter() - t0
    states = synth.bench_states(scene, count=8, seed=123, distance=synth.host_box_distance(scene))
    n = 1 << 20
    bundle = b200.DeviceBundle(halton_n=n)
    eng = RayPolicyEngine(brick, bundle, PARAMS, MAX_RANGE, device=local)
    xs = [torch.tensor(s.position, dtype=torch.float64, device=dev) for s in states]
    vs = [torch.tensor(s.velocity, dtype=torch.float64, device=dev) for s in states]
    if world > 1:
        split = FusedRaySplit(eng)
    else:
        mb = PeerMailbox(1, 0, local)
        mb.open([mb.ipc_handle])
        ep = [0]
        b0, e0 = balanced_range(n, 1, 0)

        def split(x, v):
            ep[0] += 1
            return eng.exchange(x, v, mb, ep[0], b0, e0)
    stream = torch.cuda.current_stream()

    def timed(fn, steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ms = 0.0
        for k in range(steps):
            e0_ = torch.cuda.Event(enable_timing=True)
            e1_ = torch.cuda.Event(enable_timing=True)
            e0_.record(stream)
            fn(xs[k % 8], vs[k % 8])
            e1_.record(stream)
            e1_.synchronize()
            ms += e0_.elapsed_time(e1_)
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()) / steps

    for k in range(args.warmup):
        split(xs[k % 8], vs[k % 8])
    n0 = _lib.launch_count()
    ms_fused = timed(split, args.steps)
    launches = _lib.launch_count() - n0
    res_f = split(xs[0], vs[0])
    if world > 1:
        gather = lambda x, v: split_ray_policy(eng, x, v)  # noqa: E731
    else:
        gather = lambda x, v: eng.resolve(eng.partial(x, v, 0, n).view(1, 13))  # noqa: E731
    for k in range(args.warmup):
        gather(xs[k % 8], vs[k % 8])
    ms_gather = timed(gather, args.steps)
    res_g = gather(xs[0], vs[0])
    torch.cuda.synchronize()
    sf, sg = res_f[0].view(-1).cpu().numpy(), res_g[0].view(-1).cpu().numpy()
    fused_rel = float(np.abs(sf[:12] - sg[:12]).max() / max(1e-300, np.abs(sg[:12]).max()))
    same_hits = bool(sf[12] == sg[12])
    out = None
    if rank == 0:
        out = {"metric": METRIC, "value": round(n / (ms_fused * 1e-3), 1), "unit": "rays/s",
               "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": round(ms_fused, 4), "higher_is_better": True, "scaling": "strong",
               "vs_baseline": None, "dtype": "f64", "data": "synthetic",
               "config": {"workload": "C5: one pose x 1 M Halton rays, 1000x1000x200 @0.05 m "
                                      "block-hashed TSDF (tau 0.2 m), max range 10 m, rays "
                                      f"split over {world} GPU(s)",
                          "rays_per_pose": n, "map": "BRICK 8^3, f32 apron-QUAD records", **info,
                          "build_s": round(build_s, 2),
                          "parallelism": f"ray-split x{world} (K4 peer-mailbox exchange)"},
               "hz": round(1e3 / ms_fused, 1),
               "allgather_baseline": {"ms_per_step": round(ms_gather, 4),
                                      "hz": round(1e3 / ms_gather, 1),
                                      "path": "partial kernel + NCCL all_gather + fold kernel"
                                              if world > 1 else "partial kernel + fold kernel"},
               "fused_vs_allgather": {"n_hits_equal": same_hits, "max_rel_sums": fused_rel,
                                      "note": "different ray segmentations per kernel: sums "
                                              "agree to the last bits, not bitwise"},
               "gpu_launches": int(launches)}
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return out


def l2_peaks(dev, stream, mib=32):
    """Best-of-6 GB/s of rmpb_l2_probe mode 0 (streaming 16-B reads, L1
    bypassed, 32 MiB L2-resident buffer)."""
    import ctypes

    import torch

    from paper_2301_08068_b200 import _lib

    buf = torch.ones(mib * 1024 * 1024, dtype=torch.uint8, device=dev)
    out = {}
    for mode, name, reps in ((0, "stream", 40),):
        nbytes = ctypes.c_int64(0)
        best = None
        for _ in range(6):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            _lib.call("rmpb_l2_probe", buf.data_ptr(), buf.numel(), reps, mode,
                      ctypes.byref(nbytes), stream.cuda_stream)
            e1.record(stream)
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        out[name] = round(nbytes.value / (best * 1e-3) / 1e9, 1)
    return out


# ----------------------------------------------------------------------------
# CPU legs (reference kernels from oracle/_ref; C port fallback)

def _cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def _cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(grid, states, seconds=10.0, threads=None, seconds_1t=4.0):
    """Times the reference's CPU path (oracle/_ref compiled kernels driven as
    rmpnav's ckern.py/_pool.py do) on a bounded sample of this workload."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    threads = threads or _cpu_threads()
    dirs = O.sample_directions(N_RAYS)
    vals = grid.values
    kind = "reference" if O.ref_available() else "port"
    pool = O.RefPool(threads)
    done, t0 = 0, time.perf_counter()
    per = []
    try:
        while True:
            st = states[done % len(states)]
            tc = time.perf_counter()
            if kind == "reference":
                O.ref_ray_policy(vals, grid.origin, grid.resolution, st.position, st.velocity,
                                 dirs, PARAMS, MAX_RANGE, pool)
            else:
                O.ray_policy(vals, grid.origin, grid.resolution, st.position, st.velocity, dirs,
                             PARAMS, MAX_RANGE, workers=threads)
            per.append(time.perf_counter() - tc)
            done += 1
            el = time.perf_counter() - t0
            if (el >= seconds and done >= 3) or done >= 100000:
                break
    finally:
        pool.close()
    rays_s = done * N_RAYS / el
    # W = 1 (the reference harness at one worker and at all cores)
    one, t1 = 0, time.perf_counter()
    pool1 = O.RefPool(1)
    try:
        while True:
            st = states[one % len(states)]
            if kind == "reference":
                O.ref_ray_policy(vals, grid.origin, grid.resolution, st.position, st.velocity,
                                 dirs, PARAMS, MAX_RANGE, pool1)
            else:
                O.ray_policy(vals, grid.origin, grid.resolution, st.position, st.velocity, dirs,
                             PARAMS, MAX_RANGE, workers=1)
            one += 1
            el1 = time.perf_counter() - t1
            if el1 >= seconds_1t and one >= 2:
                break
    finally:
        pool1.close()
    per_ms = sorted(1e3 * t for t in per)
    return {"value": round(rays_s, 1), "unit": "rays/s", "cores": threads, "kind": kind,
            "hz": round(done / el, 2),
            "call_ms_median": round(statistics.median(per_ms), 3),
            "call_ms_best": round(per_ms[0], 3),
            "call_ms_p95": round(per_ms[min(len(per_ms) - 1, int(0.95 * len(per_ms)))], 3),
            "cpu_model": _cpu_model(),
            "value_1_thread": round(one * N_RAYS / el1, 1), "hz_1_thread": round(one / el1, 2),
            "sample": f"{done} poses x {N_RAYS} rays of the same workload in {el:.1f} s "
                      f"({threads} threads, reference chunk pool, CHUNK=2048)"}


def run_reference(args):
    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    if rank != 0:
        return None
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    threads = _cpu_threads()
    kind = "reference" if O.ref_available() else "port"
    if kind == "reference":
        K = O.ref()

        def bake(pack, origin, res, dims):
            out = np.empty(tuple(dims))
            nx = dims[0]
            pool = O.RefPool(threads)
            args_ = (pack["kinds"], pack["ops"], pack["centers"], pack["sizes"],
                     pack["velocities"], pack["empty_dist"])
            pool.run(lambda i, s, e: K.bake_chunk(*args_, origin[0], origin[1], origin[2], res,
                                                  s, e, out), nx, chunk=max(1, nx // (4 * threads)))
            pool.close()
            return out

        def distance_factory(scene):
            pk = scene.packed()
            a = (pk["kinds"], pk["ops"], pk["centers"], pk["sizes"], pk["velocities"],
                 pk["empty_dist"])

            def d(x):
                out = np.empty(1)
                K.scene_distance_chunk(*a, 0.0, np.ascontiguousarray(x.reshape(1, 3)), 0, 1, out)
                return float(out[0])
            return d
    else:
        bake = O.bake_values

        def distance_factory(scene):
            return lambda x: float(O.scene_distance_many(scene.packed(), x.reshape(1, 3), 0.0)[0])

    from paper_2301_08068_b200 import synth

    scene = synth.c1_scene()
    grid = synth.c1_grid(scene, bake=bake)
    states = synth.bench_states(scene, count=args.poses, seed=123,
                                distance=distance_factory(scene))
    dirs = O.sample_directions(N_RAYS)
    pool = O.RefPool(threads)
    sample = args.ref_poses_per_step

    def one_step(base):
        for j in range(sample):
            st = states[(base + j) % len(states)]
            if kind == "reference":
                O.ref_ray_policy(grid.values, grid.origin, grid.resolution, st.position,
                                 st.velocity, dirs, PARAMS, MAX_RANGE, pool)
            else:
                O.ray_policy(grid.values, grid.origin, grid.resolution, st.position, st.velocity,
                             dirs, PARAMS, MAX_RANGE, workers=threads)

    for w in range(args.warmup):
        one_step(w * sample)
    t0 = time.perf_counter()
    for k in range(args.steps):
        one_step((args.warmup + k) * sample)
    el = time.perf_counter() - t0
    pool.close()
    rays = args.steps * sample * N_RAYS
    value = rays / el
    ms = el / args.steps * 1e3
    return {
        "impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": "rays/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": "C4-shape batch on the C1 headline map (CPU: bounded sample of "
                               f"{sample} poses per step) x {N_RAYS} Halton rays, 200x200x100 "
                               "@0.1 m (200 boxes), max range 10 m, static_map",
                   "poses_per_step": sample, "rays_per_pose": N_RAYS, "max_range_m": MAX_RANGE},
        "hz": round(args.steps * sample / el, 2),
        "cpu_baseline": {"value": round(value, 1), "unit": "rays/s", "cores": threads,
                         "kind": kind,
                         "sample": f"{sample} poses x {N_RAYS} rays per step, {threads} threads"},
        "e2e": {"value": round(value, 1), "unit": "rays/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c4", choices=["c4", "c5"],
                    help="c4 (default, the driver line): 4096 poses x 65536 rays per GPU; "
                         "c5: one 1 M-ray pose on the C5 TSDF split over the GPUs")
    ap.add_argument("--poses", type=int, default=4096, help="poses per rank per step")
    ap.add_argument("--latency-calls", type=int, default=200)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true",
                    help="skip the post-run check of 8 timed poses against the reference")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the extra C3 / C2 lines")
    ap.add_argument("--ref-poses-per-step", type=int, default=8)
    ap.add_argument("--ncu-traffic", type=float, default=None,
                    help="dram bytes per launch from an ncu --set full capture")
    args = ap.parse_args(argv)
    if args.warmup < 3 and args.impl == "b200":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        out = run_reference(args)
    elif args.workload == "c5":
        out = run_c5(args)
    else:
        out = run_b200(args)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
