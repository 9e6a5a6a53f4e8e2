#!/usr/bin/env python3
"""Secondary measurements for BASELINE.json configs C2 (ray-count x range
sweep), C3 (LiDAR-direct 128x1024 scans) and C5 (1000x1000x200 block-hashed
TSDF, 1 M rays per pose, ray split) on ONE B200, each beside the reference's
CPU path timed on the box's host cores (bounded samples).  One JSON object
per line on stdout.  bench.py stays the driver contract; this script is the
evidence for the other rows of SURVEY.md §8.

usage: python scripts/bench_configs.py [--only c2,c3,c5] [--quick]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

STATIC = (88.0, 1.4, 140.0, 1.2, 1e-6, 2.4, 0.2)
LIDAR = (1.2, 1.5, 3.0, 1.0, 1e-6, 1.3, 1.0)


def ev_time(fn, reps=3, flush=None):
    import torch

    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts), statistics.median(ts)


def wall_med(fn, n=50):
    for _ in range(5):
        fn(0)
    ts = []
    for i in range(n):
        t0 = time.perf_counter()
        fn(i)
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def c2(args, out):
    import torch

    import oracle as O
    from paper_2301_08068_b200 import synth
    from paper_2301_08068_b200._kernels import b200
    from paper_2301_08068_b200.device import RayPolicyEngine

    scene = synth.c1_scene()
    grid = synth.c1_grid(scene)
    dist = synth.host_box_distance(scene)
    ns = [4096, 16384, 65536, 262144, 1048576]
    ranges = [2.0, 5.0, 10.0, 20.0]
    if args.quick:
        ns, ranges = [4096, 65536, 1048576], [2.0, 10.0]
    states = synth.bench_states(scene, count=8192, seed=123, distance=dist)
    xa, va = synth.states_arrays(states)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    threads = cpu_threads()
    pool = O.RefPool(threads) if O.ref_available() else None
    dg = b200.DeviceGrid(grid.values, grid.origin, grid.resolution)
    for n in ns:
        bundle = b200.DeviceBundle(halton_n=n)
        dirs_ref = O.sample_directions(n)
        P = max(1, min(8192, (1 << 28) // n))
        x = torch.from_numpy(xa[:P].copy()).cuda()
        v = torch.from_numpy(va[:P].copy()).cuda()
        for mr in ranges:
            eng = RayPolicyEngine(dg, bundle, STATIC, mr)
            ctr = torch.zeros(1, dtype=torch.int64, device="cuda")
            eng.evaluate(x, v, step_counter=ctr)
            torch.cuda.synchronize()
            steps = int(ctr.item())
            best, med = ev_time(lambda: eng.evaluate(x, v), reps=3, flush=flush)
            x1, v1 = x[:1].contiguous(), v[:1].contiguous()
            lat_best, lat_med = ev_time(lambda: eng.evaluate(x1, v1), reps=20)
            rec = {"config": "C2", "rays": n, "max_range_m": mr, "poses_per_launch": P,
                   "ms_per_launch": round(med, 4), "rays_per_s": round(P * n / (med * 1e-3), 1),
                   "hz_throughput": round(P / (med * 1e-3), 1),
                   "voxel_steps_per_s": round(steps / (med * 1e-3), 1),
                   "steps_per_ray": round(steps / (P * n), 3),
                   "single_pose_kernel_us_events": round(lat_med * 1e3, 1)}
            if pool is not None:
                k = 0
                t0 = time.perf_counter()
                while True:
                    st = states[k % len(states)]
                    O.ref_ray_policy(grid.values, grid.origin, grid.resolution, st.position,
                                     st.velocity, dirs_ref, STATIC, mr, pool)
                    k += 1
                    el = time.perf_counter() - t0
                    if el > (1.0 if args.quick else 3.0) or k >= 200:
                        break
                rec["cpu_reference"] = {"rays_per_s": round(k * n / el, 1),
                                        "hz": round(k / el, 2), "threads": threads,
                                        "sample": f"{k} poses"}
            print(json.dumps(rec), flush=True)
            out.append(rec)
    if pool is not None:
        pool.close()


def c3(args, out):
    import torch

    import oracle as O
    from paper_2301_08068_b200 import synth
    from paper_2301_08068_b200.device import lidar_points_batch_device, lidar_policy_batch_device
    from paper_2301_08068_b200.policies import lidar_policy, preset
    from paper_2301_08068_b200.rays import scan_pattern

    scene = synth.c1_scene()
    states = synth.bench_states(scene, count=10, seed=123,
                                distance=synth.host_box_distance(scene))
    scans = synth.lidar_scans(scene, states, 128, 1024, 20.0)
    lp = preset("lidar").obstacle
    n = 128 * 1024
    # single scan through the public API (host buffers, lattice cached on device)
    lat = wall_med(lambda i: lidar_policy(states[i % 10].velocity, scans[i % 10], lp), n=100)
    # throughput: S scans per launch, device resident
    S = 1024
    dirs = torch.from_numpy(np.ascontiguousarray(scan_pattern(128, 1024))).cuda()
    rg = torch.from_numpy(np.stack([scans[i % 10].ranges for i in range(S)])).cuda()
    vl = torch.from_numpy(np.stack([scans[i % 10].valid for i in range(S)]).astype(np.uint8)).cuda()
    R = torch.from_numpy(np.stack([scans[i % 10].orientation for i in range(S)])
                         .reshape(S, 9).copy()).cuda()
    v = torch.from_numpy(np.stack([states[i % 10].velocity for i in range(S)])).cuda()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    best, med = ev_time(lambda: lidar_policy_batch_device(dirs, R, rg, vl, v, LIDAR, 0.3),
                        reps=5, flush=flush)
    beam_bytes = 8 + 1  # range f64 + valid u8 per beam (lattice L2-resident)
    gbs = S * n * beam_bytes / (med * 1e-3) / 1e9
    rec = {"config": "C3", "beams_per_scan": n, "scans_per_launch": S,
           "ms_per_launch": round(med, 4), "scans_per_s": round(S / (med * 1e-3), 1),
           "beams_per_s": round(S * n / (med * 1e-3), 1),
           "stream_GBps": round(gbs, 1), "hbm_frac": round(gbs / 6541.8, 3),
           "single_scan_api_us_median": round(lat * 1e6, 1),
           "single_scan_hz": round(1.0 / lat, 1)}
    # K2b: the same scans as raw f32 sensor-frame points (invalid -> 0)
    pts = torch.where(vl.bool()[:, :, None], dirs[None] * rg[:, :, None], 0.0).float()
    pts = torch.nan_to_num(pts, nan=0.0, posinf=0.0, neginf=0.0).contiguous()
    _bp, mp = ev_time(lambda: lidar_points_batch_device(pts, R, v, LIDAR, 0.3), reps=5,
                      flush=flush)
    pgbs = S * n * 12 / (mp * 1e-3) / 1e9
    rec["points"] = {"ms_per_launch": round(mp, 4), "scans_per_s": round(S / (mp * 1e-3), 1),
                     "stream_GBps": round(pgbs, 1), "hbm_frac": round(pgbs / 6541.8, 3),
                     "bytes_per_point": 12}
    if O.ref_available():
        pool = O.RefPool(cpu_threads())
        wd = [np.ascontiguousarray(s.world_directions()) for s in scans]

        def ref_one(i):
            s = scans[i % 10]
            O.ref_lidar_policy(wd[i % 10], s.ranges, s.valid, states[i % 10].velocity, LIDAR, 0.3,
                               pool)
        lat_ref = wall_med(ref_one, n=30)
        pool.close()
        pool1 = O.RefPool(1)

        def ref_one1(i):
            s = scans[i % 10]
            O.ref_lidar_policy(wd[i % 10], s.ranges, s.valid, states[i % 10].velocity, LIDAR, 0.3,
                               pool1)
        lat_ref1 = wall_med(ref_one1, n=30)
        rec["cpu_reference"] = {"single_scan_ms_median_all_threads": round(lat_ref * 1e3, 3),
                                "single_scan_ms_median_1_thread": round(lat_ref1 * 1e3, 3),
                                "threads": cpu_threads(),
                                "note": "rmpnav lidar_policy reduce with world dirs precomputed"}
    print(json.dumps(rec), flush=True)
    out.append(rec)


def c5(args, out):
    import torch

    import oracle as O
    from paper_2301_08068_b200 import _lib as L, synth
    from paper_2301_08068_b200._kernels import b200
    from paper_2301_08068_b200.device import RayPolicyEngine
    from paper_2301_08068_b200.parallel import balanced_range

    t0 = time.perf_counter()
    scene = synth.c5_scene()
    dg_dense, dg_brick, info = synth.c5_grids(scene)
    bake_s = time.perf_counter() - t0
    states = synth.bench_states(scene, count=8, seed=123,
                                distance=synth.host_box_distance(scene))
    n = 1 << 20
    bundle = b200.DeviceBundle(halton_n=n)
    rec = {"config": "C5", "dims": list(synth.C5_DIMS), "res_m": synth.C5_RES,
           "boxes": len(scene.primitives), "tau_m": synth.C5_TAU, "rays": n,
           "bake_and_build_s": round(bake_s, 2), **info}
    res = {}
    for name, dg in (("dense_quad", dg_dense), ("brick", dg_brick)):
        eng = RayPolicyEngine(dg, bundle, STATIC, 10.0)
        x = torch.from_numpy(np.stack([s.position for s in states])).cuda()
        v = torch.from_numpy(np.stack([s.velocity for s in states])).cuda()
        ctr = torch.zeros(1, dtype=torch.int64, device="cuda")
        eng.evaluate(x, v, step_counter=ctr)
        torch.cuda.synchronize()
        best, med = ev_time(lambda: eng.evaluate(x, v), reps=3)
        x1, v1 = x[0].contiguous(), v[0].contiguous()
        one_best, one_med = ev_time(lambda: eng.evaluate(x1.view(1, 3), v1.view(1, 3)), reps=10)
        # 8-way ray split of one pose: per-GPU share and the fixed-order fold
        shares = []
        parts = []
        for r in range(8):
            b_, e_ = balanced_range(n, 8, r)
            sb, sm = ev_time(lambda: eng.partial(x1, v1, b_, e_), reps=5)
            shares.append(sm)
            parts.append(eng.partial(x1, v1, b_, e_))
        # K4 fused: one rank's share + mailbox post/wait + fold + pinv in one
        # launch (world-1 mailbox on this GPU: the epilogue's own cost)
        from paper_2301_08068_b200.device import PeerMailbox
        mb = PeerMailbox(1, 0)
        b0, e0 = balanced_range(n, 8, 0)
        ep = [0]

        def fused():
            ep[0] += 1
            eng.exchange(x1, v1, mb, ep[0], b0, e0)
        fb, fm = ev_time(fused, reps=5)
        pb, pm = ev_time(lambda: eng.partial(x1, v1, b0, e0), reps=5)
        slot_split, acc_split = eng.resolve(torch.stack(parts))
        slot_whole, acc_whole = eng.evaluate(x1.view(1, 3), v1.view(1, 3))
        torch.cuda.synchronize()
        sw, aw = slot_whole[0].cpu().numpy(), acc_whole[0].cpu().numpy()
        ss, as_ = slot_split.cpu().numpy(), acc_split.cpu().numpy()
        res[name] = {"ms_per_launch_8_poses": round(med, 3),
                     "rays_per_s": round(8 * n / (med * 1e-3), 1),
                     "voxel_steps_per_s": round(int(ctr.item()) / (med * 1e-3), 1),
                     "steps_per_ray": round(int(ctr.item()) / (8 * n), 3),
                     "single_pose_ms": round(one_med, 3),
                     "ray_split_8_share_ms_max": round(max(shares), 3),
                     "k4_fused_share_ms_world1": round(fm, 4),
                     "partial_only_share_ms": round(pm, 4),
                     "split_vs_whole_rel": float(np.abs(ss[:12] - sw[:12]).max() /
                                                 max(1e-300, np.abs(sw[:12]).max())),
                     "split_n_hits_equal": bool(ss[12] == sw[12])}
    rec["gpu"] = res
    # parity of the block-hashed map vs the dense map and the CPU oracle on a
    # sample of the pose's rays
    x0 = states[0].position
    samp = np.ascontiguousarray(O.sample_directions(4096))
    tb, cb, _ = b200.grid_trace_ex(dg_brick, synth.C5_ORIGIN, synth.C5_RES, x0, samp, 10.0,
                                   0.5 * synth.C5_RES, 0.9, with_cells=True)
    td, cd, _ = b200.grid_trace_ex(dg_dense, synth.C5_ORIGIN, synth.C5_RES, x0, samp, 10.0,
                                   0.5 * synth.C5_RES, 0.9, with_cells=True)
    rec["brick_vs_dense_bit_exact"] = bool(np.array_equal(tb, td) and np.array_equal(cb, cd))
    if args.oracle_c5:
        vals = synth.c5_values_host(scene)
        tr, cr = O.grid_trace(vals, synth.C5_ORIGIN, synth.C5_RES, x0, samp, 10.0,
                              0.5 * synth.C5_RES, 0.9, with_cells=True, workers=cpu_threads())
        rec["brick_vs_oracle_bit_exact"] = bool(np.array_equal(tb, tr) and np.array_equal(cb, cr))
        if O.ref_available():
            pool = O.RefPool(cpu_threads())
            st = states[0]
            k = 0
            t1 = time.perf_counter()
            dirs_ref = O.sample_directions(n)
            O.ref_ray_policy(vals, synth.C5_ORIGIN, synth.C5_RES, st.position, st.velocity,
                             dirs_ref, STATIC, 10.0, pool)
            el = time.perf_counter() - t1
            pool.close()
            rec["cpu_reference_1pose_s"] = round(el, 3)
            rec["cpu_reference_threads"] = cpu_threads()
    print(json.dumps(rec), flush=True)
    out.append(rec)


def c4loop(args, out):
    """Row f1: closed-loop ticks for a batch of robots on the C1 map (every
    tick = checks + fused 65536-ray policy + combine + clamp + Euler, on
    device, no host round trip)."""
    import torch

    import paper_2301_08068_b200 as P
    from paper_2301_08068_b200 import synth
    from paper_2301_08068_b200.rollout import BatchRolloutConfig, RolloutBatch

    scene = synth.c1_scene()
    grid = synth.c1_grid(scene)
    dist = synth.host_box_distance(scene)
    n_rob = 1024 if args.quick else 4096
    starts = synth.states_arrays(synth.bench_states(scene, n_rob, seed=123, distance=dist))[0]
    goals = synth.states_arrays(synth.bench_states(scene, n_rob, seed=321, distance=dist))[0]
    bundle = P.sample_directions(65536)
    cfg = BatchRolloutConfig(params=P.preset("static_map"), dt=0.01, max_time=60.0,
                             max_range=10.0)
    rb = RolloutBatch(scene, grid, bundle, starts, goals, cfg)
    rb.run(2)
    torch.cuda.synchronize()
    ticks = 10 if args.quick else 30
    t0 = time.perf_counter()
    left = rb.run(ticks)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    res = rb.result()
    rec = {"config": "C4-closed-loop", "robots": n_rob, "rays_per_robot": 65536,
           "ticks": ticks, "s_per_tick": round(el / ticks, 5),
           "robot_steps_per_s": round(n_rob * ticks / el, 1),
           "still_running": left,
           "outcomes": {k: res.outcome.count(k) for k in set(res.outcome)},
           "note": "wall clock around rmpb_rollout_run (3 launches per tick, polled every 16)"}
    # the same robots with policy_only rays (stopped at the activation radius)
    import dataclasses
    cfg_po = dataclasses.replace(cfg, policy_only=True)
    rbp = RolloutBatch(scene, grid, bundle, starts, goals, cfg_po)
    rbp.run(2)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rbp.run(ticks)
    torch.cuda.synchronize()
    el_po = time.perf_counter() - t0
    rec["policy_only_s_per_tick"] = round(el_po / ticks, 5)
    rec["policy_only_robot_steps_per_s"] = round(n_rob * ticks / el_po, 1)
    # small batches are launch-bound: ticks replayed from a captured CUDA graph
    # (16 per graph launch) vs eager launches
    from paper_2301_08068_b200 import _lib as L
    small = {}
    for nr in (1, 64):
        for gr in (0, 1):
            L.call("rmpb_set_option", b"graphs", gr)
            rb2 = RolloutBatch(scene, grid, bundle, starts[:nr], goals[:nr], cfg)
            rb2.run(32)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rb2.run(96)
            torch.cuda.synchronize()
            small[f"robots{nr}_{'graph' if gr else 'eager'}_us_per_tick"] = round(
                (time.perf_counter() - t0) / 96 * 1e6, 1)
    L.call("rmpb_set_option", b"graphs", 1)
    rec["small_batches"] = small
    print(json.dumps(rec), flush=True)
    out.append(rec)


def k5(args, out):
    """K5: Amanatides-Woo DDA over the C1 occupancy (bit-packed, 500 KB),
    4096 poses x 65536 rays per launch -- a different traversal from the
    reference's sphere trace, reported separately."""
    import torch

    from paper_2301_08068_b200 import synth
    from paper_2301_08068_b200._kernels import b200
    from paper_2301_08068_b200.device import DdaPolicyEngine

    scene = synth.c1_scene()
    grid = synth.c1_grid(scene)
    states = synth.bench_states(scene, count=4096, seed=123,
                                distance=synth.host_box_distance(scene))
    x = torch.from_numpy(synth.states_arrays(states)[0]).cuda()
    v = torch.from_numpy(synth.states_arrays(states)[1]).cuda()
    bundle = b200.DeviceBundle(halton_n=65536)
    eng = DdaPolicyEngine(b200.DeviceGrid(grid.values, grid.origin, grid.resolution), bundle,
                          STATIC, 10.0)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    best, med = ev_time(lambda: eng.evaluate(x, v), reps=3, flush=flush)
    t, vox, steps = eng.occ.trace(states[0].position, np.ascontiguousarray(
        b200.DeviceBundle(halton_n=65536).directions()), 10.0)
    rec = {"config": "K5-DDA (C1 map, occupancy = value <= 0)", "poses_per_launch": 4096,
           "rays_per_pose": 65536, "ms_per_launch": round(med, 3),
           "rays_per_s": round(4096 * 65536 / (med * 1e-3), 1),
           "hz_throughput": round(4096 / (med * 1e-3), 1),
           "voxels_visited_per_ray_pose0": round(float(steps.mean()), 2),
           "hit_fraction_pose0": round(float(np.isfinite(t).mean()), 4),
           "occupancy_bytes": int(eng.occ.bits().nbytes)}
    print(json.dumps(rec), flush=True)
    out.append(rec)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c2,c3,c5,c4loop,k5")
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--oracle-c5", action="store_true",
                    help="also check C5 against the dense CPU oracle (needs ~1 GB host RAM)")
    args = ap.parse_args()
    out = []
    for name in args.only.split(","):
        {"c2": c2, "c3": c3, "c5": c5, "c4loop": c4loop, "k5": k5}[name.strip()](args, out)


if __name__ == "__main__":
    main()
