"""Reduced workload that launches every librmpb kernel family once at small
sizes, for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

  compute-sanitizer --tool memcheck --target-processes all \
      python scripts/sanitize_suite.py

Kernels: k_ray_policy2 (batch, exact: plain / per-ray outputs / FAST,
inside + outside poses, segmented + ticket fold), k_ray_policy (lean) and
its K4 exchange variant (world-1 mailbox), k_ray_server (LatencyServer),
k_lidar_warp (lattice + raw points, multi-unit fold), the rollout kernels,
the DDA kernels, bake / TSDF bake / brick build, scene trace / distance,
ESDF lookup, the unfused grid_trace / policy_reduce, pinv, Halton / lattice
bundles, the region update.  Exits 0 after printing one line per family;
the sanitizer's own summary reports the errors.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2301_08068_b200 as P  # noqa: E402
from paper_2301_08068_b200 import _lib, synth  # noqa: E402
from paper_2301_08068_b200._kernels import b200  # noqa: E402
from paper_2301_08068_b200.device import (DdaPolicyEngine, PeerMailbox, RayPolicyEngine,  # noqa: E402
                                          lidar_points_batch_device, lidar_policy_batch_device)

STATIC = (88.0, 1.4, 140.0, 1.2, 1e-6, 2.4, 0.2)
LIDAR = (1.2, 1.5, 3.0, 1.0, 1e-6, 1.3, 1.0)


def say(what):
    torch.cuda.synchronize()
    print("ok", what, flush=True)


def main():
    scene = synth.c1_scene(n_boxes=12, hi=np.array([3.9, 3.9, 1.9]))
    dims = (40, 40, 20)
    vals = b200.bake_values(scene.packed(), np.zeros(3), 0.1, dims)
    vals = vals.astype(np.float32).astype(np.float64)
    say("bake")
    grid = P.EsdfGrid(np.zeros(3), 0.1, dims, vals)
    bundle = P.sample_directions(2048)
    say("halton bundle")
    states = synth.bench_states(scene, count=6, seed=3, distance=synth.host_box_distance(scene))
    xs = np.stack([s.position for s in states] + [[-0.5, 1.0, 0.5], [1.0, 1.0, 3.0]])
    vs = np.tile([[0.4, -0.2, 0.1]], (len(xs), 1))
    dirs = bundle.directions
    b200.ray_policy_batch(grid.values, grid.origin, 0.1, xs, vs, dirs, STATIC, 10.0, 0.05, 0.9)
    _lib.set_option("seg_rays", 512)  # several segments per pose: partials + ticket fold
    b200.ray_policy_batch(grid.values, grid.origin, 0.1, xs, vs, dirs, STATIC, 10.0, 0.05, 0.9)
    _lib.set_option("seg_rays", 0)
    _lib.set_option("kernel", 2)
    b200.ray_policy_fused(grid.values, grid.origin, 0.1, xs[0], vs[0], dirs, STATIC, 10.0, 0.05,
                          0.9, with_rays=True)
    b200.ray_policy_fused(grid.values, grid.origin, 0.1, xs[-2], vs[0], dirs, STATIC, 10.0, 0.05,
                          0.9, with_rays=True)
    _lib.set_option("kernel", 0)
    say("k_ray_policy2 (batch, segmented, RAYOUT, outside pose)")
    eng = RayPolicyEngine(grid, bundle, STATIC, 10.0)
    x = torch.from_numpy(xs).cuda()
    v = torch.from_numpy(vs).cuda()
    eng.evaluate(x, v)
    ctr = torch.zeros(1, dtype=torch.int64, device="cuda")
    eng.evaluate(x, v, step_counter=ctr)
    fast = RayPolicyEngine(grid, bundle, STATIC, 10.0, mode="fast")
    fast.evaluate(x, v)
    say("engine exact / step counter / FAST")
    P.ray_policy(states[0], grid, bundle, P.preset("static_map").obstacle, 10.0)
    b200.grid_trace_ex(grid.values, grid.origin, 0.1, xs[0], dirs, 10.0, 0.05, 0.9, True, True)
    say("k_ray_policy (lean) + k_grid_trace")
    mb = PeerMailbox(1, 0)
    mb.open([mb.ipc_handle])
    for ep in (1, 2, 3):
        eng.exchange(x[0].contiguous(), v[0].contiguous(), mb, ep, 0, eng.n_rays)
    parts = torch.stack([eng.partial(x[0].contiguous(), v[0].contiguous(), a, b)
                         for a, b in ((0, 700), (700, 2048))])
    eng.resolve(parts)
    mb.close()
    say("K4 exchange (world 1), partial + fold")
    with P.LatencyServer(grid, bundle, P.preset("static_map").obstacle, 10.0,
                         idle_timeout_s=0.2) as srv:
        for s in states[:3]:
            srv.policy(s)
    say("k_ray_server")
    n, S = 4096 + 37, 5
    rng = np.random.default_rng(1)
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    rgs = rng.uniform(0.0, 3.0, (S, n))
    valid = rng.random((S, n)) < 0.8
    Rs = np.stack([np.linalg.qr(rng.normal(size=(3, 3)))[0] for _ in range(S)]).reshape(S, 9)
    for tgt in (38000, 3):
        _lib.set_option("lidar_warps", tgt)
        lidar_policy_batch_device(torch.from_numpy(d).cuda(), torch.from_numpy(Rs.copy()).cuda(),
                                  torch.from_numpy(rgs).cuda(),
                                  torch.from_numpy(valid.astype(np.uint8)).cuda(),
                                  torch.from_numpy(rng.normal(size=(S, 3))).cuda(), LIDAR, 0.3)
        pts = torch.from_numpy(rng.uniform(-2, 2, (S, n, 3)).astype(np.float32)).cuda()
        lidar_points_batch_device(pts, None, torch.from_numpy(rng.normal(size=(S, 3))).cuda(),
                                  LIDAR, 0.3)
    _lib.set_option("lidar_warps", 38000)
    scan = synth.lidar_scans(scene, states[:1], 16, 64, 10.0)[0]
    P.lidar_policy(states[0].velocity, scan, P.preset("lidar").obstacle)
    say("k_lidar_warp (lattice, points, fold) + scene trace")
    from paper_2301_08068_b200.rollout import BatchRolloutConfig, rollout_batch

    cfg = BatchRolloutConfig(params=P.preset("static_map"), dt=0.02, max_time=0.2, max_range=5.0)
    starts = np.stack([s.position for s in states[:3]])
    goals = starts + np.array([1.0, 0.5, 0.0])
    rollout_batch(scene, grid, bundle, starts, goals, cfg, record_ticks=4)
    say("rollout kernels")
    dda = DdaPolicyEngine(grid, bundle, STATIC, 5.0)
    dda.evaluate(x, v)
    dda.occ.trace(xs[0], dirs[:256], 5.0)
    say("DDA")
    ds = b200.device_scene(scene.packed())
    tsdf = b200.DeviceGrid.bake_tsdf(ds, np.zeros(3), 0.1, dims, 0.2)
    tsdf.values()
    b200.grid_trace_ex(tsdf, np.zeros(3), 0.1, xs[0], dirs[:512], 5.0, 0.05, 0.9)
    say("TSDF bake + brick build + brick trace + readback")
    b200.esdf_sample_many(grid.values, grid.origin, 0.1, rng.uniform(0, 4, (300, 3)))
    b200.scene_distance_many(scene.packed(), rng.uniform(0, 4, (300, 3)), 0.0)
    m, w, nh = b200.policy_reduce(dirs[:100], rng.uniform(0, 3, 100), [1, 0, 0], STATIC)
    P.pinv_psd(np.stack([np.eye(3), np.zeros((3, 3))]), 1e-3)
    say("esdf lookup / scene distance / policy_reduce / pinv")
    grid.update((slice(5, 9), 7, slice(2, 6)), -0.25)
    P.ray_policy(states[0], grid, bundle, P.preset("static_map").obstacle, 10.0)
    P.RayBundle(b200.DeviceBundle(lattice=(8, 16, 30.0)).directions())
    say("region update + lattice bundle")
    print("SANITIZE_SUITE_DONE", flush=True)


if __name__ == "__main__":
    main()
