"""Generate the golden vectors in tests/golden/ BY RUNNING THE REFERENCE.

Run in the build container (where /root/reference exists):

    python oracle/build_ref.py && python tests/golden/make_golden.py

It assembles an importable copy of the reference package in a temporary
directory (the read-only mount cannot take the compiled module), drops in
the reference's own compiled ``_ckern`` from oracle/_ref, imports ``rmpnav``
and calls its PUBLIC API (``bake_esdf``, ``sample_directions``,
``raycast_many``, ``ray_policy``, ``lidar_policy``, ``synthesize_scan``,
``esdf_lookup``, ``pinv_psd``, ``halton``) with backend="compiled".  The
outputs are written to ``tests/golden/rmpnav_golden.npz``; nothing from the
reference's sources is stored.  The GPU box never runs this script.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import sys
import sysconfig
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src/rmpnav"


def import_reference(tmp: str):
    dst = os.path.join(tmp, "rmpnav")
    shutil.copytree(REF_SRC, dst)
    so = "_ckern" + sysconfig.get_config_var("EXT_SUFFIX")
    shutil.copy(os.path.join(ROOT, "oracle", "_ref", so), os.path.join(dst, "_kernels", so))
    sys.path.insert(0, tmp)
    import rmpnav

    assert "compiled" in rmpnav.available_backends(), "reference compiled backend missing"
    return rmpnav


def main():
    with tempfile.TemporaryDirectory(prefix="rmpnav_golden_") as tmp:
        R = import_reference(tmp)
        import rmpnav.bench  # noqa: F401
        import rmpnav.core  # noqa: F401
        import rmpnav.rays  # noqa: F401
        be = "compiled"
        g = {}
        # --- SPEC known-answer checks on the reference itself -----------------
        g["kat_halton"] = np.array([R.halton(1, 2), R.halton(3, 2), R.halton(1, 3),
                                    R.halton(7, 2), R.halton(10, 3)])
        g["kat_dir1"] = R.sample_directions(1).directions.copy()
        sph = R.Scene(R.Aabb.cube(12.0), [R.Primitive.sphere((0, 0, 0), 1.0)])
        g["kat_sphere_ray"] = np.array(R.raycast(sph, (5, 0, 0), (-1, 0, 0)))

        # --- a small cluttered world (spheres, boxes, subtraction) -----------
        scene, start, goal = R.generate_world(3, 30, bounds=R.Aabb.cube(6.0))
        pk = scene.packed()
        for k in ("kinds", "ops", "centers", "sizes", "velocities"):
            g["scene_" + k] = np.asarray(pk[k])
        g["scene_empty"] = np.array(pk["empty_dist"])
        g["scene_bounds"] = np.stack([scene.bounds.lo, scene.bounds.hi])
        grid = R.bake_esdf(scene, 0.2, pad=1.0)
        g["grid_origin"] = grid.origin
        g["grid_res"] = np.array(grid.resolution)
        g["grid_dims"] = np.array(grid.dims)
        g["grid_sha256_f64"] = np.frombuffer(
            hashlib.sha256(grid.values.tobytes()).digest(), dtype=np.uint8)
        # the traced grid is the f32-rounded bake (SURVEY.md §8c recipe)
        g32 = R.EsdfGrid(grid.origin, grid.resolution, grid.dims,
                         grid.values.astype(np.float32).astype(np.float64))
        n = 2048
        dirs = R.sample_directions(n).directions.copy()
        g["dirs"] = dirs
        states = R.bench.bench_states(scene, count=6, seed=5)
        xs = np.array([s.position for s in states])
        vs = np.array([s.velocity for s in states])
        g["pose_x"], g["pose_v"] = xs, vs
        p = R.preset("static_map").obstacle
        T, SL, AC, MET = [], [], [], []
        for s in states:
            t = R.raycast_many(g32, s.position, dirs, 10.0, backend=be)
            metric, weighted, nh = R.get_backend(be).policy_reduce(dirs, t, s.velocity,
                                                                   p.as_tuple(), 0.0)
            pol = R.ray_policy(s, g32, R.RayBundle(dirs), p, 10.0, backend=be)
            T.append(t)
            SL.append(np.concatenate([metric.ravel(), weighted, [nh]]))
            AC.append(pol.accel)
            MET.append(pol.metric)
        g["trace_t"] = np.array(T)
        g["slots"] = np.array(SL)
        g["accels"] = np.array(AC)
        g["metrics"] = np.array(MET)
        # an f64 (not f32-exact) grid trace for pose 0
        g["trace_t_f64grid"] = R.raycast_many(grid, states[0].position, dirs, 10.0, backend=be)
        # --- LiDAR-direct ----------------------------------------------------
        lp = R.preset("lidar").obstacle
        rot = np.array([[0.0, -1.0, 0.0], [1.0, 0.0, 0.0], [0.0, 0.0, 1.0]])
        LR, LV, LA, LM = [], [], [], []
        for i, s in enumerate(states[:3]):
            scan = R.synthesize_scan(scene, s.position, 16, 128, max_range=20.0,
                                     orientation=rot if i == 1 else None, dropout=0.1, rng=i,
                                     backend=be)
            pol = R.lidar_policy(s.velocity, scan, lp, backend=be)
            LR.append(scan.ranges)
            LV.append(scan.valid)
            LA.append(pol.accel)
            LM.append(pol.metric)
        g["lidar_ranges"], g["lidar_valid"] = np.array(LR), np.array(LV)
        g["lidar_accels"], g["lidar_metrics"] = np.array(LA), np.array(LM)
        g["lidar_rot"] = rot
        g["lidar_dirs"] = R.rays.scan_pattern(16, 128).copy()
        # --- scene trace / distance / esdf lookup ------------------------------
        sd = R.sample_directions(256).directions.copy()
        g["scene_trace_dirs"] = sd
        g["scene_trace_t"] = R.raycast_many(scene, states[1].position, sd, 20.0, backend=be)
        rng = np.random.default_rng(11)
        pts = rng.uniform(scene.bounds.lo - 1.5, scene.bounds.hi + 1.5, size=(64, 3))
        g["esdf_pts"] = pts
        d, gr, fl = R.get_backend(be).esdf_sample_many(grid.values, grid.origin,
                                                       grid.resolution, pts)
        g["esdf_d"], g["esdf_g"], g["esdf_flag"] = d, gr, fl
        g["scene_dist"] = R.get_backend(be).scene_distance_many(pk, pts, 0.0)
        # --- pinv_psd KATs ----------------------------------------------------
        mats = np.array([np.diag([2.0, 1.0, 0.0]), np.zeros((3, 3)), np.eye(3) * 4,
                         np.outer([1.0, 2.0, 2.0], [1.0, 2.0, 2.0]), MET[0]])
        g["pinv_in"] = mats
        g["pinv_out"] = np.array([R.core.pinv_psd(m) for m in mats])
        # --- closed-loop rollouts (row f1): reference sim.rollout, ray planner ---
        import rmpnav.sim as S
        g["roll_start"], g["roll_goal"] = start, goal
        RB = []
        for k, (max_acc, n_rays) in enumerate(((40.0, 1024), (2.0, 512))):
            rcfg = S.RolloutConfig(planner=S.PlannerSpec("ray", n_rays=n_rays),
                                   params=R.preset("static_map"), dt=0.01, max_time=1.5,
                                   max_accel=max_acc, max_range=10.0, backend=be)
            tr = S.rollout(scene, start, goal, rcfg, grid=grid)
            g[f"roll{k}_pos"], g[f"roll{k}_vel"], g[f"roll{k}_acc"] = tr.positions, tr.velocities, tr.accels
            g[f"roll{k}_outcome"] = np.array(tr.outcome.value)
            g[f"roll{k}_nclamped"] = np.array(tr.n_clamped)
            g[f"roll{k}_dirs"] = R.sample_directions(n_rays).directions.copy()
            g[f"roll{k}_maxacc"] = np.array(max_acc)
        out = os.path.join(HERE, "rmpnav_golden.npz")
        np.savez_compressed(out, **g)
        print(f"wrote {out} ({os.path.getsize(out)} bytes)")


if __name__ == "__main__":
    main()
