"""GPU parity: the CUDA path through the C ABI vs the CPU oracle and the
reference's golden vectors.

Bars (BASELINE.json north_star):
  * hit distance t, hit/miss mask, hit cell, step count: BIT-EXACT;
  * n_hits: exact;
  * summed metric / weighted force: within 1e-9 relative of the oracle (the
    contract is 1e-5; only libm exp/log1p ulps and the reduction order
    differ), resolved acceleration within 1e-6 relative (pinv amplifies
    the sum error by cond(sum A) <= ~1e4 here).
"""

import numpy as np
import pytest

from conftest import LIDAR, STATIC_MAP, golden_pack, rel_err

pytestmark = pytest.mark.gpu

SUM_TOL = 1e-9
ACC_TOL = 1e-6


@pytest.fixture(scope="module")
def be():
    from paper_2301_08068_b200 import _lib
    from paper_2301_08068_b200._kernels import b200

    _lib.load()
    assert _lib.device_count() >= 1, "no CUDA device visible"
    return b200


@pytest.fixture(scope="module")
def gworld(be, golden):
    g = golden
    pack = golden_pack(g)
    vals = be.bake_values(pack, g["grid_origin"], float(g["grid_res"]), tuple(g["grid_dims"]))
    return pack, vals


@pytest.fixture(scope="module")
def c1(be, oracle):
    from paper_2301_08068_b200 import synth

    scene = synth.c1_scene()
    grid = synth.c1_grid(scene)
    states = synth.bench_states(scene, count=10, seed=123)
    dirs = oracle.sample_directions(65536)
    return scene, grid, states, dirs


def check_policy(slot, acc, slot_ref, acc_ref):
    assert slot[12] == slot_ref[12]
    assert rel_err(slot[:9], slot_ref[:9]) <= SUM_TOL
    assert rel_err(slot[9:12], slot_ref[9:12]) <= SUM_TOL
    assert rel_err(acc, acc_ref) <= ACC_TOL


# --- golden vectors (produced by running the reference) -----------------------

def test_gpu_bake_bit_exact_vs_reference(gworld, golden):
    import hashlib

    _, vals = gworld
    assert hashlib.sha256(vals.tobytes()).digest() == golden["grid_sha256_f64"].tobytes()


def test_fused_ray_policy_vs_golden(be, gworld, golden):
    g = golden
    vals = gworld[1].astype(np.float32).astype(np.float64)
    res = float(g["grid_res"])
    for k in range(g["pose_x"].shape[0]):
        slot, acc, t, cells, steps = be.ray_policy_fused(
            vals, g["grid_origin"], res, g["pose_x"][k], g["pose_v"][k], g["dirs"], STATIC_MAP,
            10.0, 0.5 * res, 0.9, with_rays=True)
        assert np.array_equal(t, g["trace_t"][k]), f"pose {k}: t differs"
        assert np.array_equal(np.isfinite(t), np.isfinite(g["trace_t"][k]))
        check_policy(slot, acc, g["slots"][k], g["accels"][k])
        assert rel_err(slot[:9].reshape(3, 3), g["metrics"][k]) <= SUM_TOL


def test_unfused_protocol_vs_golden(be, gworld, golden):
    g = golden
    vals = gworld[1].astype(np.float32).astype(np.float64)
    res = float(g["grid_res"])
    for k in (0, 3):
        t = be.grid_trace(vals, g["grid_origin"], res, g["pose_x"][k], g["dirs"], 10.0,
                          0.5 * res, 0.9)
        assert np.array_equal(t, g["trace_t"][k])
        m, w, n = be.policy_reduce(g["dirs"], t, g["pose_v"][k], STATIC_MAP, 0.0)
        assert n == int(g["slots"][k][12])
        assert rel_err(m.ravel(), g["slots"][k][:9]) <= SUM_TOL
        assert rel_err(w, g["slots"][k][9:12]) <= SUM_TOL


def test_f64_grid_trace_vs_golden(be, gworld, golden):
    g = golden
    vals = gworld[1]  # not f32-exact -> f64 storage
    res = float(g["grid_res"])
    grid = be.DeviceGrid(vals, g["grid_origin"], res)
    assert grid.storage == "f64"
    t = be.grid_trace(vals, g["grid_origin"], res, g["pose_x"][0], g["dirs"], 10.0, 0.5 * res, 0.9)
    assert np.array_equal(t, g["trace_t_f64grid"])


def test_public_api_vs_golden(be, gworld, golden):
    import paper_2301_08068_b200 as P

    g = golden
    vals = gworld[1].astype(np.float32).astype(np.float64)
    grid = P.EsdfGrid(g["grid_origin"], float(g["grid_res"]), tuple(g["grid_dims"]), vals)
    bundle = P.RayBundle(g["dirs"])
    p = P.preset("static_map").obstacle
    for k in range(g["pose_x"].shape[0]):
        pol = P.ray_policy(P.RobotState(g["pose_x"][k], g["pose_v"][k]), grid, bundle, p, 10.0)
        assert rel_err(pol.metric, g["metrics"][k]) <= SUM_TOL
        assert rel_err(pol.accel, g["accels"][k]) <= ACC_TOL
    acc, met, nh = P.ray_policy_batch((g["pose_x"], g["pose_v"]), grid, bundle, p, 10.0)
    assert np.array_equal(nh, g["slots"][:, 12].astype(np.int64))
    for k in range(len(nh)):
        assert rel_err(met[k], g["metrics"][k]) <= SUM_TOL
        assert rel_err(acc[k], g["accels"][k]) <= ACC_TOL


def test_lidar_vs_golden(be, golden):
    import paper_2301_08068_b200 as P

    g = golden
    lp = P.preset("lidar").obstacle
    for i in range(g["lidar_ranges"].shape[0]):
        R = g["lidar_rot"] if i == 1 else np.eye(3)
        scan = P.RangeScan(g["lidar_dirs"], g["lidar_ranges"][i], g["lidar_valid"][i],
                           g["pose_x"][i], R, 16, 128)
        pol = P.lidar_policy(g["pose_v"][i], scan, lp)
        assert rel_err(pol.metric, g["lidar_metrics"][i]) <= SUM_TOL
        assert rel_err(pol.accel, g["lidar_accels"][i]) <= ACC_TOL


def test_scene_esdf_pinv_vs_golden(be, gworld, golden):
    g = golden
    pack, vals = gworld
    t = be.scene_trace(pack, g["pose_x"][1], g["scene_trace_dirs"], 20.0, 1e-4, 0.0)
    assert np.array_equal(t, g["scene_trace_t"])
    assert np.array_equal(be.scene_distance_many(pack, g["esdf_pts"], 0.0), g["scene_dist"])
    d, gr, fl = be.esdf_sample_many(vals, g["grid_origin"], float(g["grid_res"]), g["esdf_pts"])
    assert np.array_equal(d, g["esdf_d"])
    assert np.allclose(gr, g["esdf_g"], rtol=0, atol=1e-15)
    assert np.array_equal(fl, g["esdf_flag"])
    out = be.pinv_psd(g["pinv_in"])
    for a, b in zip(out, g["pinv_out"]):
        assert rel_err(a, b) <= 1e-10 or np.abs(a - b).max() <= 1e-13


def test_spec_kats(be, golden):
    import paper_2301_08068_b200 as P

    sph = P.Scene(P.Aabb([-6, -6, -6], [6, 6, 6]), [P.Primitive.sphere((0, 0, 0), 1.0)])
    assert P.raycast(sph, (5, 0, 0), (-1, 0, 0)) == float(golden["kat_sphere_ray"]) == 4.0
    empty = P.Scene(P.Aabb([-6, -6, -6], [6, 6, 6]), [])
    assert np.isinf(P.raycast(empty, (0, 0, 0), (1, 0, 0)))
    d1 = P.sample_directions(1).directions
    assert np.allclose(d1, golden["kat_dir1"], rtol=0, atol=1e-15)


# --- full-size C1 (headline config) --------------------------------------------

def test_c1_full_size_bit_exact(be, oracle, c1):
    from paper_2301_08068_b200 import synth

    scene, grid, states, dirs = c1
    assert synth.grid_sha_prefix(grid) == synth.C1_SHA_PREFIX
    for st in states[:4]:
        slot, acc, t, cells, steps = be.ray_policy_fused(
            grid.values, grid.origin, grid.resolution, st.position, st.velocity, dirs, STATIC_MAP,
            10.0, 0.05, 0.9, with_rays=True)
        t_r, c_r, s_r = oracle.grid_trace(grid.values, grid.origin, grid.resolution, st.position,
                                          dirs, 10.0, 0.05, 0.9, with_cells=True, with_steps=True,
                                          workers=8)
        assert np.array_equal(t, t_r)
        assert np.array_equal(cells, c_r)
        assert np.array_equal(steps, s_r)
        slot_r = oracle.policy_slot(dirs, t_r, st.velocity, STATIC_MAP)
        check_policy(slot, acc, slot_r, oracle.accel_from_slot(slot_r))


def test_c1_batch_matches_single_and_oracle(be, oracle, c1):
    from paper_2301_08068_b200 import synth

    scene, grid, states, dirs = c1
    x, v = synth.states_arrays(states)
    slots, accs = be.ray_policy_batch(grid.values, grid.origin, grid.resolution, x, v, dirs,
                                      STATIC_MAP, 10.0, 0.05, 0.9)
    for k, st in enumerate(states):
        slot_r, acc_r, _ = oracle.ray_policy(grid.values, grid.origin, grid.resolution,
                                             st.position, st.velocity, dirs, STATIC_MAP, 10.0,
                                             workers=8)
        check_policy(slots[k], accs[k], slot_r, acc_r)
    # pose with an all-zero metric (SURVEY.md App. B pose 3): accel exactly 0
    assert slots[3][12] == 11597 and not slots[3][:12].any() and not accs[3].any()


def test_determinism_bitwise(be, c1):
    scene, grid, states, dirs = c1
    st = states[0]
    a = be.ray_policy_fused(grid.values, grid.origin, grid.resolution, st.position, st.velocity,
                            dirs, STATIC_MAP, 10.0, 0.05, 0.9)
    for _ in range(3):
        b = be.ray_policy_fused(grid.values, grid.origin, grid.resolution, st.position,
                                st.velocity, dirs, STATIC_MAP, 10.0, 0.05, 0.9)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_l2_window_on_off_bitwise(be, c1):
    """The map's L2 access-policy window (option l2_window, default on) only
    changes cache residency: results are bitwise those of a plain launch."""
    from paper_2301_08068_b200 import _lib as L

    scene, grid, states, dirs = c1
    st = states[2]
    outs = []
    try:
        for w in (1, 0, 1):
            L.call("rmpb_set_option", b"l2_window", w)
            outs.append(be.ray_policy_fused(grid.values, grid.origin, grid.resolution, st.position,
                                            st.velocity, dirs, STATIC_MAP, 10.0, 0.05, 0.9))
    finally:
        L.call("rmpb_set_option", b"l2_window", 1)
    for o in outs[1:]:
        assert np.array_equal(outs[0][0], o[0]) and np.array_equal(outs[0][1], o[1])
    with pytest.raises(ValueError):
        L.call("rmpb_set_option", b"l2_window", 2)


def test_layouts_and_storage_identical(be, oracle, c1):
    from paper_2301_08068_b200 import _lib as L

    scene, grid, states, dirs = c1
    st = states[1]
    sub = dirs[:8192]
    t_ref = oracle.grid_trace(grid.values, grid.origin, grid.resolution, st.position, sub, 10.0,
                              0.05, 0.9)
    variants = [dict(storage=L.STORE_F32, layout=L.LAYOUT_LINEAR),
                dict(storage=L.STORE_F32, layout=L.LAYOUT_QUAD),
                dict(storage=L.STORE_F32, layout=L.LAYOUT_PAIR64),
                dict(storage=L.STORE_F64, layout=L.LAYOUT_LINEAR),
                dict(storage=L.STORE_F64, layout=L.LAYOUT_PAIR64)]
    for kw in variants:
        dg = be.DeviceGrid(grid.values, grid.origin, grid.resolution, **kw)
        t, _, _ = be.grid_trace_ex(dg, grid.origin, grid.resolution, st.position, sub, 10.0,
                                   0.05, 0.9)
        assert np.array_equal(t, t_ref), kw


@pytest.mark.parametrize("dims,f64", [((64, 48, 40), False), ((61, 45, 37), False),
                                      ((9, 17, 10), False), ((61, 45, 37), True)])
def test_brick_grid_identical_to_dense(be, oracle, dims, f64):
    """Block-hashed TSDF: a truncated field whose far bricks are uniform
    +tau -- f32 apron-QUAD bricks (dims that are not multiples of 8: bricks
    clipped at the far faces) and f64 scalar bricks; node readback and the
    trace bit-identical to the dense oracle."""
    rng = np.random.default_rng(3)
    nx, ny, nz = dims
    res, tau = 0.05, 0.2
    ii, jj, kk = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    p = np.stack([ii, jj, kk], -1) * res
    ext = np.array(dims) * res
    c = np.array([1.5, 1.2, 1.0]) if nx >= 40 else 0.45 * ext
    rad = 0.6 if nx >= 40 else 0.3 * ext.min()
    sd = np.linalg.norm(p - c, axis=-1) - rad
    vals = np.clip(sd, -tau, tau)
    if not f64:
        vals = vals.astype(np.float32).astype(np.float64)
    fill = float(np.float32(tau)) if not f64 else tau
    dg = be.DeviceGrid(vals, np.zeros(3), res, brick_fill=fill)
    nb = ((nx + 7) // 8) * ((ny + 7) // 8) * ((nz + 7) // 8)
    assert dg.layout == "brick" and 0 < dg.bricks <= nb
    assert dg.storage == ("f64" if f64 else "f32")
    assert np.array_equal(dg.values(), vals)
    dirs = rng.normal(size=(4096, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    start = np.array([0.4, 0.4, 0.3]) if nx >= 40 else 0.1 * ext
    t, cells, _ = be.grid_trace_ex(dg, np.zeros(3), res, start, dirs, 5.0, 0.5 * res, 0.9,
                                   with_cells=True)
    t_r, c_r = oracle.grid_trace(vals, np.zeros(3), res, start, dirs, 5.0, 0.5 * res, 0.9,
                                 with_cells=True)
    assert np.array_equal(t, t_r) and np.array_equal(cells, c_r)
    assert np.isfinite(t).mean() > 0.01


# --- edge cases -------------------------------------------------------------------

def test_edge_cases(be, oracle):
    rng = np.random.default_rng(5)
    nx, ny, nz, res = 30, 20, 10, 0.1
    o = np.array([0.0, 0.0, 0.0])
    free = np.full((nx, ny, nz), 5.0)
    dirs = rng.normal(size=(3000, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    dirs[:40, 0] = 0.0
    dirs[40:80, 1] = 0.0
    dirs[80:120, 2] = 0.0
    dirs[120:130] = [1.0, 0.0, 0.0]
    # all rays miss -> zero policy
    slot, acc = be.ray_policy_fused(free, o, res, [1.0, 1.0, 0.5], [1, 0, 0], dirs, STATIC_MAP,
                                    10.0, 0.05, 0.9)
    assert not slot.any() and not acc.any()
    # start inside an obstacle -> every in-domain ray hits at t = 0
    solid = np.full((nx, ny, nz), -1.0)
    t = be.grid_trace(solid, o, res, [1.0, 1.0, 0.5], dirs, 10.0, 0.05, 0.9)
    assert (t == 0.0).all()
    # start outside the domain, directions with zero components
    vals = (rng.normal(size=(nx, ny, nz)) * 0.2 + 0.15).astype(np.float32).astype(np.float64)
    for start in ([-1.0, 0.5, 0.5], [1.5, 0.9, 0.45], [1.5, 5.0, 0.2], [3.0, 1.0, 0.5]):
        t, c, s = be.grid_trace_ex(vals, o, res, start, dirs, 10.0, 0.05, 0.9, True, True)
        t_r, c_r, s_r = oracle.grid_trace(vals, o, res, start, dirs, 10.0, 0.05, 0.9,
                                          with_cells=True, with_steps=True)
        assert np.array_equal(t, t_r) and np.array_equal(c, c_r) and np.array_equal(s, s_r)
    # empty inputs
    assert be.grid_trace(vals, o, res, [0.5, 0.5, 0.5], np.zeros((0, 3)), 10.0, 0.05, 0.9).size == 0
    m, w, n = be.policy_reduce(np.zeros((0, 3)), np.zeros(0), [1, 0, 0], STATIC_MAP)
    assert n == 0 and not m.any() and not w.any()
    # NaN / inf / below-min-range distances are skipped (not counted)
    d = np.array([np.nan, np.inf, 0.1, 0.5, 1.0])
    dd = dirs[:5]
    m, w, n = be.policy_reduce(dd, d, [0.3, 0.2, 0.1], LIDAR, 0.3)
    m_r, w_r, n_r = oracle.policy_reduce(dd, d, [0.3, 0.2, 0.1], LIDAR, 0.3)
    assert n == n_r == 2
    assert rel_err(m, m_r) <= SUM_TOL and rel_err(w, w_r) <= SUM_TOL


def test_odd_sizes_and_segmentation(be, oracle, c1):
    """Ray counts that are not multiples of the CTA width, and forced
    segmentation variants, give identical traces and equal sums."""
    from paper_2301_08068_b200 import _lib

    scene, grid, states, dirs = c1
    st = states[2]
    for n in (1, 31, 257, 5000):
        sub = np.ascontiguousarray(dirs[:n])
        slot, acc, t, _, _ = be.ray_policy_fused(grid.values, grid.origin, grid.resolution,
                                                 st.position, st.velocity, sub, STATIC_MAP, 10.0,
                                                 0.05, 0.9, with_rays=True)
        t_r = oracle.grid_trace(grid.values, grid.origin, grid.resolution, st.position, sub, 10.0,
                                0.05, 0.9)
        assert np.array_equal(t, t_r)
        slot_r = oracle.policy_slot(sub, t_r, st.velocity, STATIC_MAP)
        check_policy(slot, acc, slot_r, oracle.accel_from_slot(slot_r))
    base = be.ray_policy_fused(grid.values, grid.origin, grid.resolution, st.position,
                               st.velocity, dirs, STATIC_MAP, 10.0, 0.05, 0.9)
    try:
        for sr in (256, 4096, 65536):
            _lib.set_option("seg_rays", sr)
            s2 = be.ray_policy_fused(grid.values, grid.origin, grid.resolution, st.position,
                                     st.velocity, dirs, STATIC_MAP, 10.0, 0.05, 0.9)
            check_policy(s2[0], s2[1], base[0], base[1])
    finally:
        _lib.set_option("seg_rays", 0)


def test_lidar_points_and_batch(be, oracle, c1):
    import paper_2301_08068_b200 as P
    from paper_2301_08068_b200 import synth

    scene, grid, states, dirs = c1
    scans = synth.lidar_scans(scene, states[:3], 32, 256)
    lp = P.preset("lidar").obstacle
    for st, sc in zip(states[:3], scans):
        wd = sc.world_directions()
        slot_r, acc_r = oracle.lidar_policy(wd, sc.ranges, sc.valid, st.velocity, LIDAR, 0.3)
        pol = P.lidar_policy(st.velocity, sc, lp)
        assert rel_err(pol.metric.ravel(), slot_r[:9]) <= SUM_TOL
        assert rel_err(pol.accel, acc_r) <= ACC_TOL
        # raw points: p = dir * range (f32), invalid beams -> zero points
        pts = np.where(sc.valid[:, None], sc.directions * sc.ranges[:, None], 0.0)
        pts32 = pts.astype(np.float32)
        pol2 = P.lidar_policy_points(st.velocity, pts32, lp)
        p64 = pts32.astype(np.float64)
        r = np.sqrt((p64 * p64).sum(1))
        with np.errstate(invalid="ignore", divide="ignore"):
            dd = p64 / r[:, None]
        ok = r > 0
        slot_p, acc_p = oracle.lidar_policy(np.where(ok[:, None], dd, 0.0), r, ok, st.velocity,
                                            LIDAR, 0.3)
        assert rel_err(pol2.metric.ravel(), slot_p[:9]) <= 1e-7
        assert rel_err(pol2.accel, acc_p) <= 1e-5
    acc_b, met_b, nh_b = P.lidar_policy_batch([s.velocity for s in states[:3]], scans, lp)
    for k, (st, sc) in enumerate(zip(states[:3], scans)):
        slot_r, acc_r = oracle.lidar_policy(sc.world_directions(), sc.ranges, sc.valid,
                                            st.velocity, LIDAR, 0.3)
        assert nh_b[k] == int(slot_r[12])
        assert rel_err(met_b[k].ravel(), slot_r[:9]) <= SUM_TOL
        assert rel_err(acc_b[k], acc_r) <= ACC_TOL


def test_ray_split_partials_fold(be, c1):
    """Config C5 mechanics: ray ranges of one pose -> per-range slots ->
    fixed-order fold + pinv on device == the whole-pose evaluation."""
    import torch

    from paper_2301_08068_b200.device import RayPolicyEngine

    scene, grid, states, dirs = c1
    st = states[0]
    eng = RayPolicyEngine(grid, dirs, STATIC_MAP, 10.0, device=0)
    x = torch.tensor(st.position, dtype=torch.float64, device="cuda")
    v = torch.tensor(st.velocity, dtype=torch.float64, device="cuda")
    whole_s, whole_a = eng.evaluate(x.view(1, 3), v.view(1, 3))
    n = eng.n_rays
    edges = [0, n // 8, n // 3, n // 2, n]
    parts = torch.stack([eng.partial(x, v, a, b) for a, b in zip(edges[:-1], edges[1:])])
    s, a = eng.resolve(parts)
    torch.cuda.synchronize()
    check_policy(s.cpu().numpy(), a.cpu().numpy(), whole_s[0].cpu().numpy(),
                 whole_a[0].cpu().numpy())


def test_device_halton_close_to_reference(be, oracle):
    import paper_2301_08068_b200 as P

    n = 65536
    d = P.sample_directions(n).directions
    r = oracle.sample_directions(n)
    assert d.shape == r.shape
    assert np.abs(d - r).max() <= 1e-15  # libdevice vs NumPy SIMD trig: a few ulp
    assert np.allclose(np.linalg.norm(d, axis=1), 1.0, atol=1e-12)


@pytest.mark.parametrize("rows,cols,vfov", [(128, 1024, 45.0), (1, 360, 45.0), (7, 5, 30.0),
                                             (64, 2048, 22.5)])
def test_device_lattice_close_to_reference(be, oracle, rows, cols, vfov):
    """Spherical-grid (LiDAR lattice) bundle generated on device vs the
    reference's scan_pattern (rays.py:176-199, NumPy trig: a few ulp), and a
    LiDAR policy on the device lattice vs the oracle on NumPy's lattice."""
    from paper_2301_08068_b200 import _lib as L

    b = be.DeviceBundle(lattice=(rows, cols, vfov), order=L.ORDER_IDENTITY)
    d = b.directions()
    r = oracle.scan_pattern(rows, cols, vfov)
    assert d.shape == r.shape == (rows * cols, 3)
    assert np.abs(d - r).max() <= 1e-15
    rng = np.random.default_rng(rows * cols)
    ranges = rng.uniform(0.0, 3.0, rows * cols)
    valid = rng.random(rows * cols) < 0.7
    v = np.array([0.4, -0.7, 0.2])
    slot = np.empty(13)
    acc = np.empty(3)
    vl = valid.astype(np.uint8)  # keep the temporaries alive across the call
    prm = np.asarray(LIDAR, dtype=np.float64)
    L.call("rmpb_lidar_policy_bundle", b.handle, None, ranges.ctypes.data, vl.ctypes.data,
           v.ctypes.data, prm.ctypes.data, 0.3, slot.ctypes.data, acc.ctypes.data, None)
    slot_r, acc_r = oracle.lidar_policy(r, ranges, valid, v, LIDAR, 0.3)
    assert slot[12] == slot_r[12]
    assert rel_err(slot[:12], slot_r[:12]) <= 1e-9
    with pytest.raises(ValueError):
        be.DeviceBundle(lattice=(0, 5, 45.0))


def test_tsdf_bake_bricks_and_readback(be, oracle):
    """Truncated (TSDF) GPU bake: brick-culled bake == clamp of the full
    oracle bake; BRICK / QUAD / LINEAR layouts read back the same nodes and
    trace bit-identically to the oracle on the dense values."""
    from paper_2301_08068_b200 import _lib as L, synth

    scene = synth.c1_scene(n_boxes=60, seed=4, hi=np.array([6.35, 4.75, 3.15]))
    dims, res, tau = (128, 96, 64), 0.05, 0.2
    ds = be.device_scene(scene.packed())
    brick = be.DeviceGrid.bake_tsdf(ds, np.zeros(3), res, dims, tau, storage=L.STORE_F32,
                                    layout=L.LAYOUT_BRICK)
    quad = be.DeviceGrid.bake_tsdf(ds, np.zeros(3), res, dims, tau, storage=L.STORE_F32,
                                   layout=L.LAYOUT_QUAD)
    full = oracle.bake_values(scene.packed(), np.zeros(3), res, dims, workers=8)
    want = np.clip(full, -tau, tau).astype(np.float32).astype(np.float64)
    vb, vq = brick.values(), quad.values()
    assert np.array_equal(vb, want) and np.array_equal(vq, want)
    assert 0 < brick.bricks < np.prod([(d + 7) // 8 for d in dims])
    lin = be.DeviceGrid(want, np.zeros(3), res, layout=L.LAYOUT_LINEAR)
    assert np.array_equal(lin.values(), want)
    rng = np.random.default_rng(9)
    dirs = rng.normal(size=(8192, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    start = np.array([3.1, 2.2, 1.5])
    t_r, c_r = oracle.grid_trace(want, np.zeros(3), res, start, dirs, 6.0, 0.5 * res, 0.9,
                                 with_cells=True)
    for g in (brick, quad, lin):
        t, c, _ = be.grid_trace_ex(g, np.zeros(3), res, start, dirs, 6.0, 0.5 * res, 0.9,
                                   with_cells=True)
        assert np.array_equal(t, t_r) and np.array_equal(c, c_r)
    # fused policy on the brick map == oracle
    v = np.array([0.5, -0.4, 0.2])
    slot, acc = be.ray_policy_fused(brick, np.zeros(3), res, start, v, dirs, STATIC_MAP, 6.0,
                                    0.5 * res, 0.9)
    slot_r = oracle.policy_slot(dirs, t_r, v, STATIC_MAP)
    check_policy(slot, acc, slot_r, oracle.accel_from_slot(slot_r))


def _golden_scene(g):
    import paper_2301_08068_b200 as P

    prims = []
    for k, o, c, s_, v in zip(g["scene_kinds"], g["scene_ops"], g["scene_centers"],
                              g["scene_sizes"], g["scene_velocities"]):
        kind = "sphere" if k == 0 else "box"
        size = s_[0] if kind == "sphere" else s_
        prims.append(P.Primitive(kind, c, size, "union" if o == 0 else "subtract", v))
    lo, hi = g["scene_bounds"]
    return P.Scene(P.Aabb(lo, hi), prims)


@pytest.mark.parametrize("policy_only", [False, True])
def test_batched_rollout_vs_reference_golden(be, gworld, golden, policy_only):
    """Row f1: closed-loop rollouts on device reproduce the reference's
    sim.rollout trajectories (ray planner): outcome, clamp count, every
    (x, v, command) sample of the trajectory -- also with the opt-in
    policy_only rays (stopped at the activation radius: the same policy up
    to the summation order)."""
    import paper_2301_08068_b200 as P
    from paper_2301_08068_b200.rollout import BatchRolloutConfig, RolloutBatch

    g = golden
    scene = _golden_scene(g)
    pack, vals = gworld
    grid = P.EsdfGrid(g["grid_origin"], float(g["grid_res"]), tuple(g["grid_dims"]), vals)
    for k in (0, 1):
        cfg = BatchRolloutConfig(params=P.preset("static_map"), dt=0.01, max_time=1.5,
                                 max_accel=float(g[f"roll{k}_maxacc"]), max_range=10.0,
                                 policy_only=policy_only)
        n_rec = g[f"roll{k}_pos"].shape[0] - 1
        # 3 identical robots: lockstep batches must not interfere
        starts = np.repeat(g["roll_start"][None], 3, axis=0)
        goals = np.repeat(g["roll_goal"][None], 3, axis=0)
        rb = RolloutBatch(scene, grid, P.RayBundle(g[f"roll{k}_dirs"]), starts, goals, cfg,
                          record_ticks=n_rec)
        rb.run()
        res = rb.result()
        for r in range(3):
            assert res.outcome[r] == str(g[f"roll{k}_outcome"])
            assert res.n_clamped[r] == int(g[f"roll{k}_nclamped"])
            assert res.steps[r] == n_rec
            tr = res.trajectory[r]
            assert np.abs(tr[:, 0:3] - g[f"roll{k}_pos"]).max() < 1e-9
            assert np.abs(tr[:, 3:6] - g[f"roll{k}_vel"]).max() < 1e-8
            assert np.abs(tr[:, 6:9] - g[f"roll{k}_acc"]).max() < 1e-6 * max(
                1.0, np.abs(g[f"roll{k}_acc"]).max())


def test_rollout_graph_replay_bitwise(be, c1):
    """Closed-loop ticks replayed from a captured CUDA graph (16 ticks per
    graph launch, option "graphs") give bitwise the eager ticks' states."""
    import paper_2301_08068_b200 as P
    from paper_2301_08068_b200 import _lib as L
    from paper_2301_08068_b200.rollout import BatchRolloutConfig, RolloutBatch

    scene, grid, states, dirs = c1
    starts = np.stack([s.position for s in states[:6]])
    goals = starts[::-1].copy()
    cfg = BatchRolloutConfig(params=P.preset("static_map"), dt=0.02, max_time=2.0,
                             max_accel=20.0, max_range=10.0)
    outs = []
    try:
        for gr in (0, 1):
            L.call("rmpb_set_option", b"graphs", gr)
            rb = RolloutBatch(scene, grid, P.RayBundle(dirs[:8192]), starts, goals, cfg)
            for _ in range(3):  # partial runs: eager head, graph chunks, eager tail
                rb.run(37)
            outs.append(rb.result())
    finally:
        L.call("rmpb_set_option", b"graphs", 1)
    a, b = outs
    assert list(a.outcome) == list(b.outcome)
    assert np.array_equal(a.steps, b.steps) and np.array_equal(a.n_clamped, b.n_clamped)
    assert np.array_equal(a.positions, b.positions)
    assert np.array_equal(a.velocities, b.velocities)
    assert a.steps.max() > 32


def test_k5_dda_bit_exact_vs_cpu_definition(be, oracle, c1):
    """K5 (north_star's DDA over occupancy; not reference parity): occupancy
    bits, entry distances (float32 bits) and hit voxel indices equal the CPU
    definition oracle/rmp_oracle.c orc_dda_trace, and every hit voxel is
    occupied."""
    import torch

    from paper_2301_08068_b200.device import DdaPolicyEngine

    scene, grid, states, dirs = c1
    dg = be.DeviceGrid(grid.values, grid.origin, grid.resolution)
    occ = be.DeviceOccupancy(dg)
    bits_ref = oracle.occupancy_bits(grid.values)
    assert np.array_equal(occ.bits(), bits_ref)
    for st in states[:3]:
        t, vox, steps = occ.trace(st.position, dirs, 10.0)
        t_r, vox_r, steps_r = oracle.dda_trace(grid.values, grid.origin, grid.resolution,
                                               st.position, dirs, 10.0, workers=8, bits=bits_ref)
        assert np.array_equal(t.view(np.uint32), t_r.view(np.uint32))
        assert np.array_equal(vox, vox_r) and np.array_equal(steps, steps_r)
        h = np.isfinite(t)
        assert (grid.values[vox[h, 0], vox[h, 1], vox[h, 2]] <= 0.0).all()
    # edge directions / outside starts on a random grid
    rng = np.random.default_rng(2)
    vals = rng.normal(size=(37, 21, 70)) + 1.2
    dirs2 = rng.normal(size=(3000, 3))
    dirs2 /= np.linalg.norm(dirs2, axis=1, keepdims=True)
    dirs2[:50, 0] = 0.0
    dirs2[50:100, 1] = 0.0
    dirs2[100:150, 2] = 0.0
    g2 = be.DeviceGrid(vals, np.array([-0.3, 0.2, 0.1]), 0.07)
    occ2 = be.DeviceOccupancy(g2)
    for start in ([0.5, 0.8, 2.0], [-2.0, 0.9, 2.5], [1.0, 5.0, -1.0]):
        t, vox, steps = occ2.trace(start, dirs2, 4.0)
        t_r, vox_r, steps_r = oracle.dda_trace(vals, [-0.3, 0.2, 0.1], 0.07, start, dirs2, 4.0)
        assert np.array_equal(t.view(np.uint32), t_r.view(np.uint32))
        assert np.array_equal(vox, vox_r) and np.array_equal(steps, steps_r)
    # fused DDA policy == oracle policy on the DDA distances
    eng = DdaPolicyEngine(dg, dirs, STATIC_MAP, 10.0)
    x = torch.tensor(np.stack([s.position for s in states[:4]]), dtype=torch.float64, device="cuda")
    v = torch.tensor(np.stack([s.velocity for s in states[:4]]), dtype=torch.float64, device="cuda")
    slots, accs = eng.evaluate(x, v)
    slots, accs = slots.cpu().numpy(), accs.cpu().numpy()
    for k, st in enumerate(states[:4]):
        t_r, _, _ = oracle.dda_trace(grid.values, grid.origin, grid.resolution, st.position, dirs,
                                     10.0, workers=8, bits=bits_ref)
        slot_r = oracle.policy_slot(dirs, t_r.astype(np.float64), st.velocity, STATIC_MAP)
        check_policy(slots[k], accs[k], slot_r, oracle.accel_from_slot(slot_r))


def test_fast_mode_deviation_report(be, oracle, c1):
    """Opt-in FAST mode (fp32 march) is NOT reference-exact; its deviation
    from the exact path on the C1 poses is bounded and reported here."""
    import torch

    from paper_2301_08068_b200.device import RayPolicyEngine

    scene, grid, states, dirs = c1
    x = torch.tensor(np.stack([s.position for s in states]), dtype=torch.float64, device="cuda")
    v = torch.tensor(np.stack([s.velocity for s in states]), dtype=torch.float64, device="cuda")
    ex = RayPolicyEngine(grid, dirs, STATIC_MAP, 10.0)
    fa = RayPolicyEngine(ex.grid, ex.bundle, STATIC_MAP, 10.0, mode="fast")
    se, ae = (t.cpu().numpy() for t in ex.evaluate(x, v))
    sf, af = (t.cpu().numpy() for t in fa.evaluate(x, v))
    hit_dev = np.abs(sf[:, 12] - se[:, 12]).max() / 65536
    sum_dev = max(rel_err(sf[k, :12], se[k, :12]) for k in range(len(states)))
    print(f"FAST vs EXACT: max |n_hits diff| / rays = {hit_dev:.2e}, max sum rel dev = {sum_dev:.2e}")
    assert hit_dev < 1e-3
    assert sum_dev < 1e-2


def test_public_map_and_scan_entry_points_vs_golden(be, golden):
    """bake_esdf / esdf_policy / synthesize_scan / grid update / device-resident
    grid creation through the public API, against the reference goldens."""
    import hashlib

    import torch

    import paper_2301_08068_b200 as P
    from paper_2301_08068_b200 import _lib as L

    g = golden
    scene = _golden_scene(g)
    grid = P.bake_esdf(scene, 0.2, pad=1.0)
    assert hashlib.sha256(grid.values.tobytes()).digest() == g["grid_sha256_f64"].tobytes()
    assert grid.dims == tuple(g["grid_dims"]) and np.array_equal(grid.origin, g["grid_origin"])
    # synthesize_scan (analytic scene trace on device + seeded dropout)
    rot = g["lidar_rot"]
    for i in range(g["lidar_ranges"].shape[0]):
        sc = P.synthesize_scan(scene, g["pose_x"][i], 16, 128, max_range=20.0,
                               orientation=rot if i == 1 else None, dropout=0.1, rng=i)
        assert np.array_equal(sc.valid, g["lidar_valid"][i])
        assert np.array_equal(sc.ranges, g["lidar_ranges"][i])
    # esdf_policy: one lookup + obstacle_ray_policy (policies.py:166-172)
    st = P.RobotState(g["esdf_pts"][3], [0.2, -0.4, 0.1])
    pol = P.esdf_policy(st, grid, P.preset("static_map").obstacle)
    d, gr = g["esdf_d"][3], g["esdf_g"][3]
    want = (P.Policy.zero() if not gr.any() else
            P.obstacle_ray_policy(st.velocity, gr, d, P.preset("static_map").obstacle))
    assert np.allclose(pol.accel, want.accel, rtol=1e-12, atol=1e-12)
    assert np.allclose(pol.metric, want.metric, rtol=1e-12, atol=1e-12)
    # grid update + device-resident creation trace like the oracle
    vals32 = grid.values.astype(np.float32).astype(np.float64)
    dg = be.DeviceGrid(grid.values, grid.origin, grid.resolution)
    L.call("rmpb_grid_update", dg.handle, vals32.ctypes.data, L.RMPB_F64)
    t1, _, _ = be.grid_trace_ex(dg, grid.origin, grid.resolution, g["pose_x"][0], g["dirs"], 10.0,
                                0.1, 0.9)
    assert np.array_equal(t1, g["trace_t"][0])
    tens = torch.from_numpy(vals32).cuda()
    dd = be.DeviceGrid.from_device(tens.data_ptr(), False, grid.dims, grid.origin, grid.resolution)
    t2, _, _ = be.grid_trace_ex(dd, grid.origin, grid.resolution, g["pose_x"][0], g["dirs"], 10.0,
                                0.1, 0.9)
    assert np.array_equal(t2, g["trace_t"][0])


def test_lidar_points_batch_device(be, oracle, c1):
    import torch

    from paper_2301_08068_b200 import synth
    from paper_2301_08068_b200.device import lidar_points_batch_device

    scene, grid, states, dirs = c1
    scans = synth.lidar_scans(scene, states[:4], 16, 256)
    pts = np.stack([np.where(s.valid[:, None], s.directions * s.ranges[:, None], 0.0)
                    for s in scans]).astype(np.float32)
    v = np.stack([s.velocity for s in states[:4]])
    slots, accs = lidar_points_batch_device(torch.from_numpy(pts).cuda(), None,
                                            torch.from_numpy(v).cuda(), LIDAR, 0.3)
    slots, accs = slots.cpu().numpy(), accs.cpu().numpy()
    for k in range(4):
        p64 = pts[k].astype(np.float64)
        r = np.sqrt((p64 * p64).sum(1))
        ok = r > 0
        with np.errstate(invalid="ignore", divide="ignore"):
            dd = np.where(ok[:, None], p64 / r[:, None], 0.0)
        slot_r, acc_r = oracle.lidar_policy(dd, r, ok, v[k], LIDAR, 0.3)
        assert slots[k][12] == slot_r[12]
        assert rel_err(slots[k][:12], slot_r[:12]) <= 1e-7
        assert rel_err(accs[k], acc_r) <= 1e-5


# LiDAR warp-unit decompositions: the default target (many short units,
# multi-unit fold per scan), 1000 and 3 units per launch (long units: many
# 128-beam groups per warp, ring wrap-around)
LIDAR_WARP_TARGETS = (38000, 1000, 3)


@pytest.mark.parametrize("n,S", [(131072, 1), (1000, 5), (131, 3), (97, 2), (4096, 40), (8192, 3)])
def test_lidar_kernels_ragged_and_misaligned(be, oracle, n, S):
    """The LiDAR kernel at every unit decomposition (LIDAR_WARP_TARGETS) vs the oracle on ragged beam counts, odd rows (16-B misaligned
    range rows / 4-B misaligned validity rows -> scalar path), with and
    without rotation / validity; variant 3 with the default warp targets
    also exercises the multi-warp fold (S = 1: 512 warp partials)."""
    import torch

    from paper_2301_08068_b200 import _lib
    from paper_2301_08068_b200.device import lidar_policy_batch_device

    rng = np.random.default_rng(n * 7 + S)
    dirs = rng.standard_normal((n, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    ranges = rng.uniform(0.0, 4.0, (S, n))
    ranges[:, ::17] = np.inf
    ranges[:, 3::29] = np.nan
    valid = rng.random((S, n)) < 0.8
    v = rng.standard_normal((S, 3))
    Rs = []
    for _ in range(S):
        q, _r = np.linalg.qr(rng.standard_normal((3, 3)))
        Rs.append(q)
    Rs = np.stack(Rs)
    d_dirs = torch.from_numpy(dirs).cuda()
    d_rg = torch.from_numpy(ranges).cuda()
    d_v = torch.from_numpy(v).cuda()
    try:
        for use_R in (True, False):
            for use_valid in (True, False):
                d_R = torch.from_numpy(Rs.reshape(S, 9).copy()).cuda() if use_R else None
                d_vl = torch.from_numpy(valid.astype(np.uint8)).cuda() if use_valid else None
                outs = {}
                for k in LIDAR_WARP_TARGETS:
                    _lib.call("rmpb_set_option", b"lidar_warps", k)
                    got = []
                    for persist in (1, 0):  # persistent warps claiming units / one unit per warp
                        _lib.call("rmpb_set_option", b"lidar_persist", persist)
                        sl, ac = lidar_policy_batch_device(d_dirs, d_R, d_rg, d_vl, d_v, LIDAR, 0.3)
                        got.append((sl.cpu().numpy(), ac.cpu().numpy()))
                    _lib.call("rmpb_set_option", b"lidar_persist", 1)
                    assert np.array_equal(got[0][0], got[1][0], equal_nan=True)  # same units
                    assert np.array_equal(got[0][1], got[1][1], equal_nan=True)
                    outs[k] = got[0]
                for s in range(S):
                    wd = dirs @ Rs[s].T if use_R else dirs
                    vv = valid[s] if use_valid else np.ones(n, bool)
                    slot_r, acc_r = oracle.lidar_policy(wd, ranges[s], vv, v[s], LIDAR, 0.3)
                    for k in LIDAR_WARP_TARGETS:
                        sl, ac = outs[k]
                        assert sl[s][12] == slot_r[12], (k, s)
                        assert rel_err(sl[s][:12], slot_r[:12]) <= SUM_TOL, (k, s)
                        if slot_r[12] > 0 and np.abs(slot_r[:9]).max() > 0:
                            assert rel_err(ac[s], acc_r) <= ACC_TOL, (k, s)
    finally:
        _lib.call("rmpb_set_option", b"lidar_warps", 38000)
        _lib.call("rmpb_set_option", b"lidar_persist", 1)


@pytest.mark.parametrize("n,S", [(131072, 1), (1001, 4), (131, 3), (4096, 6)])
def test_lidar_points_kernels_ragged(be, oracle, n, S):
    """Raw-point kernels (1: per-thread, 3: warp units) vs the oracle on
    ragged / misaligned rows (12-B points: odd n -> scalar path), zero and
    non-finite points, with and without rotation."""
    import torch

    from paper_2301_08068_b200 import _lib
    from paper_2301_08068_b200.device import lidar_points_batch_device

    rng = np.random.default_rng(n + 11 * S)
    pts = rng.uniform(-3.0, 3.0, (S, n, 3)).astype(np.float32)
    pts[:, ::13] = 0.0
    pts[:, 5::31, 1] = np.nan
    v = rng.standard_normal((S, 3))
    Rs = np.stack([np.linalg.qr(rng.standard_normal((3, 3)))[0] for _ in range(S)])
    try:
        for use_R in (True, False):
            d_R = torch.from_numpy(Rs.reshape(S, 9).copy()).cuda() if use_R else None
            outs = {}
            for k in LIDAR_WARP_TARGETS:
                _lib.call("rmpb_set_option", b"lidar_warps", k)
                sl, ac = lidar_points_batch_device(torch.from_numpy(pts).cuda(), d_R,
                                                   torch.from_numpy(v).cuda(), LIDAR, 0.3)
                outs[k] = (sl.cpu().numpy(), ac.cpu().numpy())
            for s in range(S):
                p64 = pts[s].astype(np.float64)
                r = np.sqrt((p64 * p64).sum(1))
                ok = r > 0
                with np.errstate(invalid="ignore", divide="ignore"):
                    dd = np.where(ok[:, None], p64 / r[:, None], 0.0)
                wd = dd @ Rs[s].T if use_R else dd
                slot_r, acc_r = oracle.lidar_policy(wd, r, ok, v[s], LIDAR, 0.3)
                for k in LIDAR_WARP_TARGETS:
                    sl, ac = outs[k]
                    assert sl[s][12] == slot_r[12], (k, s)
                    assert rel_err(sl[s][:12], slot_r[:12]) <= SUM_TOL, (k, s)
    finally:
        _lib.call("rmpb_set_option", b"lidar_warps", 38000)
        _lib.call("rmpb_set_option", b"lidar_persist", 1)


# --- host fast path: repeated calls with the same arrays -----------------------

def test_public_ray_policy_repeated_and_map_edits(be, oracle):
    """The control-loop pattern: the same EsdfGrid / RayBundle objects every
    call (identity cache), then map edits through EsdfGrid.update -- a
    single node (patched in place on the device), a box of obstacle nodes,
    and values that are not f32-exact (the f32 device copy cannot hold them:
    re-uploaded) -- each seen by the very next call; the in-place write to
    EsdfGrid.values itself raises (read-only)."""
    import time

    import paper_2301_08068_b200 as P
    from paper_2301_08068_b200 import synth

    scene = synth.c1_scene(n_boxes=20, hi=np.array([5.9, 5.9, 2.9]))
    vals = be.bake_values(scene.packed(), np.zeros(3), 0.1, (60, 60, 30))
    vals = vals.astype(np.float32).astype(np.float64)
    grid = P.EsdfGrid(np.zeros(3), 0.1, (60, 60, 30), vals)
    dirs = oracle.sample_directions(4096)
    bundle = P.RayBundle(dirs)
    params = P.preset("static_map").obstacle
    st = synth.bench_states(scene, count=1, seed=5, distance=synth.host_box_distance(scene))[0]

    def check():
        ref = oracle.ray_policy(grid.values, grid.origin, 0.1, st.position, st.velocity, dirs,
                                params.as_tuple(), 10.0)
        pol = P.ray_policy(st, grid, bundle, params, 10.0)
        assert rel_err(pol.metric, ref[0][:9].reshape(3, 3)) <= SUM_TOL
        assert rel_err(pol.accel, ref[1]) <= ACC_TOL
        t = be.grid_trace(grid.values, grid.origin, 0.1, st.position, dirs, 10.0, 0.05, 0.9)
        t_r = oracle.grid_trace(grid.values, grid.origin, 0.1, st.position, dirs, 10.0, 0.05, 0.9)
        assert np.array_equal(t, t_r)
        return pol

    p0 = check()
    for _ in range(2):
        check()
    # identity fast path of the map lookup stays cheap
    be.device_grid(grid.values, grid.origin, 0.1)
    t0 = time.perf_counter()
    for _ in range(200):
        be.device_grid(grid.values, grid.origin, 0.1)
    assert (time.perf_counter() - t0) / 200 < 5e-6
    with pytest.raises(ValueError):
        grid.values[1, 1, 1] = 0.0
    # one node of the pose's own cell (every ray's first interpolation),
    # patched in place on the device
    i, j, kk = (int(c) for c in np.floor(st.position / 0.1))
    grid.update((i + 1, j, kk), -0.5)
    p1 = check()
    assert not np.array_equal(p1.metric, p0.metric)
    grid.update((slice(i - 2, i + 3), slice(j - 2, j + 3), slice(kk - 1, kk + 2)), -0.25)
    p2 = check()
    assert not np.array_equal(p2.metric, p1.metric)
    grid.update((slice(i, i + 2), j, kk), 0.1234567890123)  # not f32-exact
    check()


def test_concurrent_host_threads_bitwise(be, c1):
    """The C ABI is thread-safe (per-(device, stream) workspaces, each behind
    its own lock): host threads calling the public ray_policy / lidar_policy
    concurrently get bitwise the results of sequential calls."""
    from concurrent.futures import ThreadPoolExecutor

    import paper_2301_08068_b200 as P

    scene, grid, states, dirs = c1
    esdf = grid if isinstance(grid, P.EsdfGrid) else P.EsdfGrid(
        grid.origin, grid.resolution, grid.values.shape, grid.values)
    bundle = P.RayBundle(dirs)
    params = P.preset("static_map").obstacle
    seq = [P.ray_policy(st, esdf, bundle, params, 10.0) for st in states]

    def one(k):
        pol = P.ray_policy(states[k % len(states)], esdf, bundle, params, 10.0)
        return k % len(states), pol

    with ThreadPoolExecutor(max_workers=6) as ex:
        for k, pol in ex.map(one, range(48)):
            assert np.array_equal(pol.metric, seq[k].metric)
            assert np.array_equal(pol.accel, seq[k].accel)


def test_c5_full_size_properties(be, oracle):
    """Config C5 at its full size (1000x1000x200 TSDF @0.05 m, 1 M rays per
    pose): size-independent properties.  The block-hashed map evaluates
    bitwise like the dense one; the 8-way ray split folds to the whole pose's
    result (hit count exact, sums to 1e-12); a 2048-ray sample traces
    bit-identically to the CPU oracle on the read-back node values."""
    import torch

    from paper_2301_08068_b200 import synth
    from paper_2301_08068_b200.device import RayPolicyEngine
    from paper_2301_08068_b200.parallel import balanced_range

    scene = synth.c5_scene()
    dense, brick, info = synth.c5_grids(scene)
    assert 0 < info["bricks_allocated"] < info["bricks_total"]
    states = synth.bench_states(scene, count=2, seed=123, distance=synth.host_box_distance(scene))
    n = 1 << 20
    bundle = be.DeviceBundle(halton_n=n)
    x = torch.tensor(np.stack([s.position for s in states]), dtype=torch.float64, device="cuda")
    v = torch.tensor(np.stack([s.velocity for s in states]), dtype=torch.float64, device="cuda")
    outs = []
    for dg in (dense, brick):
        eng = RayPolicyEngine(dg, bundle, STATIC_MAP, 10.0)
        s, a = eng.evaluate(x, v)
        outs.append((s.cpu().numpy(), a.cpu().numpy(), eng))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    eng = outs[1][2]
    x1, v1 = x[0].contiguous(), v[0].contiguous()
    parts = torch.stack([eng.partial(x1, v1, *balanced_range(n, 8, r)) for r in range(8)])
    ss, sa = eng.resolve(parts)
    ss, sa = ss.cpu().numpy(), sa.cpu().numpy()
    whole = outs[1][0][0]
    assert ss[12] == whole[12] > 0
    assert rel_err(ss[:12], whole[:12]) <= 1e-12
    vals = brick.values()
    samp = np.ascontiguousarray(oracle.sample_directions(2048))
    t, c, _ = be.grid_trace_ex(brick, synth.C5_ORIGIN, synth.C5_RES, states[0].position, samp,
                               10.0, 0.5 * synth.C5_RES, 0.9, with_cells=True)
    t_r, c_r = oracle.grid_trace(vals, synth.C5_ORIGIN, synth.C5_RES, states[0].position, samp,
                                 10.0, 0.5 * synth.C5_RES, 0.9, with_cells=True, workers=8)
    assert np.array_equal(t, t_r) and np.array_equal(c, c_r)
    assert np.isfinite(t).mean() > 0.3


@pytest.mark.parametrize("n,S", [(131072, 2), (4096, 8), (131, 3)])
def test_lidar_fast_mode_within_north_star_tolerance(be, oracle, n, S):
    """Opt-in LiDAR mode="fast" (per-beam policy math in fp32, fp64
    accumulation): the same beams counted (n_hits exact) and the sums
    within north_star's 1e-5 relative bar (measured ~1e-7), lattice scans and
    raw points."""
    import torch

    from paper_2301_08068_b200.device import lidar_points_batch_device, lidar_policy_batch_device

    rng = np.random.default_rng(n + S)
    dirs = rng.standard_normal((n, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    ranges = rng.uniform(0.0, 3.0, (S, n))
    ranges[:, ::17] = np.inf
    valid = rng.random((S, n)) < 0.8
    v = rng.standard_normal((S, 3))
    Rs = np.stack([np.linalg.qr(rng.standard_normal((3, 3)))[0] for _ in range(S)])
    sl, ac = lidar_policy_batch_device(torch.from_numpy(dirs).cuda(),
                                       torch.from_numpy(Rs.reshape(S, 9).copy()).cuda(),
                                       torch.from_numpy(ranges).cuda(),
                                       torch.from_numpy(valid.astype(np.uint8)).cuda(),
                                       torch.from_numpy(v).cuda(), LIDAR, 0.3, mode="fast")
    sl = sl.cpu().numpy()
    for s in range(S):
        slot_r, _ = oracle.lidar_policy(dirs @ Rs[s].T, ranges[s], valid[s], v[s], LIDAR, 0.3)
        assert sl[s][12] == slot_r[12]
        assert rel_err(sl[s][:12], slot_r[:12]) <= 1e-5
    pts = rng.uniform(-3.0, 3.0, (S, n, 3)).astype(np.float32)
    sp, _ = lidar_points_batch_device(torch.from_numpy(pts).cuda(), None,
                                      torch.from_numpy(v).cuda(), LIDAR, 0.3, mode="fast")
    se, _ = lidar_points_batch_device(torch.from_numpy(pts).cuda(), None,
                                      torch.from_numpy(v).cuda(), LIDAR, 0.3)
    sp, se = sp.cpu().numpy(), se.cpu().numpy()
    assert np.array_equal(sp[:, 12], se[:, 12])
    assert rel_err(sp[:, :12], se[:, :12]) <= 1e-5
    with pytest.raises(ValueError):
        lidar_points_batch_device(torch.from_numpy(pts).cuda(), None, torch.from_numpy(v).cuda(),
                                  LIDAR, 0.3, mode="fp16")
