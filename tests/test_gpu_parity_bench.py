"""GPU parity of the EXACT launch shapes the bench times.

* the throughput kernel ``k_ray_policy2`` with per-ray outputs (option
  ``kernel=2`` + ``with_rays``): t, hit cell, step count BIT-EXACT vs the
  oracle (the RAYOUT variant, including the shared first step);
* the bench launch itself (P = 4096 poses, default segmentation: 4 segments
  of 16384 rays, ``INSIDE=true`` body) through ``RayPolicyEngine.evaluate``:
  32 strided poses vs the oracle, n_hits exact, sums <= 1e-9 relative;
* a batch mixing poses outside the map (the ``INSIDE=false`` body);
* C2's ranges 2 / 5 / 20 m and 262 k / 1 M rays on the C1 map;
* subnormal / tiny direction components from starts outside the slab
  (the reference MISSes; an overflowing reciprocal must not turn that into
  a hit), tiny map-relative coordinates;
* the shared-first-step edge cases: a pose inside an obstacle, a -0.0
  coordinate, max_range shorter than the first step.

Reference: rmpnav/_kernels/_ckern.pyx:171-248 (trace), 278-321 (policy).
"""

import numpy as np
import pytest

from conftest import STATIC_MAP, rel_err

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
def c1(be, oracle):
    from paper_2301_08068_b200 import synth

    scene = synth.c1_scene()
    grid = synth.c1_grid(scene)
    states = synth.bench_states(scene, count=4096, seed=123)
    dirs = oracle.sample_directions(65536)
    return scene, grid, states, dirs


class _opt:
    """Temporarily set a librmpb option."""

    def __init__(self, name, value):
        self.name, self.value = name, value

    def __enter__(self):
        from paper_2301_08068_b200 import _lib

        _lib.set_option(self.name, self.value)

    def __exit__(self, *exc):
        from paper_2301_08068_b200 import _lib

        _lib.set_option(self.name, 0)


def _check(slot, acc, slot_r, acc_r):
    assert slot[12] == slot_r[12]
    assert rel_err(slot[:12], slot_r[:12]) <= SUM_TOL
    if np.abs(slot_r[:9]).max() > 0:
        assert rel_err(acc, acc_r) <= ACC_TOL


def _trace_both(be, oracle, vals, origin, res, start, dirs, max_range, kernel):
    with _opt("kernel", kernel):
        out = be.ray_policy_fused(vals, origin, res, start, [0.3, -0.2, 0.1], dirs, STATIC_MAP,
                                  max_range, 0.5 * res, 0.9, with_rays=True)
    t_r, c_r, s_r = oracle.grid_trace(vals, origin, res, start, dirs, max_range, 0.5 * res, 0.9,
                                      with_cells=True, with_steps=True, workers=8)
    return out, (t_r, c_r, s_r)


def test_throughput_kernel_rays_bit_exact(be, oracle, c1):
    """k_ray_policy2 (RAYOUT) per-ray t / cell / steps == oracle, 4 C1 poses."""
    scene, grid, states, dirs = c1
    for st in states[:4]:
        with _opt("kernel", 2):
            slot, acc, t, cells, steps = be.ray_policy_fused(
                grid.values, grid.origin, grid.resolution, st.position, st.velocity, dirs,
                STATIC_MAP, 10.0, 0.05, 0.9, with_rays=True)
        t_r, c_r, s_r = oracle.grid_trace(grid.values, grid.origin, grid.resolution,
                                          st.position, dirs, 10.0, 0.05, 0.9, with_cells=True,
                                          with_steps=True, workers=8)
        assert np.array_equal(t, t_r)
        assert np.array_equal(cells, c_r)
        assert np.array_equal(steps, s_r)
        slot_r = oracle.policy_slot(dirs, t_r, st.velocity, STATIC_MAP)
        _check(slot, acc, slot_r, oracle.accel_from_slot(slot_r))


def test_bench_launch_vs_oracle(be, oracle, c1):
    """The bench step: 4096 poses x 65536 device-Halton rays, one launch
    (RayPolicyEngine.evaluate, default segmentation), 32 strided poses vs
    the oracle fed the same direction array."""
    import torch

    import paper_2301_08068_b200 as P
    from paper_2301_08068_b200 import synth
    from paper_2301_08068_b200.device import RayPolicyEngine

    scene, grid, states, _ = c1
    bundle = P.sample_directions(65536)
    eng = RayPolicyEngine(grid, bundle, STATIC_MAP, 10.0)
    x_h, v_h = synth.states_arrays(states)
    x = torch.from_numpy(x_h).cuda()
    v = torch.from_numpy(v_h).cuda()
    s, a = eng.evaluate(x, v)
    s, a = s.cpu().numpy(), a.cpu().numpy()
    dirs = bundle.directions
    for k in range(0, 4096, 128):
        slot_r, acc_r, _ = oracle.ray_policy(grid.values, grid.origin, grid.resolution,
                                             x_h[k], v_h[k], dirs, STATIC_MAP, 10.0, workers=8)
        _check(s[k], a[k], slot_r, acc_r)
    # the step counter variant (bench calibration) gives the same slots
    ctr = torch.zeros(1, dtype=torch.int64, device="cuda")
    s2, a2 = eng.evaluate(x, v, step_counter=ctr)
    assert np.array_equal(s2.cpu().numpy(), s) and np.array_equal(a2.cpu().numpy(), a)
    assert ctr.item() > 4096 * 65536


def test_outside_poses_batch(be, oracle, c1):
    """Poses outside the map domain (INSIDE=false body) mixed with inside
    ones in one batch; per-ray bit-exact through the RAYOUT kernel."""
    scene, grid, states, dirs = c1
    sub = np.ascontiguousarray(dirs[:16384])
    outside = np.array([[-1.5, 5.0, 3.0], [10.0, 21.0, 4.0], [5.0, 5.0, 11.0],
                        [25.0, -3.0, -2.0], [19.9, 19.9, 9.9], [0.0, 0.0, 0.0]])
    for x in outside:
        (slot, acc, t, c, s), (t_r, c_r, s_r) = _trace_both(be, oracle, grid.values, grid.origin,
                                                             grid.resolution, x, sub, 10.0, 2)
        assert np.array_equal(t, t_r) and np.array_equal(c, c_r) and np.array_equal(s, s_r)
    xs = np.concatenate([outside, np.stack([s.position for s in states[:10]])])
    vs = np.tile([[0.4, -0.3, 0.2]], (len(xs), 1))
    slots, accs = be.ray_policy_batch(grid.values, grid.origin, grid.resolution, xs, vs, sub,
                                      STATIC_MAP, 10.0, 0.05, 0.9)
    for k in range(len(xs)):
        slot_r, acc_r, _ = oracle.ray_policy(grid.values, grid.origin, grid.resolution, xs[k],
                                             vs[k], sub, STATIC_MAP, 10.0, workers=8)
        _check(slots[k], accs[k], slot_r, acc_r)


@pytest.mark.parametrize("max_range", [2.0, 5.0, 20.0])
def test_c2_ranges(be, oracle, c1, max_range):
    scene, grid, states, dirs = c1
    xs = np.stack([s.position for s in states[:3]])
    vs = np.stack([s.velocity for s in states[:3]])
    for kernel in (1, 2):
        with _opt("kernel", kernel):
            slots, accs = be.ray_policy_batch(grid.values, grid.origin, grid.resolution, xs, vs,
                                              dirs, STATIC_MAP, max_range, 0.05, 0.9)
        for k in range(3):
            slot_r, acc_r, _ = oracle.ray_policy(grid.values, grid.origin, grid.resolution,
                                                 xs[k], vs[k], dirs, STATIC_MAP, max_range,
                                                 workers=8)
            _check(slots[k], accs[k], slot_r, acc_r)
    st = states[1]
    (slot, acc, t, c, s), (t_r, c_r, s_r) = _trace_both(be, oracle, grid.values, grid.origin,
                                                         grid.resolution, st.position,
                                                         dirs[:8192], max_range, 2)
    assert np.array_equal(t, t_r) and np.array_equal(c, c_r) and np.array_equal(s, s_r)


@pytest.mark.parametrize("n", [262144, 1048576])
def test_c2_ray_counts(be, oracle, c1, n):
    scene, grid, states, _ = c1
    dirs = oracle.sample_directions(n)
    xs = np.stack([s.position for s in states[:2]])
    vs = np.stack([s.velocity for s in states[:2]])
    slots, accs = be.ray_policy_batch(grid.values, grid.origin, grid.resolution, xs, vs, dirs,
                                      STATIC_MAP, 10.0, 0.05, 0.9)
    for k in range(2):
        slot_r, acc_r, _ = oracle.ray_policy(grid.values, grid.origin, grid.resolution, xs[k],
                                             vs[k], dirs, STATIC_MAP, 10.0, workers=8)
        _check(slots[k], accs[k], slot_r, acc_r)


def _odd_dirs(rng, n):
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    tiny = np.array([1e-310, -4e-320, 5e-324, -1e-300, 3e-305, 1e-200, -2.5e-308])
    for a in range(3):
        blk = slice(200 * a, 200 * a + 200)
        d[blk, a] = rng.choice(tiny, size=200)
    d[600:610] = [[1.0, 1e-310, 0.0]] * 10
    d[610:620] = [[0.0, -1e-310, 1.0]] * 10
    return np.ascontiguousarray(d)


@pytest.mark.parametrize("kernel", [1, 2])
def test_subnormal_direction_components(be, oracle, kernel):
    """Direction components below 2^-1000 (subnormal included) from starts
    outside the slab of that axis: the reference's _box_span MISSes (its
    quotient is +-inf); the exact FMA division's reciprocal would overflow
    (NaN -> the constraint silently dropped).  Bit-exact t / cell / steps."""
    rng = np.random.default_rng(17)
    nx, ny, nz, res = 40, 30, 20, 0.1
    vals = (rng.normal(size=(nx, ny, nz)) * 0.3 + 0.4).astype(np.float32).astype(np.float64)
    o = np.zeros(3)
    dirs = _odd_dirs(rng, 2048)
    for start in ([-0.5, 1.0, 0.8], [2.0, 3.5, 0.8], [2.0, 1.0, -0.3], [1.9, 1.4, 0.9],
                  [0.0, 1.0, 0.8], [1.0, 0.0, 0.0], [4.5, 2.0, 1.0]):
        (slot, acc, t, c, s), (t_r, c_r, s_r) = _trace_both(be, oracle, vals, o, res, start,
                                                             dirs, 6.0, kernel)
        assert np.array_equal(t, t_r), start
        assert np.array_equal(c, c_r), start
        assert np.array_equal(s, s_r), start
        slot_r = oracle.policy_slot(dirs, t_r, [0.3, -0.2, 0.1], STATIC_MAP)
        _check(slot, acc, slot_r, oracle.accel_from_slot(slot_r))


@pytest.mark.parametrize("kernel", [1, 2])
def test_tiny_coordinates(be, oracle, kernel):
    """Map-relative coordinates in the subnormal range: poses on the origin
    planes (map origin 0) with tiny direction components, in launches that
    take the shared first step.  (Non-finite directions are undefined in the
    reference -- NaN cell indices read outside the map -- and not compared.)"""
    rng = np.random.default_rng(23)
    nx, ny, nz, res = 32, 32, 16, 0.1
    vals = (rng.random((nx, ny, nz)) * 0.6 + 0.05).astype(np.float32).astype(np.float64)
    vals[10:14, 10:14, :6] = -0.2
    o = np.zeros(3)
    dirs = _odd_dirs(rng, 1024)
    for start in ([0.0, 0.0, 0.0], [1e-310, 1.0, 5e-320], [1.5, 1.5, 0.0], [1.2, 1.3, 0.7]):
        (slot, acc, t, c, s), (t_r, c_r, s_r) = _trace_both(be, oracle, vals, o, res, start,
                                                             dirs, 4.0, kernel)
        assert np.array_equal(t, t_r), start
        assert np.array_equal(c, c_r), start
        assert np.array_equal(s, s_r), start


@pytest.mark.parametrize("kernel", [1, 2])
def test_shared_first_step_edge_cases(be, oracle, c1, kernel):
    """Pose inside an obstacle (every ray hits at t = 0: no shared step), a
    -0.0 coordinate, and max_range shorter than the first step (rays end
    after one step) -- through the throughput kernel with per-ray outputs."""
    scene, grid, states, dirs = c1
    sub = np.ascontiguousarray(dirs[:4096])
    vals = grid.values
    occ = np.argwhere(vals < -0.05)
    solid = grid.origin + occ[len(occ) // 2] * grid.resolution
    cases = [(solid, 10.0), (states[3].position, 0.01), (states[3].position, 0.0),
             (np.array([-0.0, 5.0, 2.0]), 10.0), (np.array([4.0, -0.0, -0.0]), 3.0),
             (states[5].position, -1.0)]
    for x, mr in cases:
        (slot, acc, t, c, s), (t_r, c_r, s_r) = _trace_both(be, oracle, vals, grid.origin,
                                                             grid.resolution, x, sub, mr, kernel)
        assert np.array_equal(t, t_r), (x, mr)
        assert np.array_equal(c, c_r), (x, mr)
        assert np.array_equal(s, s_r), (x, mr)


@pytest.mark.parametrize("rcond", [1e-8, 1e-3, 0.3, 0.0])
def test_pinv_psd_rcond(be, oracle, rcond):
    """pinv_psd with the reference's rcond argument (core.py:103-115)."""
    import paper_2301_08068_b200 as P

    rng = np.random.default_rng(7)
    for _ in range(20):
        q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
        lam = np.array([1.0, 10.0 ** rng.uniform(-6, 0), 10.0 ** rng.uniform(-10, -1)])
        a = (q * lam) @ q.T
        ref = oracle.pinv_psd(a, rcond)
        got = P.pinv_psd(a, rcond)
        assert rel_err(got, ref) <= 1e-6, (rcond, lam)


def test_server_parks_for_device_sync(be, c1):
    """A resident LatencyServer does not stall librmpb calls that must
    synchronise the device (a workspace growing, a map freed): they park it,
    and the next request relaunches it -- results unchanged."""
    import time

    import paper_2301_08068_b200 as P

    scene, grid, states, dirs = c1
    bundle = P.RayBundle(dirs)
    params = P.preset("static_map").obstacle
    with P.LatencyServer(grid, bundle, params, 10.0, idle_timeout_s=30.0) as srv:
        a = srv.policy(states[0])
        t0 = time.perf_counter()
        tmp = be.DeviceGrid(grid.values[:40, :40, :20].copy(), grid.origin, grid.resolution)
        del tmp  # cudaFree while the server kernel spins
        xs = np.stack([s.position for s in states[:300]])
        vs = np.stack([s.velocity for s in states[:300]])
        be.ray_policy_batch(grid.values, grid.origin, grid.resolution, xs, vs, dirs[:4096],
                            STATIC_MAP, 10.0, 0.05, 0.9)  # grows the workspaces
        assert time.perf_counter() - t0 < 5.0
        b = srv.policy(states[0])
        assert np.array_equal(a.accel, b.accel) and np.array_equal(a.metric, b.metric)


@pytest.mark.parametrize("res,origin", [(0.375, (0.0, 0.0, 0.0)),      # division not proven: 4-op
                                        (0.1, (-0.0, 0.0, -0.0)),      # -0 origin: 2-op, keeps p - o
                                        (0.1, (0.3, -1.2, 0.05)),      # 2-op, p - o
                                        (0.05, (0.0, 0.0, 0.0))])      # 2-op, origin +0 (no p - o)
def test_quad_division_paths(be, oracle, res, origin):
    """The three f32 QUAD trace paths (exdiv / exdiv2 / exdiv2 without p - o,
    chosen per map by rmpb_div2_exact and the origin) are all bit-exact."""
    rng = np.random.default_rng(int(res * 1000) + 7)
    nx, ny, nz = 40, 30, 20
    o = np.array(origin)
    ii, jj, kk = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    c = np.array([nx, ny, nz]) * 0.5
    vals = (np.sqrt(((ii - c[0]) * res) ** 2 + ((jj - c[1]) * res) ** 2) - 3.0 * res
            + 0.02 * rng.standard_normal((nx, ny, nz)))
    vals = vals.astype(np.float32).astype(np.float64)
    dirs = _odd_dirs(rng, 3000)
    center = o + c * res
    hits = []
    for start in (center + [0.0, 0.0, 0.1 * res], o + [1.5 * res, 2.5 * res, 1.0 * res],
                  o - [2.0 * res, 0.0, 0.0]):
        for kernel in (1, 2):
            (slot, acc, t, cl, s), (t_r, c_r, s_r) = _trace_both(be, oracle, vals, o, res, start,
                                                                 dirs, 50.0 * res, kernel)
            assert np.array_equal(t, t_r), (start, kernel)
            assert np.array_equal(cl, c_r), (start, kernel)
            assert np.array_equal(s, s_r), (start, kernel)
            hits.append(np.isfinite(t).mean())
    assert max(hits) > 0.1  # the field is actually hit


def test_map_update_reaches_latency_server(be, oracle):
    """EsdfGrid.update on a map a LatencyServer is serving: a region patch
    (f32-exact values) and a whole re-upload into the same handle (values
    that are not f32-exact: the QUAD f32 copy switches to the f64 layout)
    both reach the resident kernel; its next answer equals the oracle on the
    edited map."""
    import paper_2301_08068_b200 as P
    from paper_2301_08068_b200 import synth

    scene = synth.c1_scene(n_boxes=20, hi=np.array([5.9, 5.9, 2.9]))
    vals = be.bake_values(scene.packed(), np.zeros(3), 0.1, (60, 60, 30))
    vals = vals.astype(np.float32).astype(np.float64)
    grid = P.EsdfGrid(np.zeros(3), 0.1, (60, 60, 30), vals)
    dirs = oracle.sample_directions(4096)
    bundle = P.RayBundle(dirs)
    params = P.preset("static_map").obstacle
    st = synth.bench_states(scene, count=1, seed=9, distance=synth.host_box_distance(scene))[0]
    i, j, k = (int(c) for c in np.floor(st.position / 0.1))
    with P.LatencyServer(grid, bundle, params, 10.0, idle_timeout_s=30.0) as srv:
        for edit in ((slice(i + 1, i + 3), slice(j, j + 2), slice(k, k + 2), -0.5),
                     ((i, j + 1, k), 0.1234567890123)):
            srv.policy(st)
            grid.update(tuple(edit[:-1]) if len(edit) == 4 else edit[0], edit[-1])
            pol = srv.policy(st)
            ref = oracle.ray_policy(grid.values, grid.origin, 0.1, st.position, st.velocity,
                                    dirs, params.as_tuple(), 10.0)
            assert pol.metric.ravel().tolist() != [0.0] * 9
            assert rel_err(pol.metric.ravel(), ref[0][:9]) <= SUM_TOL
            assert rel_err(pol.accel, ref[1]) <= ACC_TOL
