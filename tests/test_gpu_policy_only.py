"""GPU: policy-only evaluation (``policy_only=True``: rays stop at the
activation radius, rays.policy_range) against the oracle's FULL-range
policy on the C1 map -- same sums (<= 1e-9 relative), same acceleration,
n_hits = the oracle's hits within the radius -- and per-ray t / cell / steps
bit-exact vs the oracle traced to the same limit.  Through the batch kernel,
the RAYOUT kernel, the public ray_policy and the LatencyServer."""

import numpy as np
import pytest

from conftest import STATIC_MAP, rel_err

pytestmark = pytest.mark.gpu

SUM_TOL = 1e-9
ACC_TOL = 1e-6
R = STATIC_MAP[5]


@pytest.fixture(scope="module")
def c1(oracle):
    from paper_2301_08068_b200 import _lib, synth

    _lib.load()
    scene = synth.c1_scene()
    grid = synth.c1_grid(scene)
    states = synth.bench_states(scene, count=4096, seed=123)
    return scene, grid, states


def _full(oracle, grid, x, v, dirs):
    return oracle.ray_policy(grid.values, grid.origin, grid.resolution, x, v, dirs, STATIC_MAP,
                             10.0, workers=8)


def _check_vs_full(slot, acc, full_slot, full_acc, t_full):
    assert slot[12] == (np.isfinite(t_full) & (t_full <= R)).sum()
    assert rel_err(slot[:12], full_slot[:12]) <= SUM_TOL
    if np.abs(full_slot[:9]).max() > 0:
        assert rel_err(acc, full_acc) <= ACC_TOL


def test_engine_batch_policy_only(oracle, c1):
    import torch

    import paper_2301_08068_b200 as P
    from paper_2301_08068_b200 import synth
    from paper_2301_08068_b200.device import RayPolicyEngine

    scene, grid, states = c1
    bundle = P.sample_directions(65536)
    eng = RayPolicyEngine(grid, bundle, STATIC_MAP, 10.0, policy_only=True)
    assert eng.max_range == R
    x_h, v_h = synth.states_arrays(states)
    s, a = eng.evaluate(torch.from_numpy(x_h).cuda(), torch.from_numpy(v_h).cuda())
    s, a = s.cpu().numpy(), a.cpu().numpy()
    full_eng = RayPolicyEngine(grid, bundle, STATIC_MAP, 10.0)
    sf, af = full_eng.evaluate(torch.from_numpy(x_h).cuda(), torch.from_numpy(v_h).cuda())
    sf, af = sf.cpu().numpy(), af.cpu().numpy()
    assert rel_err(s[:, :12], sf[:, :12]) <= 1e-12
    assert (s[:, 12] <= sf[:, 12]).all()
    for k in range(0, 4096, 256):
        slot_r, acc_r, t_r = _full(oracle, grid, x_h[k], v_h[k], bundle.directions)
        _check_vs_full(s[k], a[k], slot_r, acc_r, t_r)


@pytest.mark.parametrize("kernel", [1, 2])
def test_rays_policy_only_bit_exact(be_lib, oracle, c1, kernel):
    from paper_2301_08068_b200 import _lib
    from paper_2301_08068_b200._kernels import b200
    from paper_2301_08068_b200.rays import policy_range

    scene, grid, states = c1
    dirs = oracle.sample_directions(65536)
    for st in states[:3]:
        _lib.set_option("kernel", kernel)
        try:
            slot, acc, t, cells, steps = b200.ray_policy_fused(
                grid.values, grid.origin, grid.resolution, st.position, st.velocity, dirs,
                STATIC_MAP, policy_range(10.0, R), 0.05, 0.9, with_rays=True)
        finally:
            _lib.set_option("kernel", 0)
        t_r, c_r, s_r = oracle.grid_trace(grid.values, grid.origin, grid.resolution, st.position,
                                          dirs, R, 0.05, 0.9, with_cells=True, with_steps=True,
                                          workers=8)
        assert np.array_equal(t, t_r) and np.array_equal(cells, c_r)
        assert np.array_equal(steps, s_r)
        slot_r, acc_r, t_full = _full(oracle, grid, st.position, st.velocity, dirs)
        assert np.array_equal(t, np.where(np.isfinite(t_full) & (t_full <= R), t_full, np.inf))
        _check_vs_full(slot, acc, slot_r, acc_r, t_full)


def test_public_api_and_server_policy_only(oracle, c1):
    import paper_2301_08068_b200 as P

    scene, grid, states = c1
    bundle = P.sample_directions(65536)
    prm = P.preset("static_map").obstacle
    with P.LatencyServer(grid, bundle, prm, 10.0, policy_only=True) as srv:
        assert srv.max_range == R
        for st in states[:6]:
            full = P.ray_policy(st, grid, bundle, prm, 10.0)
            cut = P.ray_policy(st, grid, bundle, prm, 10.0, policy_only=True)
            sv = srv.policy(st)
            for pol in (cut, sv):
                assert rel_err(pol.metric, full.metric) <= 1e-12
                assert rel_err(pol.accel, full.accel) <= 1e-9
    accs, metrics, hits = P.ray_policy_batch(states[:8], grid, bundle, prm, 10.0,
                                             policy_only=True)
    accs_f, metrics_f, hits_f = P.ray_policy_batch(states[:8], grid, bundle, prm, 10.0)
    assert rel_err(metrics, metrics_f) <= 1e-12 and rel_err(accs, accs_f) <= 1e-9
    assert (hits <= hits_f).all()


@pytest.fixture(scope="module")
def be_lib():
    from paper_2301_08068_b200 import _lib

    _lib.load()
    assert _lib.device_count() >= 1
    return _lib


def test_policy_only_outside_poses_and_exchange(be_lib, oracle, c1):
    """Poses outside the map (INSIDE=false body) and the K4 exchange path
    (world-1 mailbox) with policy_only engines: the full-range oracle
    policy, n_hits = the oracle's hits within the radius."""
    import torch

    from paper_2301_08068_b200._kernels import b200
    from paper_2301_08068_b200.device import PeerMailbox, RayPolicyEngine

    scene, grid, states = c1
    dirs = oracle.sample_directions(16384)
    eng = RayPolicyEngine(grid, b200.DeviceBundle(dirs), STATIC_MAP, 10.0, policy_only=True)
    xs = np.array([[-1.5, 5.0, 3.0], [10.0, 21.0, 4.0], [5.0, 5.0, 11.0], [19.9, 19.9, 9.9]]
                  + [s.position for s in states[:4]])
    vs = np.tile([[0.4, -0.3, 0.2]], (len(xs), 1))
    s, a = eng.evaluate(torch.from_numpy(xs).cuda(), torch.from_numpy(vs).cuda())
    s, a = s.cpu().numpy(), a.cpu().numpy()
    mb = PeerMailbox(1, 0)
    mb.open([mb.ipc_handle])
    try:
        for k in range(len(xs)):
            slot_r, acc_r, t_full = _full(oracle, grid, xs[k], vs[k], dirs)
            _check_vs_full(s[k], a[k], slot_r, acc_r, t_full)
            xs_t = torch.from_numpy(xs[k].copy()).cuda()
            vs_t = torch.from_numpy(vs[k].copy()).cuda()
            se, ae = eng.exchange(xs_t, vs_t, mb, k + 1, 0, eng.n_rays)
            _check_vs_full(se.cpu().numpy(), ae.cpu().numpy(), slot_r, acc_r, t_full)
    finally:
        mb.close()
