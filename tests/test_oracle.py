"""CPU: pin the oracle (C restatement) against the reference's golden vectors
and, where built, against the reference's own compiled kernels."""

import hashlib

import numpy as np
import pytest

from conftest import LIDAR, STATIC_MAP, golden_pack, rel_err


def golden_grid(oracle, g, f32=True):
    pack = golden_pack(g)
    vals = oracle.bake_values(pack, g["grid_origin"], float(g["grid_res"]), tuple(g["grid_dims"]))
    return vals.astype(np.float32).astype(np.float64) if f32 else vals


def test_bake_matches_reference_hash(oracle, golden):
    vals = golden_grid(oracle, golden, f32=False)
    assert hashlib.sha256(vals.tobytes()).digest() == golden["grid_sha256_f64"].tobytes()


def test_spec_kats(oracle, golden):
    # SPEC.md:180-188 halton; 190-198 sample_directions(1); 200-208 sphere ray
    h = [oracle.radical_inverse([i], b)[0] for i, b in ((1, 2), (3, 2), (1, 3), (7, 2), (10, 3))]
    assert np.array_equal(h, golden["kat_halton"])
    assert h[:3] == [0.5, 0.75, 1.0 / 3.0]
    d1 = oracle.sample_directions(1)
    assert np.allclose(d1, golden["kat_dir1"], rtol=0, atol=1e-15)
    pack = {"kinds": np.array([0], np.int8), "ops": np.array([0], np.int8),
            "centers": np.zeros((1, 3)), "sizes": np.ones((1, 3)), "velocities": np.zeros((1, 3)),
            "empty_dist": float(np.linalg.norm([12.0, 12.0, 12.0]))}
    t = oracle.scene_trace(pack, [5, 0, 0], np.array([[-1.0, 0, 0]]), 20.0, 1e-4, 0.0)
    assert t[0] == golden["kat_sphere_ray"] == 4.0


def test_trace_bit_exact_vs_golden(oracle, golden):
    g = golden
    vals = golden_grid(oracle, g)
    for k in range(g["pose_x"].shape[0]):
        t = oracle.grid_trace(vals, g["grid_origin"], float(g["grid_res"]), g["pose_x"][k],
                              g["dirs"], 10.0, 0.5 * float(g["grid_res"]), 0.9)
        assert np.array_equal(t, g["trace_t"][k]), f"pose {k}"


def test_trace_f64_grid_bit_exact(oracle, golden):
    g = golden
    vals = golden_grid(oracle, g, f32=False)
    t = oracle.grid_trace(vals, g["grid_origin"], float(g["grid_res"]), g["pose_x"][0], g["dirs"],
                          10.0, 0.5 * float(g["grid_res"]), 0.9)
    assert np.array_equal(t, g["trace_t_f64grid"])


def test_policy_slots_bit_exact_vs_golden(oracle, golden):
    g = golden
    for k in range(g["pose_x"].shape[0]):
        slot = oracle.policy_slot(g["dirs"], g["trace_t"][k], g["pose_v"][k], STATIC_MAP)
        assert np.array_equal(slot, g["slots"][k]), f"pose {k}"
        acc = oracle.accel_from_slot(slot)
        assert rel_err(acc, g["accels"][k]) < 1e-12


def test_lidar_vs_golden(oracle, golden):
    g = golden
    for i in range(g["lidar_ranges"].shape[0]):
        R = g["lidar_rot"] if i == 1 else np.eye(3)
        wd = g["lidar_dirs"] @ R.T
        slot, acc = oracle.lidar_policy(wd, g["lidar_ranges"][i], g["lidar_valid"][i],
                                        g["pose_v"][i], LIDAR, 0.3)
        assert rel_err(slot[:9].reshape(3, 3), g["lidar_metrics"][i]) < 1e-12
        assert rel_err(acc, g["lidar_accels"][i]) < 1e-10


def test_scene_and_esdf_vs_golden(oracle, golden):
    g = golden
    pack = golden_pack(g)
    t = oracle.scene_trace(pack, g["pose_x"][1], g["scene_trace_dirs"], 20.0, 1e-4, 0.0)
    assert np.array_equal(t, g["scene_trace_t"])
    assert np.array_equal(oracle.scene_distance_many(pack, g["esdf_pts"], 0.0), g["scene_dist"])
    vals = golden_grid(oracle, g, f32=False)
    d, gr, fl = oracle.esdf_sample_many(vals, g["grid_origin"], float(g["grid_res"]), g["esdf_pts"])
    assert np.array_equal(d, g["esdf_d"]) and np.array_equal(gr, g["esdf_g"])
    assert np.array_equal(fl, g["esdf_flag"])


def test_pinv_vs_golden(oracle, golden):
    for a, b in zip(golden["pinv_in"], golden["pinv_out"]):
        assert np.allclose(oracle.pinv_psd(a), b, rtol=0, atol=1e-15 * max(1, np.abs(b).max()))


def test_pairwise_fold_shape(oracle):
    s = np.arange(7 * 13, dtype=float).reshape(7, 13)
    assert np.array_equal(oracle.pairwise_fold(s), oracle.ref_pairwise_fold(s.copy()))


@pytest.mark.skipif("not __import__('oracle').ref_available()", reason="oracle/_ref not built")
def test_port_bit_exact_vs_reference_module(oracle):
    """The C restatement equals the reference's own compiled kernels, on a
    random world with every branch (x/y/z-zero directions, outside starts)."""
    rng = np.random.default_rng(7)
    nx, ny, nz = 23, 17, 29
    vals = (rng.normal(size=(nx, ny, nz)) * 0.3 + 0.25).astype(np.float32).astype(np.float64)
    origin, res = np.array([-1.0, 0.5, -2.0]), 0.13
    dirs = rng.normal(size=(3000, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    dirs[:50, 0] = 0.0
    dirs[50:100, 1] = 0.0
    dirs[100:150, 2] = 0.0
    dirs[150:160] = [[0, 0, 1.0]] * 10
    for start in ([0.2, 1.3, 0.1], [-3.0, 1.0, 0.0], [0.3, 5.0, 30.0]):
        a = oracle.grid_trace(vals, origin, res, start, dirs, 6.0, 0.5 * res, 0.9)
        b = oracle.ref_grid_trace(vals, origin, res, np.array(start, float), dirs, 6.0, 0.5 * res,
                                  0.9)
        assert np.array_equal(a, b)
        v = rng.normal(size=3)
        m1, w1, n1 = oracle.policy_reduce(dirs, a, v, STATIC_MAP, 0.0)
        m2, w2, n2 = oracle.ref_policy_reduce(dirs, b, v, STATIC_MAP, 0.0)
        assert np.array_equal(m1, m2) and np.array_equal(w1, w2) and n1 == n2
