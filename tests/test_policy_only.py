"""CPU: the policy-only march limit (rays.policy_range) leaves the policy
unchanged.  On the oracle (the reference's algorithm, _ckern.pyx:171-321):
tracing to min(max_range, radius) instead of max_range gives BITWISE the same
sum A f / sum A (hits at d >= radius have activation weight 0 and are not
summed, _ckern.pyx:300-306), per-ray t equal where t <= radius, and a hit
count of the hits within the radius."""

import numpy as np

from conftest import STATIC_MAP
from test_oracle import golden_grid

from paper_2301_08068_b200.rays import policy_range


def test_policy_range_values():
    assert policy_range(10.0, 2.4) == 2.4
    assert policy_range(1.0, 2.4) == 1.0
    assert policy_range(10.0, float("nan")) == 10.0
    assert policy_range(10.0, float("inf")) == 10.0
    assert policy_range(0.0, 2.4) == 0.0


def test_oracle_policy_unchanged_by_radius_cut(oracle, golden):
    g = golden
    vals = golden_grid(oracle, g)
    res = float(g["grid_res"])
    radius = STATIC_MAP[5]
    for params in (STATIC_MAP, STATIC_MAP[:5] + (0.7,) + STATIC_MAP[6:]):
        r = params[5]
        for k in range(g["pose_x"].shape[0]):
            x, v = g["pose_x"][k], g["pose_v"][k]
            full, acc_f, t_f = oracle.ray_policy(vals, g["grid_origin"], res, x, v, g["dirs"],
                                                 params, 10.0)
            cut, acc_c, t_c = oracle.ray_policy(vals, g["grid_origin"], res, x, v, g["dirs"],
                                                params, policy_range(10.0, r))
            assert np.array_equal(cut[:12], full[:12]), f"pose {k}"
            assert np.array_equal(acc_c, acc_f)
            within = np.isfinite(t_f) & (t_f <= r)
            assert cut[12] == within.sum()
            assert np.array_equal(t_c, np.where(within, t_f, np.inf))
    assert radius == 2.4
