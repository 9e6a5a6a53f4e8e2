"""CPU: the host fast path of the single-pose call (identity cache of the
grid / bundle arrays, trusted Policy construction) keeps the reference's
semantics: in-place edits are seen, non-finite results still raise."""

import numpy as np
import pytest

from paper_2301_08068_b200 import core, policies
from paper_2301_08068_b200._kernels import b200


class _Dev:  # stands in for a DeviceGrid / DeviceBundle (no GPU here)
    pass


def test_identity_cache_sees_in_place_edits():
    b200.invalidate_caches()
    a = np.random.default_rng(0).random((40, 30, 20))
    dev = _Dev()
    extra = ([0.0, 0.0, 0.0], 0.1, 0)
    b200._fast_put(a, extra, b200._frozen(a), dev)
    assert b200._fast_get(a, extra) is dev
    assert b200._fast_get(a, ([0.0, 0.0, 0.1], 0.1, 0)) is None  # other origin
    assert b200._fast_get(a.copy(), extra) is None               # other object
    idx = b200._sample_idx(a.size)
    a.reshape(-1)[idx[5]] += 1.0                                  # a sampled node
    assert b200._fast_get(a, extra) is None
    b200.invalidate_caches()
    assert b200._fast_get(a, extra) is None


def test_identity_cache_frozen_arrays_skip_sampling():
    b200.invalidate_caches()
    d = np.random.default_rng(1).normal(size=(1000, 3))
    d.flags.writeable = False
    dev = _Dev()
    b200._fast_put(d, 0, b200._frozen(d), dev)
    assert b200._fast.get(id(d))[2] is None
    assert b200._fast_get(d, 0) is dev
    b200.invalidate_caches()


def test_sample_covers_both_ends():
    idx = b200._sample_idx(10_000)
    assert idx[0] == 0 and idx[-1] == 9_999 and len(idx) == 72
    assert np.array_equal(b200._sample_idx(300), np.arange(300))


def test_trusted_policy_equals_checked_policy():
    rng = np.random.default_rng(2)
    for _ in range(50):
        m = rng.normal(size=(3, 3)) * 10.0 ** rng.integers(-5, 6)
        m = m + m.T
        slot = np.concatenate([m.reshape(-1), rng.normal(size=3), [7.0]])
        acc = rng.normal(size=3)
        fast = policies._policy_from_slot(slot, acc)
        ref = core.Policy(acc.copy(), slot[0:9].reshape(3, 3).copy())
        assert np.array_equal(fast.accel, ref.accel)
        assert np.array_equal(fast.metric, ref.metric)


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_fast_policy_still_raises_on_non_finite(bad):
    slot = np.zeros(13)
    acc = np.zeros(3)
    acc[1] = bad
    with pytest.raises(ValueError):
        policies._policy_from_slot(slot, acc)
    slot2 = np.zeros(13)
    slot2[4] = bad
    with pytest.raises(ValueError):
        policies._policy_from_slot(slot2, np.zeros(3))


def test_fast_policy_symmetrises_asymmetric_and_huge():
    slot = np.zeros(13)
    slot[1], slot[3] = 1.0, 3.0  # not symmetric -> Policy's own path
    p = policies._policy_from_slot(slot, np.zeros(3))
    assert p.metric[0, 1] == p.metric[1, 0] == 2.0
    slot = np.zeros(13)
    slot[0] = 1.5e308  # 0.5 * (m + m.T) overflows: the reference raises
    with pytest.raises(ValueError):
        policies._policy_from_slot(slot, np.zeros(3))
