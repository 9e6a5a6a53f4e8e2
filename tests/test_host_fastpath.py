"""CPU: the host fast path of the single-pose call (identity cache of the
grid / bundle arrays, trusted Policy construction) keeps the reference's
semantics: a map edit is always seen (never a stale device copy), non-finite
results still raise."""

import numpy as np
import pytest

from paper_2301_08068_b200 import core, policies
from paper_2301_08068_b200._kernels import b200


class _Dev:  # stands in for a DeviceGrid / DeviceBundle (no GPU here)
    made = 0

    def __init__(self, *a, **k):
        _Dev.made += 1


def test_identity_cache_only_for_frozen_arrays(monkeypatch):
    """Deeply read-only arrays (EsdfGrid.values, RayBundle.directions) are
    served by identity; writable ones never take the identity path."""
    b200.invalidate_caches()
    monkeypatch.setattr(b200, "DeviceGrid", _Dev)
    a = np.random.default_rng(0).random((40, 30, 20))
    origin = np.zeros(3)
    g1 = b200.device_grid(a, origin, 0.1)
    assert id(a) not in b200._fast                      # writable: keyed path only
    f = a.copy()
    f.setflags(write=False)
    g2 = b200.device_grid(f, origin, 0.1)
    assert b200._fast_get(f, ([0.0, 0.0, 0.0], 0.1, b200._device)) is g2
    assert b200._fast_get(f, ([0.0, 0.0, 0.1], 0.1, b200._device)) is None  # other origin
    assert g1 is not g2
    b200.invalidate_caches()


def test_keyed_cache_sees_any_single_node_edit(monkeypatch):
    """Writable arrays are re-validated bit for bit on every hit: an edit of
    ONE node anywhere (not just at sampled positions) forces a re-upload --
    the reference re-reads the map on every call (ckern.py:49-62)."""
    b200.invalidate_caches()
    monkeypatch.setattr(b200, "DeviceGrid", _Dev)
    a = np.random.default_rng(0).random((40, 30, 20))
    origin = np.zeros(3)
    g1 = b200.device_grid(a, origin, 0.1)
    assert b200.device_grid(a, origin, 0.1) is g1       # unchanged: cache hit
    rng = np.random.default_rng(1)
    for _ in range(20):
        i, j, k = (int(rng.integers(0, n)) for n in a.shape)
        a[i, j, k] += 1e-12
        g2 = b200.device_grid(a, origin, 0.1)
        assert g2 is not g1
        g1 = g2
        assert b200.device_grid(a, origin, 0.1) is g1
    a[3, 4, 5] = np.nan                                   # NaN-safe (bitwise) compare
    g3 = b200.device_grid(a, origin, 0.1)
    assert g3 is not g1 and b200.device_grid(a, origin, 0.1) is g3
    b200.invalidate_caches()


def test_bundle_cache_sees_in_place_edits(monkeypatch):
    b200.invalidate_caches()
    monkeypatch.setattr(b200, "DeviceBundle", _Dev)
    d = np.random.default_rng(1).normal(size=(1000, 3))
    b1 = b200.device_bundle(d)
    assert b200.device_bundle(d) is b1
    d[517, 1] *= -1.0
    assert b200.device_bundle(d) is not b1
    b200.invalidate_caches()


def test_esdf_grid_values_are_private_and_read_only():
    from paper_2301_08068_b200 import EsdfGrid

    a = np.random.default_rng(2).random((6, 5, 4))
    g = EsdfGrid(np.zeros(3), 0.1, a.shape, a)
    assert not g.values.flags.writeable and g.values is not a
    with pytest.raises(ValueError):
        g.values[1, 1, 1] = 0.0
    a[1, 1, 1] = 123.0                      # the caller's array is not aliased
    assert g.values[1, 1, 1] != 123.0
    assert b200._frozen(g.values)
    # a deeply frozen input is adopted as is (no copy)
    g2 = EsdfGrid(np.zeros(3), 0.1, a.shape, g.values)
    assert g2.values is g.values


def test_esdf_grid_update_patches_and_notifies(monkeypatch):
    from paper_2301_08068_b200 import EsdfGrid

    calls = []
    monkeypatch.setattr(b200, "grid_updated", lambda v, c, sub: calls.append((v, c, sub.copy())))
    a = np.random.default_rng(3).random((8, 7, 6))
    g = EsdfGrid(np.zeros(3), 0.1, a.shape, a)
    vid = id(g.values)
    g.update((slice(2, 4), 3, slice(None)), -0.5)
    assert (g.values[2:4, 3, :] == -0.5).all() and g.values[1, 3, 0] == a[1, 3, 0]
    assert id(g.values) == vid and not g.values.flags.writeable
    v, corner, sub = calls[-1]
    assert v is g.values and corner == (2, 3, 0) and sub.shape == (2, 1, 6)
    # an adopted (shared) array is copied before the first edit
    g2 = EsdfGrid(np.zeros(3), 0.1, a.shape, g.values)
    g2.update((0, 0, 0), 9.0)
    assert g2.values is not g.values and g.values[0, 0, 0] != 9.0 and g2.values[0, 0, 0] == 9.0
    with pytest.raises(ValueError):
        g.update((slice(0, 4, 2), 0, 0), 1.0)
    with pytest.raises(IndexError):
        g.update((8, 0, 0), 1.0)


def test_ray_bundle_private_copy():
    from paper_2301_08068_b200 import RayBundle

    d = np.random.default_rng(4).normal(size=(10, 3))
    rb = RayBundle(d)
    d[0, 0] = 99.0
    assert rb.directions[0, 0] != 99.0 and not rb.directions.flags.writeable
    assert RayBundle(rb.directions).directions is rb.directions


def test_no_temporary_pointer_arguments():
    """ctypes arguments must not be pointers into temporaries (the buffer is
    freed before the C call runs): no `f(...).ctypes.data` in the backend."""
    import pathlib
    import re

    src = pathlib.Path(b200.__file__).read_text()
    assert not re.search(r"\)\.ctypes\.data", src)


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
