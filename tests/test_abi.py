"""CPU: the C-ABI library loads, exports every symbol include/rmpb.h declares,
and the host layer's registry / argument handling behaves like the
reference's (no compute without a GPU)."""

import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "rmpb.h")
LIB = os.path.join(ROOT, "paper_2301_08068_b200", "librmpb.so")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"RMPB_EXPORT\s+[\w\s\*]+?\b(rmpb_\w+)\s*\(", src)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for must in ("rmpb_grid_trace", "rmpb_policy_reduce", "rmpb_ray_policy",
                 "rmpb_ray_policy_batch_device", "rmpb_lidar_policy", "rmpb_pinv_psd",
                 "rmpb_bake", "rmpb_scene_trace", "rmpb_esdf_sample", "rmpb_fold_resolve_device"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "librmpb.so not built (run __graft_entry__.build())"
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (rmpb_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, f"declared but not exported: {missing}"


def test_ctypes_binding_covers_header():
    from paper_2301_08068_b200 import _lib

    assert sorted(_lib.EXPORTED) == declared_symbols()
    lib = _lib.load()
    assert lib.rmpb_api_version() == 1


def test_built_for_sm100a_with_fmad_off():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    # the exact trace is fp64 DMUL/DADD (fused DFMA only inside IEEE division)
    fn = sass.split("k_grid_traceINS_11QuadGridF32")[1].split("Function :")[0]
    assert "DMUL" in fn and "DADD" in fn and "MUFU.RCP64H" in fn


def test_registry_mirrors_reference():
    import paper_2301_08068_b200 as P

    assert P.available_backends() == ["b200"]
    assert P.default_backend_name() == "b200"
    with pytest.raises(ValueError):
        P.get_backend("numpy")
    with pytest.raises(ValueError):
        P.set_default_backend("compiled")
    be = P.get_backend()
    for fn in ("scene_distance_many", "bake_values", "esdf_sample_many", "grid_trace",
               "scene_trace", "policy_reduce"):
        assert callable(getattr(be, fn))
    assert be.name == "b200" and be.compiled is True


def test_invalid_arguments_raise_value_error():
    from paper_2301_08068_b200 import _lib

    # NULL handles / bad sizes are rejected before any device work
    with pytest.raises(ValueError):
        _lib.call("rmpb_ray_policy", None, None, None, None, None, 10.0, 0.05, 0.9, None, None,
                  None, None, None, None)
    with pytest.raises(ValueError):
        _lib.call("rmpb_fold_resolve_device", None, 0, None, None, None)
    with pytest.raises(ValueError):
        _lib.call("rmpb_set_option", b"no_such_knob", 1)


def test_no_cpu_fallback_without_gpu():
    """Without a CUDA device every compute call fails loudly (RuntimeError)."""
    from paper_2301_08068_b200 import _lib
    from paper_2301_08068_b200._kernels import b200

    if _lib.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError):
        b200.grid_trace(np.ones((4, 4, 4)), np.zeros(3), 0.1, np.zeros(3), np.eye(3), 1.0, 0.05,
                        0.9)
    with pytest.raises(RuntimeError):
        b200.policy_reduce(np.eye(3), np.ones(3), np.zeros(3), (1, 1, 1, 1, 1e-6, 1, 1))


def test_host_types_validate_like_reference():
    import paper_2301_08068_b200 as P

    with pytest.raises(ValueError):
        P.RobotState([0, 0, np.nan])
    with pytest.raises(ValueError):
        P.ObstacleParams(0.0, 1, 1, 1, 1, 1)
    with pytest.raises(ValueError):
        P.EsdfGrid(np.zeros(3), 0.1, (1, 4, 4), np.zeros((1, 4, 4)))
    with pytest.raises(ValueError):
        P.preset("nope")
    assert P.preset("static_map").obstacle.as_tuple() == (88.0, 1.4, 140.0, 1.2, 1e-6, 2.4, 0.2)
    pol = P.Policy([1, 2, 3], [[1, 2, 0], [0, 1, 0], [0, 0, 1]])
    assert np.array_equal(pol.metric, pol.metric.T)
    assert P.halton(1, 2) == 0.5 and P.halton(3, 2) == 0.75 and P.halton(1, 3) == 1.0 / 3.0


def test_scan_pattern_matches_reference_lattice(oracle, golden):
    import paper_2301_08068_b200 as P

    assert np.array_equal(P.scan_pattern(16, 128), golden["lidar_dirs"])
    assert np.array_equal(P.scan_pattern(128, 1024), oracle.scan_pattern(128, 1024))


def test_esdf_file_roundtrip(tmp_path):
    """ESDF binary cache (geometry.py:455-488): the documented 52-byte header
    (the reference's own struct format has an extra field and raises)."""
    import paper_2301_08068_b200 as P

    rng = np.random.default_rng(1)
    vals = rng.normal(size=(7, 5, 6)).astype(np.float32).astype(np.float64)
    g = P.EsdfGrid([0.5, -1.0, 2.0], 0.25, (7, 5, 6), vals)
    path = tmp_path / "m.esdf"
    P.save_esdf(g, path)
    assert path.stat().st_size == 52 + 4 * vals.size
    h = P.load_esdf(path)
    assert h.dims == g.dims and h.resolution == g.resolution
    assert np.array_equal(h.origin, g.origin) and np.array_equal(h.values, vals)
    raw = path.read_bytes()
    bad = tmp_path / "bad.esdf"
    bad.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(ValueError):
        P.load_esdf(bad)
    bad.write_bytes(raw[:60])
    with pytest.raises(ValueError):
        P.load_esdf(bad)
