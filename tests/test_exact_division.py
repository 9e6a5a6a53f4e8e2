"""CPU: the arithmetic substitutions of the CUDA trace reproduce the
reference bit-for-bit: the FMA-based division (rmpb_device.cuh ``exdiv``)
equals IEEE a/b, and the round-toward-zero floor + boundary fix-up
(``cell_floor`` / ``cell_fix``) equals the reference clamp/floor/min."""

import os
import subprocess

from conftest import ROOT


def test_markstein_division_bit_exact(tmp_path):
    src = os.path.join(ROOT, "oracle", "check_exact_div.c")
    exe = str(tmp_path / "check_exact_div")
    subprocess.run(["gcc", "-O2", "-mfma", "-ffp-contract=off", "-o", exe, src, "-lm",
                    "-lpthread"], check=True)
    out = subprocess.run([exe, "40000000"], capture_output=True, text=True, check=True).stdout
    assert "mismatches=0" in out, out


def test_cell_floor_bit_exact(tmp_path):
    src = os.path.join(ROOT, "oracle", "check_cell_floor.c")
    exe = str(tmp_path / "check_cell_floor")
    subprocess.run(["gcc", "-O1", "-frounding-math", "-o", exe, src, "-lm"], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    assert "bad=0" in out, out


def test_two_op_division_bit_exact_for_proven_divisors(tmp_path):
    """exdiv2 (the trace step's division when rmpb_div2_exact proves the
    map resolution): random numerators over the proven divisor list."""
    src = os.path.join(ROOT, "oracle", "check_exact_div.c")
    exe = str(tmp_path / "check_exact_div")
    subprocess.run(["gcc", "-O2", "-mfma", "-ffp-contract=off", "-o", exe, src, "-lm",
                    "-lpthread"], check=True)
    out = subprocess.run([exe, "20000000", "2op"], capture_output=True, text=True,
                         check=True).stdout
    assert "mismatches=0" in out, out


def test_div2_proof_in_library():
    """librmpb's host-side proof (rmpb_div2_exact, no GPU needed) accepts the
    divisors of the list above and every map resolution the tests use."""
    import ctypes

    from paper_2301_08068_b200 import _lib

    lib = _lib.load()
    for b in (0.1, 0.05, 0.2, 0.25, 0.13, 0.3, 0.07, 1.0 / 3.0, 0.15, 0.02, 0.5, 0.01, 0.033,
              0.125, 0.0625, 0.9, 1.0000000000000002):
        out = ctypes.c_int(-1)
        assert lib.rmpb_div2_exact(ctypes.c_double(b), ctypes.byref(out)) == 0
        assert out.value == 1, b
    # not proven: 0.375 (mantissa 3 * 2^51: too many candidates to enumerate)
    # and 0.99999999999999989, for which the proof finds a wrongly rounded
    # quotient -- such maps keep the 4-op division
    for b in (0.375, 0.99999999999999989):
        out = ctypes.c_int(-1)
        lib.rmpb_div2_exact(ctypes.c_double(b), ctypes.byref(out))
        assert out.value == 0, b
    out = ctypes.c_int(-1)
    lib.rmpb_div2_exact(ctypes.c_double(float("nan")), ctypes.byref(out))
    assert out.value == 0
