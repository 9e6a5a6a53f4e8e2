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
