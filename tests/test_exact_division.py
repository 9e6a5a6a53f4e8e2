"""CPU: the FMA-based exact division the CUDA trace uses instead of IEEE
`/` (rmpb_device.cuh ``exdiv``) reproduces a/b bit-for-bit."""

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
