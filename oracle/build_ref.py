"""Build the REFERENCE's own compiled kernel module into ``oracle/_ref/``.

TEST INFRASTRUCTURE ONLY.  This recipe compiles the reference's Cython
source ``/root/reference/pkg/src/rmpnav/_kernels/_ckern.pyx`` exactly as
``pkg/setup.py:9-19`` does (Cython -> C, gcc ``-O3``), but writes the
generated C into a temporary directory and the shared object into
``oracle/_ref/`` (git-ignored; it travels to the GPU box like every other
built ``.so``).  Nothing is copied from the reference into the repository.

The resulting module ``_ckern`` exposes the reference's chunk kernels
(``grid_trace_chunk``, ``policy_reduce_chunk``, ``bake_chunk``,
``scene_distance_chunk``, ``scene_trace_chunk``, ``esdf_sample_chunk``;
rmpnav/_kernels/_ckern.pyx:59-321).  It is used (a) to pin the C
restatement in ``oracle/rmp_oracle.c`` and (b) as the ``kind: "reference"``
CPU arm of ``bench.py``.

Run: ``python oracle/build_ref.py`` (no-op when /root/reference is absent,
e.g. on the GPU box, where the prebuilt .so is used).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import sysconfig
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PYX = "/root/reference/pkg/src/rmpnav/_kernels/_ckern.pyx"
OUT_DIR = os.path.join(HERE, "_ref")


def ref_so_path() -> str:
    return os.path.join(OUT_DIR, "_ckern" + sysconfig.get_config_var("EXT_SUFFIX"))


def build(force: bool = False) -> str | None:
    """Compile the reference kernel module; returns the .so path or None."""
    out = ref_so_path()
    if not os.path.exists(REF_PYX):
        return out if os.path.exists(out) else None
    if os.path.exists(out) and not force and os.path.getmtime(out) >= os.path.getmtime(REF_PYX):
        return out
    import numpy as np
    from Cython.Build import cythonize  # noqa: F401  (ensures Cython present)
    from Cython.Compiler import Main as cymain

    os.makedirs(OUT_DIR, exist_ok=True)
    with tempfile.TemporaryDirectory(prefix="rmpnav_ref_") as tmp:
        pyx = os.path.join(tmp, "_ckern.pyx")
        shutil.copyfile(REF_PYX, pyx)  # scratch copy in /tmp only (reference mount is read-only)
        c_file = os.path.join(tmp, "_ckern.c")
        opts = cymain.CompilationOptions(cymain.default_options)
        opts.output_file = c_file
        opts.language_level = 3
        res = cymain.compile(pyx, opts)
        if res.num_errors:
            raise RuntimeError("cython failed on the reference _ckern.pyx")
        cmd = [
            os.environ.get("CC", "gcc"), "-shared", "-fPIC", "-O3",
            # same flags setuptools passes through on this interpreter, minus -g
            "-fno-strict-aliasing", "-fwrapv", "-ffp-contract=off",
            "-DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION",
            "-I" + sysconfig.get_paths()["include"], "-I" + np.get_include(),
            c_file, "-o", out, "-lm",
        ]
        subprocess.run(cmd, check=True)
    return out


if __name__ == "__main__":
    p = build(force="--force" in sys.argv)
    print(p if p else "reference not present; nothing built")
