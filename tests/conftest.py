import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))  # the CPU checker (tests only)

GOLDEN = os.path.join(ROOT, "tests", "golden", "rmpnav_golden.npz")
STATIC_MAP = (88.0, 1.4, 140.0, 1.2, 1e-6, 2.4, 0.2)
LIDAR = (1.2, 1.5, 3.0, 1.0, 1e-6, 1.3, 1.0)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "gpu2: needs two CUDA devices (NVLink peers); -m gpu2")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="session")
def oracle():
    import oracle as O

    O.build()
    return O


def golden_pack(g):
    return {"kinds": g["scene_kinds"], "ops": g["scene_ops"], "centers": g["scene_centers"],
            "sizes": g["scene_sizes"], "velocities": g["scene_velocities"],
            "empty_dist": float(g["scene_empty"])}


def rel_err(a, b):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    s = max(float(np.abs(b).max()) if b.size else 0.0, 1e-300)
    return float(np.abs(a - b).max()) / s if a.size else 0.0
