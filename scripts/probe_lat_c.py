"""Writes the C1 grid / bundle / 10 poses as raw files for scripts/lat_c.cu."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2301_08068_b200 import synth
import paper_2301_08068_b200 as P
scene = synth.c1_scene(); grid = synth.c1_grid(scene)
states = synth.bench_states(scene, count=10, seed=123)
grid.values.astype(np.float32).tofile("/tmp/lat_vals.f32")
np.ascontiguousarray(P.sample_directions(65536).directions).tofile("/tmp/lat_dirs.f64")
np.array([np.r_[s.position, s.velocity] for s in states]).tofile("/tmp/lat_poses.f64")
