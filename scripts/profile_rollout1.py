"""ncu target: a 1-robot closed-loop rollout on the C1 map, 32 ticks."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2301_08068_b200 as P
from paper_2301_08068_b200 import synth
from paper_2301_08068_b200.rollout import BatchRolloutConfig, RolloutBatch

scene = synth.c1_scene(); grid = synth.c1_grid(scene)
dist = synth.host_box_distance(scene)
starts = synth.states_arrays(synth.bench_states(scene, 1, seed=123, distance=dist))[0]
goals = synth.states_arrays(synth.bench_states(scene, 1, seed=321, distance=dist))[0]
cfg = BatchRolloutConfig(params=P.preset("static_map"), dt=0.01, max_time=60.0, max_range=10.0)
rb = RolloutBatch(scene, grid, P.sample_directions(65536), starts, goals, cfg)
rb.run(32)
torch.cuda.synchronize()
print("ok")
