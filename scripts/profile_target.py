"""Small fixed workload for ncu captures: 2 batched launches (P poses), then
5 single-pose launches, of k_ray_policy2 on the C1 map."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_08068_b200 import synth
from paper_2301_08068_b200.device import RayPolicyEngine
import paper_2301_08068_b200 as P

PB = int(os.environ.get("PROBE_P", "4096"))
scene = synth.c1_scene(); grid = synth.c1_grid(scene)
states = synth.bench_states(scene, count=PB, seed=123)
x_h, v_h = synth.states_arrays(states)
bundle = P.sample_directions(65536)
eng = RayPolicyEngine(grid, bundle, P.preset("static_map").obstacle.as_tuple(), 10.0)
x = torch.from_numpy(x_h).cuda(); v = torch.from_numpy(v_h).cuda()
for _ in range(2):
    eng.evaluate(x, v)
for i in range(5):
    eng.evaluate(x[i:i + 1], v[i:i + 1])
torch.cuda.synchronize()
print("ok")
