"""Single-pose launches for ncu: C1 map, one pose, max range from argv
(default 10 m); 5 warm launches through the device engine."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_08068_b200 import synth
from paper_2301_08068_b200.device import RayPolicyEngine
import paper_2301_08068_b200 as P

mr = float(sys.argv[1]) if len(sys.argv) > 1 else 10.0
scene = synth.c1_scene(); grid = synth.c1_grid(scene)
states = synth.bench_states(scene, count=10, seed=123)
bundle = P.sample_directions(65536)
eng = RayPolicyEngine(grid, bundle, P.preset("static_map").obstacle.as_tuple(), mr)
for i in range(5):
    x = torch.tensor(states[i].position, dtype=torch.float64, device="cuda").view(1, 3)
    v = torch.tensor(states[i].velocity, dtype=torch.float64, device="cuda").view(1, 3)
    eng.evaluate(x, v)
torch.cuda.synchronize()
print("ok")
