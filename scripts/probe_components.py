"""Cost split of the batched kernel: full vs no policy work (radius ~ 0)
vs prep + one step per ray (max_range ~ 0)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2301_08068_b200 import synth
from paper_2301_08068_b200._kernels import b200
from paper_2301_08068_b200.device import RayPolicyEngine
scene = synth.c1_scene(); grid = synth.c1_grid(scene)
states = synth.bench_states(scene, count=4096, seed=123, distance=synth.host_box_distance(scene))
x_h, v_h = synth.states_arrays(states)
x = torch.from_numpy(x_h).cuda(); v = torch.from_numpy(v_h).cuda()
dg = b200.DeviceGrid(grid.values, grid.origin, grid.resolution)
bundle = b200.DeviceBundle(halton_n=65536)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
def t(params, mr, mode="exact"):
    eng = RayPolicyEngine(dg, bundle, params, mr, mode=mode)
    eng.evaluate(x, v); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); eng.evaluate(x, v); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    return round(min(ts), 3)
S = (88.0, 1.4, 140.0, 1.2, 1e-6, 2.4, 0.2)
NOP = (88.0, 1.4, 140.0, 1.2, 1e-6, 1e-9, 0.2)
print(json.dumps({"full": t(S, 10.0), "no_policy": t(NOP, 10.0), "prep_1step": t(NOP, 1e-6),
                  "full_fast": t(S, 10.0, "fast"), "no_policy_fast": t(NOP, 10.0, "fast")}))
