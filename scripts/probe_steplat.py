"""Per-step latency of the single-pose kernel: GPU time (queued behind a sleep
kernel) vs the longest ray's step count, per pose; plus 1-ray bundles made of
each pose's longest ray."""
import sys, os, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np, torch
import oracle as O
from paper_2301_08068_b200 import synth, _lib as L
from paper_2301_08068_b200._kernels import b200
from paper_2301_08068_b200.device import RayPolicyEngine
import paper_2301_08068_b200 as P

scene = synth.c1_scene(); grid = synth.c1_grid(scene)
states = synth.bench_states(scene, count=10, seed=123)
bundle = P.sample_directions(65536)
params = P.preset("static_map").obstacle.as_tuple()
oslot = torch.empty((1, 13), dtype=torch.float64, device="cuda")
oacc = torch.empty((1, 3), dtype=torch.float64, device="cuda")

def gpu_time(fn, reps=20):
    for i in range(3): fn()
    torch.cuda.synchronize()
    ts = []
    for i in range(reps):
        torch.cuda._sleep(2_000_000)
        a = torch.cuda.Event(enable_timing=True); b_ = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b_.record(); b_.synchronize(); ts.append(a.elapsed_time(b_) * 1e3)
    return statistics.median(ts)

e = RayPolicyEngine(grid, bundle, params, 10.0)
out = []
for s in states:
    t, c, st = O.grid_trace(grid.values, grid.origin, grid.resolution, s.position, bundle.directions, 10.0, 0.05, 0.9, with_cells=True, with_steps=True)
    k = int(np.argmax(st))
    x = torch.tensor(s.position, dtype=torch.float64, device="cuda").view(1, 3)
    v = torch.tensor(s.velocity, dtype=torch.float64, device="cuda").view(1, 3)
    full = gpu_time(lambda: e.evaluate(x, v, oslot, oacc))
    one = RayPolicyEngine(grid, bundle.directions[k:k + 1].copy(), params, 10.0)
    t1 = gpu_time(lambda: one.evaluate(x, v, oslot, oacc))
    zero = RayPolicyEngine(grid, bundle.directions[k:k + 1].copy(), params, 1e-6)
    t0 = gpu_time(lambda: zero.evaluate(x, v, oslot, oacc))
    out.append(dict(max_steps=int(st.max()), mean_steps=float(st.mean()), full_us=round(full, 2), one_ray_us=round(t1, 2), one_ray_range0_us=round(t0, 2)))
print(json.dumps(out))
