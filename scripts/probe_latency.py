"""Single-pose latency breakdown on the C1 world (GPU box):
kernel-only (CUDA events, device-pointer entry), C-ABI host call, public API."""
import sys, os, time, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2301_08068_b200 import synth, _lib
from paper_2301_08068_b200._kernels import b200
from paper_2301_08068_b200.device import RayPolicyEngine
import paper_2301_08068_b200 as P

scene = synth.c1_scene(); grid = synth.c1_grid(scene)
states = synth.bench_states(scene, count=10, seed=123)
bundle = P.sample_directions(65536)
params = P.preset("static_map").obstacle
eng = RayPolicyEngine(grid, bundle, params.as_tuple(), 10.0)
res = {}
for P_ in (1, 2, 8, 64):
    x = torch.tensor(np.array([s.position for s in states] * 8)[:P_], dtype=torch.float64, device="cuda")
    v = torch.tensor(np.array([s.velocity for s in states] * 8)[:P_], dtype=torch.float64, device="cuda")
    for _ in range(5): eng.evaluate(x, v)
    torch.cuda.synchronize()
    ts = []
    for i in range(50):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); eng.evaluate(x, v); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    res[f"kernel_us_P{P_}"] = statistics.median(ts)
# single-pose kernel time vs max range (fixed overhead vs march)
for mr in (1e-6, 0.5, 2.0, 5.0, 10.0):
    e2 = RayPolicyEngine(eng.grid, eng.bundle, params.as_tuple(), mr)
    x1 = torch.tensor(states[0].position, dtype=torch.float64, device="cuda").view(1, 3)
    v1 = torch.tensor(states[0].velocity, dtype=torch.float64, device="cuda").view(1, 3)
    for _ in range(5): e2.evaluate(x1, v1)
    ts = []
    for i in range(30):
        a = torch.cuda.Event(enable_timing=True); b_ = torch.cuda.Event(enable_timing=True)
        a.record(); e2.evaluate(x1, v1); b_.record(); b_.synchronize(); ts.append(a.elapsed_time(b_) * 1e3)
    res[f"p1_us_range_{mr}"] = statistics.median(ts)
# C-ABI host call
def med(fn, n=200):
    for _ in range(10): fn(0)
    ts = []
    for i in range(n):
        t0 = time.perf_counter(); fn(i); ts.append((time.perf_counter() - t0) * 1e6)
    return statistics.median(ts)
res["fused_host_call_us"] = med(lambda i: b200.ray_policy_fused(grid.values, grid.origin, grid.resolution, states[i % 10].position, states[i % 10].velocity, bundle.directions, params.as_tuple(), 10.0, 0.05, 0.9))
res["public_ray_policy_us"] = med(lambda i: P.ray_policy(states[i % 10], grid, bundle, params, 10.0))
print(json.dumps(res))
