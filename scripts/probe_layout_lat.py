"""Single-pose GPU time (queued behind a sleep kernel) per map layout."""
import sys, os, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2301_08068_b200 import synth, _lib as L
from paper_2301_08068_b200._kernels import b200
from paper_2301_08068_b200.device import RayPolicyEngine
import paper_2301_08068_b200 as P

scene = synth.c1_scene(); grid = synth.c1_grid(scene)
states = synth.bench_states(scene, count=10, seed=123)
bundle = P.sample_directions(65536)
params = P.preset("static_map").obstacle.as_tuple()
xs = [torch.tensor(s.position, dtype=torch.float64, device="cuda").view(1, 3) for s in states]
vs = [torch.tensor(s.velocity, dtype=torch.float64, device="cuda").view(1, 3) for s in states]
oslot = torch.empty((1, 13), dtype=torch.float64, device="cuda")
oacc = torch.empty((1, 3), dtype=torch.float64, device="cuda")
def gpu_time(fn, reps=40):
    for i in range(10): fn(i)
    torch.cuda.synchronize()
    ts = []
    for i in range(reps):
        torch.cuda._sleep(2_000_000)
        a = torch.cuda.Event(enable_timing=True); b_ = torch.cuda.Event(enable_timing=True)
        a.record(); fn(i); b_.record(); b_.synchronize(); ts.append(a.elapsed_time(b_) * 1e3)
    return round(statistics.median(ts), 2)
res = {}
for st, lay in [("f32", "quad"), ("f64", "pair64"), ("f64", "quad"), ("f32", "linear"), ("f64", "linear")]:
    dg = b200.DeviceGrid(grid.values, grid.origin, grid.resolution,
                         storage={"f32": L.STORE_F32, "f64": L.STORE_F64}[st],
                         layout={"quad": L.LAYOUT_QUAD, "linear": L.LAYOUT_LINEAR, "pair64": L.LAYOUT_PAIR64}[lay])
    e = RayPolicyEngine(dg, bundle, params, 10.0)
    res[f"{st}_{lay}"] = gpu_time(lambda i: e.evaluate(xs[i % 10], vs[i % 10], oslot, oacc))
    print(json.dumps(res), flush=True)
