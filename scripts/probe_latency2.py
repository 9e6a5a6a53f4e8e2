"""Single-pose latency, split: GPU-only kernel time (launch queued behind a
sleep kernel so host gaps are excluded), host call floors, public API."""
import sys, os, time, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2301_08068_b200 import synth, _lib as L
from paper_2301_08068_b200._kernels import b200
from paper_2301_08068_b200.device import RayPolicyEngine
import paper_2301_08068_b200 as P

scene = synth.c1_scene(); grid = synth.c1_grid(scene)
states = synth.bench_states(scene, count=10, seed=123)
bundle = P.sample_directions(65536)
params = P.preset("static_map").obstacle
res = {}
xs = [torch.tensor(s.position, dtype=torch.float64, device="cuda").view(1, 3) for s in states]
vs = [torch.tensor(s.velocity, dtype=torch.float64, device="cuda").view(1, 3) for s in states]
oslot = torch.empty((1, 13), dtype=torch.float64, device="cuda")
oacc = torch.empty((1, 3), dtype=torch.float64, device="cuda")

def gpu_time(fn, reps=30):
    for i in range(5): fn(i)
    torch.cuda.synchronize()
    ts = []
    for i in range(reps):
        torch.cuda._sleep(2_000_000)
        a = torch.cuda.Event(enable_timing=True); b_ = torch.cuda.Event(enable_timing=True)
        a.record(); fn(i); b_.record(); b_.synchronize(); ts.append(a.elapsed_time(b_) * 1e3)
    return round(statistics.median(ts), 2)

for kopt in (0, 2):
    L.set_option("kernel", kopt)
    for mr in (1e-6, 2.0, 10.0):
        e = RayPolicyEngine(grid, bundle, params.as_tuple(), mr)
        res[f"gpu_us_k{kopt}_range{mr}"] = gpu_time(lambda i: e.evaluate(xs[i % 10], vs[i % 10], oslot, oacc))
L.set_option("kernel", 0)
e = RayPolicyEngine(grid, bundle, params.as_tuple(), 10.0)
res["gpu_us_empty_fill"] = gpu_time(lambda i: oslot.fill_(0.0))

def med(fn, n=300):
    for _ in range(20): fn(0)
    ts = []
    for i in range(n):
        t0 = time.perf_counter(); fn(i); ts.append((time.perf_counter() - t0) * 1e6)
    return round(statistics.median(ts), 2)

g = b200.device_grid(grid.values, grid.origin, grid.resolution)
bd = b200.device_bundle(bundle.directions)
lib = L.load()
pr = np.asarray(params.as_tuple(), dtype=np.float64)
xv = np.empty(6); out = np.empty(16)
def raw(i, mr=10.0):
    s = states[i % 10]
    xv[:3] = s.position; xv[3:] = s.velocity
    lib.rmpb_ray_policy(g.handle, bd.handle, xv.ctypes.data, xv.ctypes.data + 24, pr.ctypes.data,
                        mr, 0.05, 0.9, out.ctypes.data, out.ctypes.data + 104, None, None, None, None)
res["raw_ctypes_us_range10"] = med(raw)
res["raw_ctypes_us_range0"] = med(lambda i: raw(i, 1e-6))
res["fused_host_call_us"] = med(lambda i: b200.ray_policy_fused(grid.values, grid.origin, grid.resolution, states[i % 10].position, states[i % 10].velocity, bundle.directions, params.as_tuple(), 10.0, 0.05, 0.9))
res["public_ray_policy_us"] = med(lambda i: P.ray_policy(states[i % 10], grid, bundle, params, 10.0))
with P.LatencyServer(grid, bundle, params, 10.0) as srv:
    res["server_policy_us"] = med(lambda i: srv.policy(states[i % 10]))
    res["server_eval_us"] = med(lambda i: srv.evaluate(states[i % 10].position, states[i % 10].velocity))
res["torch_sync_roundtrip_us"] = med(lambda i: (oslot.fill_(0.0), torch.cuda.synchronize()))
print(json.dumps(res))
