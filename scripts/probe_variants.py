"""Kernel variant sweep on the C1 workload (GPU box): kernel v1/v2, map
storage/layout, occupancy builds (RMPB_LIBRARY). Prints one JSON line."""
import sys, os, time, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2301_08068_b200 import synth, _lib
from paper_2301_08068_b200._kernels import b200
from paper_2301_08068_b200.device import RayPolicyEngine
import paper_2301_08068_b200 as P

P_BATCH = int(os.environ.get("PROBE_P", "4096"))
scene = synth.c1_scene(); grid = synth.c1_grid(scene)
states = synth.bench_states(scene, count=P_BATCH, seed=123)
x_h, v_h = synth.states_arrays(states)
bundle = P.sample_directions(65536)
params = P.preset("static_map").obstacle.as_tuple()
x = torch.from_numpy(x_h).cuda(); v = torch.from_numpy(v_h).cuda()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
out = {"lib": os.environ.get("RMPB_LIBRARY", "default")}
L = _lib
def timed(eng, xx, vv, reps=3):
    eng.evaluate(xx, vv); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); eng.evaluate(xx, vv); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)
variants = [("f32", "quad"), ("f32", "quad_fast"), ("f64", "pair64")]
for kern in (0,):
    L.set_option("kernel", kern)
    for st, lay in variants:
        if kern == 1 and (st, lay) != ("f32", "quad"):
            continue
        fast = lay.endswith("_fast")
        lay0 = lay.replace("_fast", "")
        dg = b200.DeviceGrid(grid.values, grid.origin, grid.resolution,
                             storage={"f32": L.STORE_F32, "f64": L.STORE_F64}[st],
                             layout={"quad": L.LAYOUT_QUAD, "linear": L.LAYOUT_LINEAR, "quadb": L.LAYOUT_QUADB, "pair64": L.LAYOUT_PAIR64}[lay0])
        eng = RayPolicyEngine(dg, bundle, params, 10.0, mode="fast" if fast else "exact")
        ms = timed(eng, x, v)
        lat = []
        for i in range(30):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); eng.evaluate(x[i:i+1], v[i:i+1]); e1.record(); e1.synchronize()
            lat.append(e0.elapsed_time(e1) * 1e3)
        out[f"k{kern}_{st}_{lay}"] = {"batch_ms": round(ms, 3), "hz": round(P_BATCH / ms * 1e3, 1),
                                      "p1_us_med": round(statistics.median(lat), 1)}
        print(json.dumps({f"k{kern}_{st}_{lay}": out[f"k{kern}_{st}_{lay}"]}), flush=True)
L.set_option("kernel", 0)
print(json.dumps(out))
