"""Latency server per map layout: median host call time (C1, 10 poses)."""
import sys, os, time, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2301_08068_b200 import synth, _lib as L
import paper_2301_08068_b200 as P

scene = synth.c1_scene(); grid = synth.c1_grid(scene)
states = synth.bench_states(scene, count=10, seed=123)
bundle = P.sample_directions(65536)
params = P.preset("static_map").obstacle
def med(fn, n=400):
    for _ in range(20): fn(0)
    ts = []
    for i in range(n):
        t0 = time.perf_counter(); fn(i); ts.append((time.perf_counter() - t0) * 1e6)
    return round(statistics.median(ts), 2)
res = {}
ref = None
for name, st, lay in [("default", None, None), ("f32_quad", L.STORE_F32, L.LAYOUT_QUAD),
                      ("f32_linear", L.STORE_F32, L.LAYOUT_LINEAR),
                      ("f64_linear", L.STORE_F64, L.LAYOUT_LINEAR),
                      ("f64_pair64", L.STORE_F64, L.LAYOUT_PAIR64)]:
    with P.LatencyServer(grid, bundle, params, 10.0, storage=st, layout=lay) as srv:
        res[name] = med(lambda i: srv.evaluate(states[i % 10].position, states[i % 10].velocity))
        out = [srv.evaluate(s.position, s.velocity) for s in states]
        if ref is None:
            ref = out
        res[name + "_same"] = all(np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
                                  for a, b in zip(out, ref))
    print(json.dumps(res), flush=True)
