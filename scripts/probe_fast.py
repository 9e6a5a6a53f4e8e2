"""Exact vs opt-in FAST (fp32 march) mode on the bench workload (4096 C1
poses x 65536 rays), CUDA events, L2 flushed between reps."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2301_08068_b200 import synth
from paper_2301_08068_b200.device import RayPolicyEngine
import paper_2301_08068_b200 as P

scene = synth.c1_scene(); grid = synth.c1_grid(scene)
states = synth.bench_states(scene, count=4096, seed=123)
x_h, v_h = synth.states_arrays(states)
bundle = P.sample_directions(65536)
x = torch.from_numpy(x_h).cuda(); v = torch.from_numpy(v_h).cuda()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
out = {}
for mode in ("exact", "fast"):
    eng = RayPolicyEngine(grid, bundle, P.preset("static_map").obstacle.as_tuple(), 10.0, mode=mode)
    s, a = eng.evaluate(x, v); torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); eng.evaluate(x, v); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    out[mode] = (sorted(ts)[3], s.cpu().numpy())
rel = float(np.abs(out["fast"][1][:, :12] - out["exact"][1][:, :12]).max() /
            np.abs(out["exact"][1][:, :12]).max())
print(json.dumps({"exact_ms": round(out["exact"][0], 3), "fast_ms": round(out["fast"][0], 3),
                  "hits_equal": bool((out["fast"][1][:, 12] == out["exact"][1][:, 12]).all()),
                  "max_rel_sum_dev": rel}))
