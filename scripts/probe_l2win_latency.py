"""Single-pose kernel time after an L2-thrashing write (256 MiB), with and
without the map's L2 access-policy window (option l2_window)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_08068_b200 import synth, _lib
from paper_2301_08068_b200.device import RayPolicyEngine
import paper_2301_08068_b200 as P

scene = synth.c1_scene(); grid = synth.c1_grid(scene)
states = synth.bench_states(scene, count=64, seed=123)
x_h, v_h = synth.states_arrays(states)
bundle = P.sample_directions(65536)
eng = RayPolicyEngine(grid, bundle, P.preset("static_map").obstacle.as_tuple(), 10.0)
x = torch.from_numpy(x_h).cuda(); v = torch.from_numpy(v_h).cuda()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
out = {}
for w in (0, 1, 0, 1):
    _lib.call("rmpb_set_option", b"l2_window", w)
    for i in range(3):
        eng.evaluate(x[i:i + 1], v[i:i + 1])
    torch.cuda.synchronize()
    for flushed in (False, True):
        ts = []
        for i in range(40):
            if flushed:
                flush.fill_(float(i))
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); eng.evaluate(x[i % 64:i % 64 + 1], v[i % 64:i % 64 + 1]); e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        out.setdefault(f"win{w}_{'flushed' if flushed else 'warm'}_us_median", []).append(round(ts[len(ts) // 2], 2))
print(json.dumps(out))
