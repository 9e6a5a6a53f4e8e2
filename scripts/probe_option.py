"""Sweep one librmpb option (rmpb_set_option) on the C1 4096-pose batch (GPU box).

    python scripts/probe_option.py carveout -1 0 25 44 60 100
Prints one JSON line {value: best-of-5 ms}."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2301_08068_b200 as P  # noqa: E402
from paper_2301_08068_b200 import _lib, synth  # noqa: E402
from paper_2301_08068_b200.device import RayPolicyEngine  # noqa: E402

name = sys.argv[1]
values = [int(v) for v in sys.argv[2:]]
scene = synth.c1_scene()
grid = synth.c1_grid(scene)
x_h, v_h = synth.states_arrays(synth.bench_states(scene, count=4096, seed=123))
eng = RayPolicyEngine(grid, P.sample_directions(65536),
                      P.preset("static_map").obstacle.as_tuple(), 10.0)
x = torch.from_numpy(x_h).cuda()
v = torch.from_numpy(v_h).cuda()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
ref = None
out = {"option": name}
for rnd in range(2):
    for val in values:
        _lib.call("rmpb_set_option", name.encode(), val)
        s, a = eng.evaluate(x, v)
        torch.cuda.synchronize()
        if ref is None:
            ref = s.clone()
        same = bool(torch.equal(s, ref))
        ts = []
        for _ in range(5):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            eng.evaluate(x, v)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        key = str(val)
        out[key] = min(min(ts), out.get(key, 1e9))
        out[key + "_bitexact"] = same
print(json.dumps(out))
