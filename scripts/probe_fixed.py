"""Single-pose fixed-overhead breakdown: evaluate() vs partial() (no pinv)
at a near-zero range, plus an empty-kernel launch baseline."""
import sys, os, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2301_08068_b200 import synth, _lib
from paper_2301_08068_b200.device import RayPolicyEngine
import paper_2301_08068_b200 as P
scene = synth.c1_scene(); grid = synth.c1_grid(scene)
states = synth.bench_states(scene, count=4, seed=123)
bundle = P.sample_directions(65536)
prm = P.preset("static_map").obstacle.as_tuple()
res = {}
def med(fn, n=40):
    for _ in range(5): fn()
    ts = []
    for _ in range(n):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
    return round(statistics.median(ts), 2)
x1 = torch.tensor(states[0].position, dtype=torch.float64, device="cuda")
v1 = torch.tensor(states[0].velocity, dtype=torch.float64, device="cuda")
z = torch.zeros(1, device="cuda")
res["empty_torch_kernel_us"] = med(lambda: z.add_(1))
for mr in (1e-6, 10.0):
    eng = RayPolicyEngine(grid, bundle, prm, mr)
    res[f"evaluate_us_{mr}"] = med(lambda: eng.evaluate(x1.view(1, 3), v1.view(1, 3)))
    res[f"partial_us_{mr}"] = med(lambda: eng.partial(x1, v1, 0, 65536))
    res[f"partial_256rays_us_{mr}"] = med(lambda: eng.partial(x1, v1, 0, 256))
    slots = torch.zeros((8, 13), dtype=torch.float64, device="cuda"); slots[:, 0] = 1; slots[:, 4] = 2; slots[:, 8] = 3
    res["resolve_us"] = med(lambda: eng.resolve(slots))
    for sr in (256, 512, 1024, 4096):
        _lib.set_option("seg_rays", sr)
        res[f"evaluate_us_{mr}_seg{sr}"] = med(lambda: eng.evaluate(x1.view(1, 3), v1.view(1, 3)))
    _lib.set_option("seg_rays", 0)
print(json.dumps(res))
