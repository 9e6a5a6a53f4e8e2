"""Single-pose kernel anatomy: warm kernel time (CUDA events, median of 30)
per C1 pose at max range 10 m vs ~0 (fixed cost: launch, prep, fold, pinv),
with the pose's longest ray (steps) -- the dependent-chain floor."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2301_08068_b200 import synth
from paper_2301_08068_b200.device import RayPolicyEngine
from paper_2301_08068_b200._kernels import b200
import paper_2301_08068_b200 as P

scene = synth.c1_scene(); grid = synth.c1_grid(scene)
states = synth.bench_states(scene, count=10, seed=123)
bundle = P.sample_directions(65536)
prm = P.preset("static_map").obstacle.as_tuple()
out = []
for mr in (1e-6, 10.0):
    eng = RayPolicyEngine(grid, bundle, prm, mr)
    for i in range(10):
        x = torch.tensor(states[i].position, dtype=torch.float64, device="cuda").view(1, 3)
        v = torch.tensor(states[i].velocity, dtype=torch.float64, device="cuda").view(1, 3)
        s = torch.empty((1, 13), dtype=torch.float64, device="cuda")
        a = torch.empty((1, 3), dtype=torch.float64, device="cuda")
        for _ in range(3):
            eng.evaluate(x, v, s, a)
        ts = []
        for _ in range(30):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(200000)  # GPU busy while the host enqueues: e0 -> e1 = kernel
            e0.record(); eng.evaluate(x, v, s, a); e1.record(); e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        rec = {"max_range": mr, "pose": i, "us_median": round(ts[15], 2), "us_min": round(ts[0], 2)}
        if mr > 1:
            _, _, t, cells, steps = b200.ray_policy_fused(grid.values, grid.origin, grid.resolution,
                                                          states[i].position, states[i].velocity,
                                                          bundle.directions, prm, mr, 0.05, 0.9,
                                                          with_rays=True)
            rec.update(max_steps=int(steps.max()), mean_steps=round(float(steps.mean()), 2),
                       p99_steps=int(np.percentile(steps, 99)))
        out.append(rec)
        print(json.dumps(rec), flush=True)
