"""Single-pose fixed cost: device time (CUDA events behind a GPU spacer,
median of 30) of one C1 pose at max range ~0 and 10 m for several ray
segmentations (seg_rays: rays per CTA; 256 = one ray per thread) and both
kernels, next to a one-element torch kernel (the launch floor)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_08068_b200 import synth, _lib
from paper_2301_08068_b200.device import RayPolicyEngine
import paper_2301_08068_b200 as P

scene = synth.c1_scene(); grid = synth.c1_grid(scene)
states = synth.bench_states(scene, count=4, seed=123)
bundle = P.sample_directions(65536)
prm = P.preset("static_map").obstacle.as_tuple()


def timed(fn, reps=30):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200000)
        e0.record(); fn(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return round(ts[len(ts) // 2], 2), round(ts[0], 2)


z = torch.zeros(1, device="cuda")
print(json.dumps({"what": "torch fill_ (launch floor)", "us": timed(lambda: z.fill_(1.0))}), flush=True)
for kern in (0,):
    _lib.set_option("kernel", kern)
    for sr in (256,):
        _lib.set_option("seg_rays", sr)
        for mr in (1e-6, 1.2, 2.4, 10.0):
            eng = RayPolicyEngine(grid, bundle, prm, mr)
            res = []
            for i in range(4):
                x = torch.tensor(states[i].position, dtype=torch.float64, device="cuda").view(1, 3)
                v = torch.tensor(states[i].velocity, dtype=torch.float64, device="cuda").view(1, 3)
                s = torch.empty((1, 13), dtype=torch.float64, device="cuda")
                a = torch.empty((1, 3), dtype=torch.float64, device="cuda")
                res.append(timed(lambda: eng.evaluate(x, v, s, a))[0])
            print(json.dumps({"kernel": kern, "seg_rays": sr, "max_range": mr, "us_median_per_pose": res}),
                  flush=True)
_lib.set_option("seg_rays", 0)
_lib.set_option("kernel", 0)
