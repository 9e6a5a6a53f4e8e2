"""ncu target: single-pose lean launches with and without the on-device
pinv (accel output NULL), at max range ~0 (fixed cost only) and 10 m."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_08068_b200 import synth, _lib as L
from paper_2301_08068_b200.device import RayPolicyEngine
import paper_2301_08068_b200 as P

scene = synth.c1_scene(); grid = synth.c1_grid(scene)
st = synth.bench_states(scene, count=1, seed=123)[0]
bundle = P.sample_directions(65536)
prm = P.preset("static_map").obstacle.as_tuple()
x = torch.tensor(st.position, dtype=torch.float64, device="cuda").view(1, 3)
v = torch.tensor(st.velocity, dtype=torch.float64, device="cuda").view(1, 3)
s = torch.empty((1, 13), dtype=torch.float64, device="cuda")
a = torch.empty((1, 3), dtype=torch.float64, device="cuda")
z = torch.zeros(1, device="cuda")
for _ in range(4):
    z.fill_(1.0)  # the launch floor under ncu
for mr in (1e-6, 2.4, 10.0):
    eng = RayPolicyEngine(grid, bundle, prm, mr)
    for acc in (None, a):
        for _ in range(4):
            L.call("rmpb_ray_policy_batch_device_mode", eng.grid.handle, eng.bundle.handle,
                   x.data_ptr(), v.data_ptr(), 1, eng.params.ctypes.data, eng.max_range, eng.eps,
                   eng.step_scale, eng.mode, s.data_ptr(), None if acc is None else acc.data_ptr(),
                   None, None)
torch.cuda.synchronize()
print("ok")
