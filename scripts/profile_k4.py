"""ncu target: one C5-shape rank share (131072 of 1 M rays, C1 map for
speed) as the partial kernel and as the K4 fused exchange kernel (world-1
mailbox), 5 launches each, for the launch list's device durations."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2301_08068_b200 import synth
from paper_2301_08068_b200._kernels import b200
from paper_2301_08068_b200.device import RayPolicyEngine, PeerMailbox
from paper_2301_08068_b200.parallel import balanced_range

scene = synth.c1_scene(); grid = synth.c1_grid(scene)
st = synth.bench_states(scene, count=1, seed=123)[0]
n = 1 << 20
bundle = b200.DeviceBundle(halton_n=n)
eng = RayPolicyEngine(b200.DeviceGrid(grid.values, grid.origin, grid.resolution), bundle,
                      (88.0, 1.4, 140.0, 1.2, 1e-6, 2.4, 0.2), 10.0)
x = torch.tensor(st.position, dtype=torch.float64, device="cuda")
v = torch.tensor(st.velocity, dtype=torch.float64, device="cuda")
b0, e0 = balanced_range(n, 8, 0)
mb = PeerMailbox(1, 0)
for i in range(5):
    eng.partial(x, v, b0, e0)
for i in range(5):
    eng.exchange(x, v, mb, i + 1, b0, e0)
for i in range(5):  # post only (no wait / fold / pinv)
    eng.exchange(x, v, mb, 100 + i, b0, e0, mode=1)
parts = torch.stack([eng.partial(x, v, *balanced_range(n, 8, r)) for r in range(8)])
for i in range(3):  # fold + pinv kernel of the all-gather path
    eng.resolve(parts)
# well-conditioned metric (the whole sphere of one 65536-ray bundle, world 1):
# the fused epilogue's pinv takes the Cholesky path, as after a real C5 fold
b2 = b200.DeviceBundle(halton_n=65536)
eng2 = RayPolicyEngine(b200.DeviceGrid(grid.values, grid.origin, grid.resolution), b2,
                       (88.0, 1.4, 140.0, 1.2, 1e-6, 2.4, 0.2), 10.0)
for i in range(3):
    eng2.partial(x, v, 0, 65536)
for i in range(3):
    eng2.exchange(x, v, mb, 1000 + i, 0, 65536)
# split the epilogue: post only, then wait + fold + pinv only (same epoch)
for i in range(3):
    eng2.exchange(x, v, mb, 2000 + i, 0, 65536, mode=1)
    eng2.exchange(x, v, mb, 2000 + i, 0, 65536, mode=2)
torch.cuda.synchronize()
print("ok")
