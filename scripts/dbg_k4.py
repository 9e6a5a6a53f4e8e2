import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2301_08068_b200 import synth, _lib as L
from paper_2301_08068_b200._kernels import b200
from paper_2301_08068_b200.device import RayPolicyEngine, PeerMailbox
scene = synth.c1_scene(); grid = synth.c1_grid(scene)
st = synth.bench_states(scene, count=1, seed=123)[0]
b2 = b200.DeviceBundle(halton_n=65536)
eng2 = RayPolicyEngine(b200.DeviceGrid(grid.values, grid.origin, grid.resolution), b2, (88.0, 1.4, 140.0, 1.2, 1e-6, 2.4, 0.2), 10.0)
x = torch.tensor(st.position, dtype=torch.float64, device="cuda")
v = torch.tensor(st.velocity, dtype=torch.float64, device="cuda")
mb = PeerMailbox(1, 0)
lib = L.load()
f = lib.rmpb_debug_ex_times
for i in range(6):
    eng2.exchange(x, v, mb, 1 + i, 0, 65536)
    torch.cuda.synchronize()
    t = (ctypes.c_ulonglong * 8)()
    f(t)
    t = list(t)
    print([t[k] - t[0] for k in range(7)])
