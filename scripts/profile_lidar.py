"""ncu target: 2 launches of the batched LiDAR kernel (1024 C3 scans)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2301_08068_b200 import synth
from paper_2301_08068_b200.device import lidar_policy_batch_device
from paper_2301_08068_b200.rays import scan_pattern
scene = synth.c1_scene()
states = synth.bench_states(scene, count=10, seed=123, distance=synth.host_box_distance(scene))
scans = synth.lidar_scans(scene, states, 128, 1024, 20.0)
S = 1024
dirs = torch.from_numpy(np.ascontiguousarray(scan_pattern(128, 1024)).copy()).cuda()
rg = torch.from_numpy(np.stack([scans[i % 10].ranges for i in range(S)])).cuda()
vl = torch.from_numpy(np.stack([scans[i % 10].valid for i in range(S)]).astype(np.uint8)).cuda()
R = torch.eye(3, dtype=torch.float64, device="cuda").reshape(1, 9).repeat(S, 1).contiguous()
v = torch.from_numpy(np.stack([states[i % 10].velocity for i in range(S)])).cuda()
LIDAR = (1.2, 1.5, 3.0, 1.0, 1e-6, 1.3, 1.0)
for _ in range(2):
    lidar_policy_batch_device(dirs, R, rg, vl, v, LIDAR, 0.3)
torch.cuda.synchronize()
r = np.stack([s.ranges for s in scans]); ok = np.stack([s.valid for s in scans])
print("valid frac", ok.mean(), "within radius frac", (ok & (r < 1.3) & (r >= 0.3)).mean())
