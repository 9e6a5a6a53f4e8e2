"""Single-scan LiDAR latency on C3 (GPU box): device kernel time (events) and
the public lidar_policy call, per kernel variant / warp target."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2301_08068_b200 as P  # noqa: E402
from paper_2301_08068_b200 import _lib, synth  # noqa: E402
from paper_2301_08068_b200.device import lidar_policy_batch_device  # noqa: E402
from paper_2301_08068_b200.rays import scan_pattern  # noqa: E402

scene = synth.c1_scene()
states = synth.bench_states(scene, count=10, seed=123, distance=synth.host_box_distance(scene))
scans = synth.lidar_scans(scene, states, 128, 1024, 20.0)
lp = P.preset("lidar").obstacle
LIDAR = lp.as_tuple()
dirs = torch.from_numpy(np.ascontiguousarray(scan_pattern(128, 1024)).copy()).cuda()
rg = torch.from_numpy(scans[0].ranges.copy()).cuda().view(1, -1)
vl = torch.from_numpy(scans[0].valid.astype(np.uint8)).cuda().view(1, -1)
R = torch.from_numpy(scans[0].orientation.reshape(1, 9).copy()).cuda()
v = torch.from_numpy(states[0].velocity.reshape(1, 3).copy()).cuda()
out = {}
for arg in sys.argv[1:]:
    k, _, wt = arg.partition(":")
    _lib.call("rmpb_set_option", b"lidar_kernel", int(k))
    if wt:
        _lib.call("rmpb_set_option", b"lidar_warps", int(wt))
    for _ in range(5):
        lidar_policy_batch_device(dirs, R, rg, vl, v, LIDAR, 0.3)
    ts = []
    for _ in range(30):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        lidar_policy_batch_device(dirs, R, rg, vl, v, LIDAR, 0.3)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    out[arg + "_dev_us"] = statistics.median(ts)
    lat = []
    for i in range(60):
        t0 = time.perf_counter()
        P.lidar_policy(states[i % 10].velocity, scans[i % 10], lp)
        lat.append((time.perf_counter() - t0) * 1e6)
    out[arg + "_api_us"] = statistics.median(lat[10:])
_lib.call("rmpb_set_option", b"lidar_kernel", 0)
_lib.call("rmpb_set_option", b"lidar_warps", 76000)
print(json.dumps(out))
