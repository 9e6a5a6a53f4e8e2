"""C5 kernel choice: one 1 M-ray pose on the 1000x1000x200 TSDF (BRICK),
per pose: the K4 exchange path (lean kernel, world-1 mailbox), the batch
path with the lean kernel (option kernel=1) and with the refill kernel
k_ray_policy2 (kernel=2).  CUDA events, median of 7 per pose."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2301_08068_b200 import _lib, synth  # noqa: E402
from paper_2301_08068_b200._kernels import b200  # noqa: E402
from paper_2301_08068_b200.device import PeerMailbox, RayPolicyEngine  # noqa: E402

PARAMS = (88.0, 1.4, 140.0, 1.2, 1e-6, 2.4, 0.2)
scene = synth.c5_scene()
_dense, brick, info = synth.c5_grids(scene)
del _dense
states = synth.bench_states(scene, count=8, seed=123, distance=synth.host_box_distance(scene))
n = 1 << 20
eng = RayPolicyEngine(brick, b200.DeviceBundle(halton_n=n), PARAMS, 10.0)
xs = [torch.tensor(s.position, dtype=torch.float64, device="cuda").view(1, 3) for s in states]
vs = [torch.tensor(s.velocity, dtype=torch.float64, device="cuda").view(1, 3) for s in states]
mb = PeerMailbox(1, 0)
mb.open([mb.ipc_handle])
ep = [0]


def ex(k):
    ep[0] += 1
    eng.exchange(xs[k][0], vs[k][0], mb, ep[0], 0, n)


def timed(fn, reps=7):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return round(statistics.median(ts), 4)


if os.environ.get("C5_SWEEP"):  # kernel x seg_rays sweep of the batch path (median over poses)
    for kern in (1, 2):
        for sr in (256, 512, 1024, 2048, 4096, 8192):
            _lib.set_option("kernel", kern)
            _lib.set_option("seg_rays", sr)
            v = [timed(lambda: eng.evaluate(xs[k], vs[k]), reps=5) for k in range(8)]
            print(json.dumps({"kernel": kern, "seg_rays": sr, "median": statistics.median(v)}), flush=True)
    _lib.set_option("kernel", 0)
    _lib.set_option("seg_rays", 0)
    sys.exit(0)
out = {"exchange_auto": [], "batch_lean": [], "batch_k2": []}
slots = {}
for k in range(8):
    out["exchange_auto"].append(timed(lambda: ex(k)))
    for name, kern in (("batch_lean", 1), ("batch_k2", 2)):
        _lib.set_option("kernel", kern)
        out[name].append(timed(lambda: eng.evaluate(xs[k], vs[k])))
        s, _ = eng.evaluate(xs[k], vs[k])
        slots.setdefault(k, []).append(s.cpu().numpy()[0])
        _lib.set_option("kernel", 0)
mb.close()
for name, v in out.items():
    print(json.dumps({"path": name, "ms_per_pose": v, "median": statistics.median(v)}))
import numpy as np  # noqa: E402
print(json.dumps({"hits_equal": all(a[12] == b[12] for a, b in slots.values()),
                  "max_rel": max(float(np.abs(a[:12] - b[:12]).max() / max(np.abs(a[:12]).max(), 1e-300))
                                 for a, b in slots.values())}))
