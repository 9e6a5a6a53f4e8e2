"""TWO GPUs (marker ``gpu2``; skipped with fewer than 2 devices): the K4
fused ray split with the ranks spinning on EACH OTHER'S mailboxes
concurrently, on different GPUs over NVLink peer memory -- the case the
one-GPU tests cannot run.  Launched as 2 processes (one per GPU, NCCL for
the setup and the all-gather baseline); every rank's fused result must be
bitwise equal on both ranks and agree with the all-gather path and the
single-GPU evaluation of the whole pose.

    python -m pytest tests/test_gpu2_ray_split.py -m gpu2
"""

import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu2

WORKER = r'''
import os, sys, json
sys.path.insert(0, os.environ["RMPB_ROOT"])
import numpy as np, torch, torch.distributed as dist
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
os.environ["RMPNAV_DEVICE"] = str(rank)
from paper_2301_08068_b200 import synth
from paper_2301_08068_b200._kernels import b200
from paper_2301_08068_b200.device import RayPolicyEngine
from paper_2301_08068_b200.parallel import FusedRaySplit, split_ray_policy
b200.set_device(rank)
STATIC = (88.0, 1.4, 140.0, 1.2, 1e-6, 2.4, 0.2)
scene = synth.c1_scene()
grid = synth.c1_grid(scene)
states = synth.bench_states(scene, count=6, seed=123)
eng = RayPolicyEngine(grid, b200.DeviceBundle(halton_n=1 << 18, device=rank), STATIC, 10.0,
                      device=rank)
split = FusedRaySplit(eng)
out = []
for rep in range(3):                      # epochs of both parities, repeated
    for st in states:
        x = torch.tensor(st.position, dtype=torch.float64, device="cuda")
        v = torch.tensor(st.velocity, dtype=torch.float64, device="cuda")
        fs, fa = split(x, v)
        gs, ga = split_ray_policy(eng, x, v)
        ws, wa = eng.evaluate(x.view(1, 3), v.view(1, 3))
        torch.cuda.synchronize()
        out.append([fs.cpu().tolist(), fa.cpu().tolist(), gs.cpu().tolist(), ws[0].cpu().tolist()])
assert not split.mailbox.timed_out()
allr = [None] * world
dist.all_gather_object(allr, out)
if rank == 0:
    print("RESULT " + json.dumps(allr))
dist.destroy_process_group()
'''


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_fused_ray_split_two_gpus_concurrent(tmp_path):
    import json

    import numpy as np
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    env = dict(os.environ, RMPB_ROOT=ROOT)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node=2", "--master-addr=127.0.0.1",
                        f"--master-port={_free_port()}", str(script)],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("RESULT ")][0]
    res = json.loads(line[len("RESULT "):])
    r0, r1 = res
    for a, b in zip(r0, r1):
        assert a[0] == b[0] and a[1] == b[1]          # fused: bitwise equal on both ranks
        f, g, w = (np.array(a[k]) for k in (0, 2, 3))
        assert f[12] == g[12] == w[12]               # hit counts exact
        sc = max(1e-300, np.abs(w[:12]).max())
        assert np.abs(f[:12] - g[:12]).max() <= 1e-12 * sc
        assert np.abs(f[:12] - w[:12]).max() <= 1e-12 * sc
