"""CPU, world size 2 over gloo: the multi-GPU host logic (pose shards, ray
split -> all_gather of 13-slots -> fixed-order fold -> solve) gives every
rank the same result, equal to the single-process evaluation.  The partial
slots come from the CPU oracle standing in for the device partial kernel."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import ROOT, STATIC_MAP, rel_err


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleEngine:
    """CPU stand-in with the RayPolicyEngine interface (partial / resolve)."""

    def __init__(self, vals, origin, res, dirs):
        import oracle as O

        self.O, self.vals, self.origin, self.res, self.dirs = O, vals, origin, res, dirs
        self.n_rays = dirs.shape[0]

    def partial(self, x, v, b, e):
        d = self.dirs[b:e]
        t = self.O.grid_trace(self.vals, self.origin, self.res, x.numpy(), d, 10.0,
                              0.5 * self.res, 0.9)
        return torch.from_numpy(self.O.policy_slot(d, t, v.numpy(), STATIC_MAP))

    def resolve(self, slots):
        s = self.O.pairwise_fold(slots.numpy())
        return torch.from_numpy(s), torch.from_numpy(self.O.accel_from_slot(s))


def _world(seed=0):
    rng = np.random.default_rng(seed)
    vals = (rng.normal(size=(30, 26, 22)) * 0.4 + 0.5).astype(np.float32).astype(np.float64)
    dirs = rng.normal(size=(5000, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    return vals, np.zeros(3), 0.1, dirs


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_2301_08068_b200 import parallel

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        vals, o, res, dirs = _world()
        eng = OracleEngine(vals, o, res, dirs)
        x = torch.tensor([1.3, 1.2, 1.0], dtype=torch.float64)
        v = torch.tensor([0.3, -0.8, 0.2], dtype=torch.float64)
        slot, acc = parallel.split_ray_policy(eng, x, v)
        sh = parallel.pose_shard(4096, world, rank)
        q.put((rank, slot.numpy(), acc.numpy(), (sh.start, sh.stop)))
    finally:
        dist.destroy_process_group()


def test_balanced_range_partitions():
    from paper_2301_08068_b200.parallel import balanced_range

    for n in (0, 1, 7, 65536, 1 << 20):
        for w in (1, 2, 3, 8):
            rs = [balanced_range(n, w, r) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(e - b for b, e in rs) - min(e - b for b, e in rs) <= 1


@pytest.mark.timeout(300)
def test_ray_split_over_gloo_world2(oracle):
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    # identical on every rank
    assert np.array_equal(res[0][1], res[1][1]) and np.array_equal(res[0][2], res[1][2])
    # equals the single-process evaluation (different association: 1e-12)
    vals, o, r, dirs = _world()
    x, v = np.array([1.3, 1.2, 1.0]), np.array([0.3, -0.8, 0.2])
    slot, acc, _ = oracle.ray_policy(vals, o, r, x, v, dirs, STATIC_MAP, 10.0)
    assert res[0][1][12] == slot[12]
    assert rel_err(res[0][1][:12], slot[:12]) < 1e-12
    assert rel_err(res[0][2], acc) < 1e-9
    # pose shards tile the pose set
    assert res[0][3] == (0, 2048) and res[1][3] == (2048, 4096)


class _StubMailbox:
    def __init__(self, world, rank, device):
        self.world, self.rank = world, rank
        self.ipc_handle = bytes([rank]) * 64
        self.opened = None

    def open(self, handles):
        self.opened = list(handles)


class _StubEngine:
    n_rays = 1001
    device = 0

    def exchange(self, x, v, mailbox, epoch, b, e, mode, stream=None):
        return (mailbox.rank, epoch, b, e, mode, mailbox.opened)


def _fused_worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_2301_08068_b200 import parallel

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fs = parallel.FusedRaySplit(_StubEngine(), mailbox_factory=_StubMailbox)
        outs = [fs(None, None) for _ in range(3)]
        q.put((rank, outs))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_fused_split_host_logic_gloo_world3():
    """Mailbox handles are exchanged in rank order, every rank gets its
    balanced ray range and the epochs advance identically (1, 2, 3)."""
    world = 3
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_fused_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    handles = [bytes([r]) * 64 for r in range(world)]
    from paper_2301_08068_b200.parallel import balanced_range

    for r in range(world):
        outs = res[r]
        assert [o[1] for o in outs] == [1, 2, 3]
        b, e = balanced_range(1001, world, r)
        for o in outs:
            assert o[0] == r and (o[2], o[3]) == (b, e) and o[4] == 3 and o[5] == handles
