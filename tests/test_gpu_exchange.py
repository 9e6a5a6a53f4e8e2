"""GPU: the K4 fused ray-split exchange (config C5) on ONE GPU.

The fused kernel traces a rank's ray range, stores its 13-slot into every
rank's mailbox over peer memory, waits for all epochs, folds in rank order
and solves.  Its result must be BITWISE equal to the baseline path
(per-range partial kernel + all-gather + fold kernel) and to every other
rank's.  Ranks are never run concurrently here: the split modes (1 = post
only, 2 = wait only) let one GPU run rank k's post before rank j's wait, so
no kernel ever waits on a kernel that has not finished."""

import os
import socket

import numpy as np
import pytest
import torch

from conftest import ROOT, STATIC_MAP, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def world_small(oracle):
    from paper_2301_08068_b200 import synth
    from paper_2301_08068_b200._kernels import b200
    from paper_2301_08068_b200.device import RayPolicyEngine

    scene = synth.c1_scene(n_boxes=20, hi=np.array([5.9, 5.9, 2.9]))
    vals = b200.bake_values(scene.packed(), np.zeros(3), 0.1, (60, 60, 30))
    vals = vals.astype(np.float32).astype(np.float64)
    dirs = oracle.sample_directions(20000)
    eng = RayPolicyEngine(b200.DeviceGrid(vals, np.zeros(3), 0.1),
                          b200.DeviceBundle(dirs), STATIC_MAP, 10.0)
    x = torch.tensor([3.0, 3.1, 1.4], dtype=torch.float64, device="cuda")
    v = torch.tensor([0.6, -0.3, 0.1], dtype=torch.float64, device="cuda")
    return eng, x, v, vals, dirs


def baseline(eng, x, v, world):
    from paper_2301_08068_b200.parallel import balanced_range

    parts = [eng.partial(x, v, *balanced_range(eng.n_rays, world, r)) for r in range(world)]
    return eng.resolve(torch.stack(parts))


@pytest.fixture(params=[0, 1, 2], ids=["auto", "lean", "refill"])
def kernel_opt(request):
    """Run with librmpb option `kernel` = auto / the lean kernel / the refill
    kernel k_ray_policy2: the K4 epilogue is compiled into both."""
    from paper_2301_08068_b200 import _lib

    _lib.set_option("kernel", request.param)
    yield request.param
    _lib.set_option("kernel", 0)


def test_exchange_world1_equals_partial_fold(world_small, oracle, kernel_opt):
    from paper_2301_08068_b200.device import PeerMailbox

    eng, x, v, vals, dirs = world_small
    mb = PeerMailbox(1, 0)
    ref_slot, ref_acc = baseline(eng, x, v, 1)
    for epoch in (1, 2, 3, 4):  # both parities, twice
        slot, acc = eng.exchange(x, v, mb, epoch, 0, eng.n_rays)
        torch.cuda.synchronize()
        assert torch.equal(slot, ref_slot) and torch.equal(acc, ref_acc)
    assert not mb.timed_out()
    # and the oracle (sums to 1e-9 relative, like the fused single-pose path)
    o_slot, o_acc, _ = oracle.ray_policy(vals, np.zeros(3), 0.1, x.cpu().numpy(),
                                         v.cpu().numpy(), dirs, STATIC_MAP, 10.0)
    s = slot.cpu().numpy()
    assert s[12] == o_slot[12] and rel_err(s[:12], o_slot[:12]) <= 1e-9
    assert rel_err(acc.cpu().numpy(), o_acc) <= 1e-6


@pytest.mark.parametrize("world", [2, 3, 8])
def test_exchange_same_process_ranks_sequential(world_small, world, kernel_opt):
    from paper_2301_08068_b200.device import EX_POST, EX_WAIT, PeerMailbox
    from paper_2301_08068_b200.parallel import balanced_range

    eng, x, v, _, _ = world_small
    mbs = [PeerMailbox(world, r) for r in range(world)]
    for a in mbs:
        for b in mbs:
            if a is not b:
                a.attach(b)
    ref_slot, ref_acc = baseline(eng, x, v, world)
    rng = [balanced_range(eng.n_rays, world, r) for r in range(world)]
    for epoch in (1, 2, 3):
        # ranks 1..W-1 post; rank 0 posts and waits; ranks 1..W-1 wait
        for r in range(1, world):
            eng.exchange(x, v, mbs[r], epoch, *rng[r], mode=EX_POST)
        outs = [eng.exchange(x, v, mbs[0], epoch, *rng[0], mode=EX_POST | EX_WAIT)]
        for r in range(1, world):
            outs.append(eng.exchange(x, v, mbs[r], epoch, *rng[r], mode=EX_WAIT))
        torch.cuda.synchronize()
        for slot, acc in outs:
            assert torch.equal(slot, ref_slot) and torch.equal(acc, ref_acc)
    assert not any(m.timed_out() for m in mbs)


def test_exchange_rejects_bad_arguments(world_small):
    from paper_2301_08068_b200.device import PeerMailbox

    eng, x, v, _, _ = world_small
    mb = PeerMailbox(2, 0)  # rank 1 never opened
    with pytest.raises(ValueError):
        eng.exchange(x, v, mb, 1, 0, 100)
    mb1 = PeerMailbox(1, 0)
    with pytest.raises(ValueError):
        eng.exchange(x, v, mb1, 0, 0, 100)      # epoch 0
    with pytest.raises(ValueError):
        eng.exchange(x, v, mb1, 1, 10, 5)       # bad range
    with pytest.raises(ValueError):
        PeerMailbox(9, 0)


def _ipc_worker(rank, port, q):
    """Two processes on cuda:0: the real CUDA-IPC mailbox path, ranks run one
    after another (gloo barriers order them)."""
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        import oracle as O
        from paper_2301_08068_b200 import parallel, synth
        from paper_2301_08068_b200._kernels import b200
        from paper_2301_08068_b200.device import EX_POST, EX_WAIT, PeerMailbox, RayPolicyEngine

        scene = synth.c1_scene(n_boxes=20, hi=np.array([5.9, 5.9, 2.9]))
        vals = O.bake_values(scene.packed(), np.zeros(3), 0.1, (60, 60, 30))
        vals = vals.astype(np.float32).astype(np.float64)
        dirs = O.sample_directions(20000)
        eng = RayPolicyEngine(b200.DeviceGrid(vals, np.zeros(3), 0.1), b200.DeviceBundle(dirs),
                              STATIC_MAP, 10.0)
        x = torch.tensor([3.0, 3.1, 1.4], dtype=torch.float64, device="cuda")
        v = torch.tensor([0.6, -0.3, 0.1], dtype=torch.float64, device="cuda")
        mb = PeerMailbox(2, rank, 0)
        mb.open(parallel.exchange_handles(mb.ipc_handle))
        b, e = parallel.balanced_range(eng.n_rays, 2, rank)
        res = None
        for epoch in (1, 2):
            if rank == 1:
                eng.exchange(x, v, mb, epoch, b, e, mode=EX_POST)
                torch.cuda.synchronize()
            dist.barrier()
            if rank == 0:
                res = eng.exchange(x, v, mb, epoch, b, e, mode=EX_POST | EX_WAIT)
                torch.cuda.synchronize()
            dist.barrier()
            if rank == 1:
                res = eng.exchange(x, v, mb, epoch, b, e, mode=EX_WAIT)
                torch.cuda.synchronize()
            dist.barrier()
        ref = eng.resolve(torch.stack([eng.partial(x, v, *parallel.balanced_range(eng.n_rays, 2, r))
                                       for r in range(2)]))
        q.put((rank, res[0].cpu().numpy(), res[1].cpu().numpy(), ref[0].cpu().numpy(),
               ref[1].cpu().numpy(), mb.timed_out()))
        mb.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_exchange_cuda_ipc_two_processes():
    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r[0], r[1:]) for r in (q.get(timeout=240) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        slot, acc, rslot, racc, to = res[r]
        assert not to
        assert np.array_equal(slot, rslot) and np.array_equal(acc, racc)
    assert np.array_equal(res[0][0], res[1][0])
