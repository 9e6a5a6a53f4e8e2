"""Multi-GPU partitioning of the hot path (one process per GPU).

* Poses (config C4) are independent: ``pose_shard`` gives each rank a
  contiguous block; the map and bundle are replicated; there is NO data-path
  collective.
* One pose whose rays are split across GPUs (config C5): each rank reduces
  its contiguous ray range to the reference's 13-slot (the partial-sum
  contract of rmpnav/_kernels/_pool.py:1-7, 61-72 and rmpnav/core.py:130-136,
  "accepts pre-reduced partial results"), the slots are exchanged and
  folded in FIXED rank order with the reference's pairwise-fold shape, then
  solved -- identically on every rank, so the result is deterministic and
  rank-independent.  An all-reduce(sum) would make the summation order
  NCCL's choice.  Two exchange paths with bitwise-equal results:
  - ``FusedRaySplit`` (the product path on GPUs): ONE kernel per rank traces
    its rays, stores the slot into every rank's mailbox over NVLink peer
    memory (CUDA IPC), waits for the others' epochs, folds and solves
    (``RayPolicyEngine.exchange``, librmpb K4);
  - ``split_ray_policy``: partial kernel, ``all_gather`` (NCCL / gloo), fold
    kernel -- the baseline, and what the CPU tests drive with the oracle.
"""

from __future__ import annotations


def balanced_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [begin, end) share of n items for ``rank`` of ``world``."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world / rank")
    q, r = divmod(int(n), int(world))
    begin = rank * q + min(rank, r)
    return begin, begin + q + (1 if rank < r else 0)


def pose_shard(n_poses: int, world: int, rank: int) -> slice:
    b, e = balanced_range(n_poses, world, rank)
    return slice(b, e)


def gather_slots(slot, group=None):
    """All-gather one 13-slot per rank -> (world, 13) tensor in rank order."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out = [torch.empty_like(slot) for _ in range(world)]
    dist.all_gather(out, slot.contiguous(), group=group)
    return torch.stack(out)


def split_ray_policy(engine, x, v, group=None, resolve=None):
    """Evaluate ONE pose with its rays split across the ranks of ``group``.

    ``engine`` provides ``n_rays``, ``partial(x, v, begin, end)`` and
    ``resolve(slots) -> (slot13, accel3)`` (``device.RayPolicyEngine`` on
    GPUs).  Returns the same (slot, accel) on every rank."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    begin, end = balanced_range(engine.n_rays, world, rank)
    part = engine.partial(x, v, begin, end)
    slots = gather_slots(part, group)
    return (resolve or engine.resolve)(slots)


def exchange_handles(local: bytes, group=None) -> list:
    """All-gather one opaque handle (the 64-byte CUDA IPC mailbox handle)
    per rank, in rank order (setup only; any backend)."""
    import torch.distributed as dist

    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(local), group=group)
    return out


class FusedRaySplit:
    """Config C5 with the K4 fused exchange: every call evaluates one pose
    with its rays split over the ranks of ``group`` and returns the same
    (slot13, accel3) on every rank.  ``mailbox_factory(world, rank, device)``
    defaults to ``device.PeerMailbox``; the CPU tests inject a stand-in."""

    def __init__(self, engine, group=None, mailbox_factory=None):
        import torch.distributed as dist

        self.engine, self.group = engine, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if engine.n_rays < self.world:
            raise ValueError(f"{engine.n_rays} rays cannot be split over {self.world} ranks")
        if mailbox_factory is None:
            from .device import PeerMailbox as mailbox_factory
        self.mailbox = mailbox_factory(self.world, self.rank, getattr(engine, "device", None))
        self.mailbox.open(exchange_handles(self.mailbox.ipc_handle, group))
        self.range = balanced_range(engine.n_rays, self.world, self.rank)
        self.epoch = 0

    def __call__(self, x, v, stream=None):
        self.epoch += 1  # same sequence on every rank: calls are collective
        return self.engine.exchange(x, v, self.mailbox, self.epoch, self.range[0], self.range[1],
                                    3, stream=stream)
