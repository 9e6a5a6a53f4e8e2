"""Multi-GPU partitioning of the hot path (one process per GPU).

* Poses (config C4) are independent: ``pose_shard`` gives each rank a
  contiguous block; the map and bundle are replicated; there is NO data-path
  collective.
* One pose whose rays are split across GPUs (config C5): each rank reduces
  its contiguous ray range to the reference's 13-slot (the partial-sum
  contract of rmpnav/_kernels/_pool.py:1-7, 61-72 and rmpnav/core.py:130-136,
  "accepts pre-reduced partial results"), the slots are all-gathered (NCCL
  over NVLink on GPUs, gloo in the CPU tests) and folded in FIXED rank order
  with the reference's pairwise-fold shape, then solved -- identically on
  every rank, so the result is deterministic and rank-independent.  An
  all-reduce(sum) would make the summation order NCCL's choice.
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
