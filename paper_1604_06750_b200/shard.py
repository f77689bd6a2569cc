"""Multi-GPU source sharding (SURVEY.md §8e option 1).

Sources are independent (the off-line ROM does not depend on them,
PAPER.md:15-17), so N GPUs each hold a replica of the operator and advance a
disjoint slice of the S sources; there is no collective on the data path.
Traces are gathered once at the end (all_gather over torch.distributed:
NCCL on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np


def shard_range(S: int, world: int, rank: int):
    """Contiguous source slice [lo, hi) of `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(S, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def shard_sources(g: np.ndarray, world: int, rank: int) -> np.ndarray:
    """This rank's columns of the projected sources g~ [sum_f M_f, S]."""
    lo, hi = shard_range(g.shape[1], world, rank)
    return np.ascontiguousarray(g[:, lo:hi])


def gather_traces(local: np.ndarray, S: int, group=None) -> np.ndarray:
    """Reassemble [steps+1, R, S] traces from every rank's [steps+1, R, S_r]
    slice (torch.distributed all_gather; padded to the largest slice)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    width = max(hi - lo for lo, hi in (shard_range(S, world, r) for r in range(world)))
    T, R, Sr = local.shape
    buf = np.zeros((T, R, width))
    buf[:, :, :Sr] = local
    t = torch.from_numpy(buf)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t, group=group)
    out = np.zeros((T, R, S))
    for r, p in enumerate(parts):
        lo, hi = shard_range(S, world, r)
        out[:, :, lo:hi] = p.cpu().numpy()[:, :, :hi - lo]
    return out
