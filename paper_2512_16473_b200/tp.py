"""Tensor-parallel plumbing (north_star (4)): one process per GPU, torch.distributed for
the process group, NCCL (inside libmoe.so) for the per-layer all-reduce.

Each rank holds the ff-slice of every expert; gate weights, routing and the cache
directory are replicated (the router kernel is deterministic), so every rank takes the
same cache decisions and only y is exchanged.
"""
from __future__ import annotations

from . import nccl_unique_id


def broadcast_nccl_id(group=None, src: int = 0) -> bytes:
    """Rank `src` creates the 128-byte NCCL unique id; every rank returns it (torch.distributed)."""
    import torch.distributed as dist
    obj = [nccl_unique_id() if dist.get_rank() == src else None]
    dist.broadcast_object_list(obj, src=src, group=group)
    return obj[0]


def ff_slice(ff: int, tp_size: int, tp_rank: int) -> tuple[int, int]:
    """[lo, hi) rows of W1/W3 (and columns of W2) held by tp_rank (moe.h: ff % (8*P) == 0)."""
    if ff % (8 * tp_size):
        raise ValueError("d_ff must be a multiple of 8 * tp_size")
    ffr = ff // tp_size
    return tp_rank * ffr, (tp_rank + 1) * ffr
