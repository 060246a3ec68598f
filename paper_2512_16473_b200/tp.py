"""Tensor-parallel plumbing (north_star (4)): one process per GPU, torch.distributed for
the process group; the per-layer sum of y either fused into the decode kernel over peer
memory (f3: ``connect_peers``, CUDA IPC handles all-gathered here) or NCCL's all-reduce
inside libmoe.so (``broadcast_nccl_id``).

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


def exchange_handles(own: bytes, group=None) -> list[bytes]:
    """All-gather every rank's 64-byte exchange-buffer IPC handle, in rank order."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, own, group=group)
    if any(not isinstance(h, (bytes, bytearray)) or len(h) != 64 for h in out):
        raise RuntimeError("bad IPC handle from a peer")
    return [bytes(h) for h in out]


def connect_peers(m, group=None) -> str:
    """f3: wire the fused peer-memory reduction of y for context ``m`` (one rank per
    process): all-gather the ranks' exchange-buffer IPC handles, open the peers', and agree
    on the outcome. If any rank failed (no P2P / IPC), every rank disconnects and the
    context keeps its NCCL all-reduce. Returns "fused-peer" or the failure reason. The
    final collective doubles as the barrier that keeps a rank's first call from reaching a
    peer whose counters are not yet reset."""
    import torch.distributed as dist
    if dist.get_world_size(group) != m.tp_size or dist.get_rank(group) != m.tp_rank:
        raise ValueError("process group does not match the context's tp_size / tp_rank")
    why = ""
    try:
        own = m.tp_exchange_buffer()["ipc_handle"]
    except Exception as e:  # noqa: BLE001 - reported to every rank below
        own, why = bytes(64), f"rank {m.tp_rank}: {e}"
    handles = exchange_handles(own, group)
    if not why:
        try:
            m.tp_connect_ipc(handles)
        except Exception as e:  # noqa: BLE001
            why = f"rank {m.tp_rank}: {e}"
    whys = [None] * dist.get_world_size(group)
    dist.all_gather_object(whys, why, group=group)
    bad = [w for w in whys if w]
    if bad:
        if not why:
            m.tp_disconnect()
        dist.barrier(group)
        return "; ".join(bad)
    return "fused-peer"
