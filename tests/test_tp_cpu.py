"""Tensor-parallel host logic on CPU: world_size-2 gloo process group, NCCL unique-id
broadcast, per-rank ff slices, all-reduce of the per-rank partial outputs == unsplit
output (the algebra the GPU path's per-layer all-reduce relies on)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import inputs
    import oracle
    from paper_2512_16473_b200 import tp
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nid = tp.broadcast_nccl_id()
        d, ff, n, K, L, T = 64, 256, 8, 2, 2, 5
        lo, hi = tp.ff_slice(ff, world, rank)
        gates = [inputs.gate_weights(l, n, d) for l in range(L)]
        tr = inputs.generate_trace(L, n, K, T, inputs.PRESETS["paper"](n))
        x, _ = inputs.make_hidden(tr, gates)
        part = oracle.decode(x, gates, lambda l, e: inputs.expert_weights(l, e, d, ff, rank, world),
                             N=L, M=2, K=K)
        y = torch.from_numpy(part.y.astype(np.float64))
        dist.all_reduce(y)
        ids = torch.tensor(list(nid), dtype=torch.int64)
        ids0 = ids.clone()
        dist.broadcast(ids0, src=0)
        exp = torch.tensor([int(v) for v in part.records["expert"]], dtype=torch.int64)
        exp0 = exp.clone()
        dist.broadcast(exp0, src=0)
        if rank == 0:
            full = oracle.decode(x, gates, lambda l, e: inputs.expert_weights(l, e, d, ff), N=L, M=2, K=K)
            err = float((y.numpy() - full.y).__abs__().max() / np.abs(full.y).max())
            q.put(("ok", err, bool(torch.equal(ids, ids0)), bool(torch.equal(exp, exp0)), (lo, hi)))
        else:
            q.put(("rank1", None, bool(torch.equal(ids, ids0)), bool(torch.equal(exp, exp0)), (lo, hi)))
    finally:
        dist.destroy_process_group()


def test_tp2_gloo_partials_allreduce_to_full_output():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    r0 = next(r for r in res if r[0] == "ok")
    r1 = next(r for r in res if r[0] == "rank1")
    assert r0[1] < 1e-5                      # sum of slices == unsplit layer
    assert r0[2] and r1[2]                   # same NCCL id on both ranks
    assert r0[3] and r1[3]                   # identical routing on both ranks
    assert r0[4] == (0, 128) and r1[4] == (128, 256)


def test_ff_slice_validation():
    from paper_2512_16473_b200 import tp
    assert tp.ff_slice(16384, 8, 7) == (14336, 16384)
    with pytest.raises(ValueError):
        tp.ff_slice(100, 4, 0)


class _FakeMoe:
    """Stands in for a TP context: records the handles tp.connect_peers hands it."""

    def __init__(self, rank, world, fail=False):
        self.tp_size, self.tp_rank = world, rank
        self.got = None
        self.fail = fail
        self.disconnected = False

    def tp_exchange_buffer(self):
        return {"dev_ptr": 0, "bytes": 0, "ipc_handle": bytes([self.tp_rank + 1]) * 64}

    def tp_connect_ipc(self, handles):
        self.got = handles
        if self.fail:
            raise RuntimeError("no P2P")

    def tp_disconnect(self):
        self.disconnected = True


def _connect_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_2512_16473_b200 import tp
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = _FakeMoe(rank, world)
        ok = tp.connect_peers(m)
        bad = _FakeMoe((rank + 1) % world, world)
        try:
            tp.connect_peers(bad)
            mismatch = False
        except ValueError:
            mismatch = True
        # rank 1 cannot open its peers: every rank must fall back together
        f = _FakeMoe(rank, world, fail=(rank == 1))
        why = tp.connect_peers(f)
        q.put((rank, m.got, mismatch, ok, why, f.disconnected))
    finally:
        dist.destroy_process_group()


def test_fused_tp_connect_gathers_ipc_handles_in_rank_order():
    """f3 host logic (world_size 2, gloo): every rank receives all ranks' 64-byte exchange
    handles in rank order and a context whose rank disagrees with the group is refused."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 2
    procs = [ctx.Process(target=_connect_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [bytes([r + 1]) * 64 for r in range(world)]
    for rank, got, mismatch, ok, why, disconnected in res:
        assert got == want and mismatch and ok == "fused-peer"
        assert why == "rank 1: no P2P"
        assert disconnected == (rank == 0)   # the rank that did connect reverts


def _group_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import bench
    g = bench.Group(world)          # bench.py's N>1 plumbing: gloo, CPU tensors
    try:
        g.barrier()
        q.put((rank, g.max(1.5 + rank)))
    finally:
        g.close()


def test_bench_group_max_over_ranks_gloo():
    """bench.py's multi-rank timing reduction (the device-timed region's max over ranks) over the
    gloo group it uses for all N>1 plumbing — no NCCL needed unless the fused peer reduction
    cannot be wired."""
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_group_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == {0: 2.5, 1: 2.5}
