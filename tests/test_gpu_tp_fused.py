"""f3 on one GPU: the fused peer-memory TP reduction (moe.h moe_tp_connect_local).

P ranks of one ff-split TP group are P contexts in this process on cuda:0 (each holding its
ff/P slice of every expert, no NCCL communicator). moe_tp_connect_local wires their
exchange buffers; the contexts then split the SMs (grid = #SMs / P each) so the P decode
kernels of one layer are co-resident and exchange y^(p) inside their epilogues exactly as
they would over NVLink between GPUs (same code path: plain stores to the peers' buffers,
system-scope release/acquire counters). Checked against the UNSPLIT oracle:
  - every rank's access trace and counters bit-exact (replicated deterministic routing);
  - every rank's y bit-identical to every other rank's (fixed-order sum of the slots);
  - y within the north_star bar (1e-2; asserted 1e-4) of the oracle's unsplit layer.
"""
import numpy as np
import pytest

import harness
import inputs
import oracle
import paper_2512_16473_b200 as moe

pytestmark = pytest.mark.gpu

TIGHT = 1e-4
EXACT_FIELDS = ("token", "layer", "rank", "hit", "expert", "evicted", "way", "coverage")
STAT_KEYS = ("accesses", "at_least_one_hit", "all_k_hit", "expert_hits", "expert_misses",
             "coverage_misses", "evictions")


def _run_group(full, P, x, ways, indexes, miss_mode=moe.MISS_FETCH, policy=moe.POLICY_LRU):
    import torch
    hps = [harness.host_model(full.L, full.d, full.ff, full.n, full.K, tp_size=P, tp_rank=p) for p in range(P)]
    ms = [harness.open_moe(hp) for hp in hps]
    try:
        for m in ms:
            m.configure(ways=ways, indexes=indexes, miss_mode=miss_mode, policy=policy, seed=5)
        moe.tp_connect_local(ms)
        infos = [m.runtime_info() for m in ms]
        T, L, d = x.shape
        dev = torch.device("cuda", 0)
        xd = torch.from_numpy(x.view(np.int16)).to(dev)
        yd = torch.empty((P, T, L, d), dtype=torch.float32, device=dev)
        streams = [torch.cuda.Stream(dev) for _ in range(P)]
        torch.cuda.synchronize()
        for t in range(T):
            for l in range(L):
                for p in range(P):  # one layer's calls are enqueued for every rank first
                    ms[p].forward(l, xd[t, l].data_ptr(), yd[p, t, l].data_ptr(), streams[p].cuda_stream)
        for s in streams:
            s.synchronize()
        traces = [m.trace() for m in ms]
        stats = [[m.stats(l) for l in range(L)] for m in ms]
        return yd.cpu().numpy(), traces, stats, infos
    finally:
        for m in ms:
            m.close()


def _check(full, P, x, ys, traces, stats, infos, ref):
    import torch
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    for info in infos:
        assert info["tp_reduce"] == "fused-peer" and info["expert_path"] == "fused"
        assert info["grid"] == nsm // P and not info["pdl"]
    for p in range(P):
        for f in EXACT_FIELDS:
            np.testing.assert_array_equal(traces[p][f].astype(np.int64), ref.records[f].astype(np.int64),
                                          err_msg=f"rank {p} {f}")
        for l in range(full.L):
            for k in STAT_KEYS:
                assert stats[p][l][k] == ref.stats[l][k], (p, l, k)
        # all ranks hold the same bits (fixed-order sum of the same slots)
        assert np.array_equal(ys[p].view(np.uint32), ys[0].view(np.uint32)), f"rank {p} differs from rank 0"
    T = x.shape[0]
    worst = 0.0
    for t in range(T):
        for l in range(full.L):
            r = ref.y[t, l]
            worst = max(worst, float(np.abs(ys[0][t, l] - r).max() / np.abs(r).max()))
    assert worst <= TIGHT, worst
    return worst


@pytest.mark.parametrize("P", [2, 4, 8])
def test_fused_peer_reduce_matches_unsplit_oracle(P):
    L, d, ff, n, K, T = 2, 256, 1024, 8, 2, 6
    full = harness.host_model(L, d, ff, n, K)
    x, _ = harness.hidden_states(full, T, "paper")
    ref = oracle.decode(x, full.gates, lambda l, e: inputs.expert_weights(l, e, d, ff), N=L, M=2, K=K)
    ys, traces, stats, infos = _run_group(full, P, x, ways=2, indexes=L)
    _check(full, P, x, ys, traces, stats, infos, ref)


def test_fused_peer_reduce_uncovered_and_host_compute():
    """Misses through both modes: one covered layer (LRU, M=2) and one beyond coverage; the
    host cores compute this rank's slice of every missed expert."""
    L, d, ff, n, K, T, P = 2, 128, 512, 8, 2, 8, 2
    full = harness.host_model(L, d, ff, n, K)
    x, _ = harness.hidden_states(full, T, "paper")
    ref = oracle.decode(x, full.gates, lambda l, e: inputs.expert_weights(l, e, d, ff), N=1, M=2, K=K)
    for mode in (moe.MISS_FETCH, moe.MISS_HOST_COMPUTE):
        ys, traces, stats, infos = _run_group(full, P, x, ways=2, indexes=1, miss_mode=mode)
        _check(full, P, x, ys, traces, stats, infos, ref)


def test_fused_peer_reduce_top1():
    """K = 1: the kernel writes y^(p) directly (no reduction onto zero)."""
    L, d, ff, n, K, T, P = 2, 128, 256, 4, 1, 5, 2
    full = harness.host_model(L, d, ff, n, K)
    x, _ = harness.hidden_states(full, T, "paper")
    ref = oracle.decode(x, full.gates, lambda l, e: inputs.expert_weights(l, e, d, ff), N=L, M=2, K=K)
    ys, traces, stats, infos = _run_group(full, P, x, ways=2, indexes=L)
    _check(full, P, x, ys, traces, stats, infos, ref)


@pytest.mark.slow
def test_fused_peer_reduce_mixtral_8x22b_slice_shape():
    """BASELINE configs[4] per-rank shape (d = 6144, ff = 16384 split over P = 2: ff/P = 8192),
    one layer, warm M = 8 (all hits)."""
    c = inputs.CONFIGS["mixtral-8x22b"]
    L, T, P = 1, 3, 2
    full = harness.host_model(L, c["d"], c["ff"], c["n"], c["K"])
    x, _ = harness.hidden_states(full, T, "paper")
    ref = oracle.decode(x, full.gates, lambda l, e: inputs.expert_weights(l, e, full.d, full.ff),
                        N=L, M=c["n"], K=full.K, warm_start=True)
    ys, traces, stats, infos = _run_group_warm(full, P, x)
    _check(full, P, x, ys, traces, stats, infos, ref)


def _run_group_warm(full, P, x):
    import torch
    hps = [harness.host_model(full.L, full.d, full.ff, full.n, full.K, tp_size=P, tp_rank=p) for p in range(P)]
    ms = [harness.open_moe(hp) for hp in hps]
    try:
        for m in ms:
            m.configure(ways=full.n, indexes=full.L, warm_start=True)
        moe.tp_connect_local(ms)
        infos = [m.runtime_info() for m in ms]
        T, L, d = x.shape
        xd = torch.from_numpy(x.view(np.int16)).cuda()
        yd = torch.empty((P, T, L, d), dtype=torch.float32, device="cuda")
        streams = [torch.cuda.Stream() for _ in range(P)]
        torch.cuda.synchronize()
        for t in range(T):
            for l in range(L):
                for p in range(P):
                    ms[p].forward(l, xd[t, l].data_ptr(), yd[p, t, l].data_ptr(), streams[p].cuda_stream)
        for s in streams:
            s.synchronize()
        return yd.cpu().numpy(), [m.trace() for m in ms], [[m.stats(l) for l in range(L)] for m in ms], infos
    finally:
        for m in ms:
            m.close()


def test_tp_without_nccl_or_connect_is_rejected():
    import torch
    L, d, ff, n, K = 1, 64, 128, 8, 2
    hp = harness.host_model(L, d, ff, n, K, tp_size=2, tp_rank=0)
    with harness.open_moe(hp) as m:
        m.configure(ways=2, indexes=L)
        x = torch.zeros(d, dtype=torch.int16, device="cuda")
        y = torch.empty(d, dtype=torch.float32, device="cuda")
        with pytest.raises(moe.MoeError) as ei:
            m.forward(0, x.data_ptr(), y.data_ptr())
        assert ei.value.status == 5 and "moe_tp_connect" in str(ei.value)
        assert m.runtime_info()["tp_reduce"] == "none"
        e = m.tp_exchange_buffer()
        assert e["bytes"] == 256 + 2 * 2 * K * d * 8 and len(e["ipc_handle"]) == 64 and e["dev_ptr"]


def _ipc_worker(rank, world, port, q):
    import os
    import torch
    import torch.distributed as dist
    from paper_2512_16473_b200 import tp
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L, d, ff, n, K, T = 2, 256, 1024, 8, 2, 4
        hp = harness.host_model(L, d, ff, n, K, tp_size=world, tp_rank=rank)
        x, _ = harness.hidden_states(hp, T, "paper")
        with harness.open_moe(hp, device=0) as m:
            m.configure(ways=2, indexes=L)
            how = tp.connect_peers(m)
            y = harness.run_decode(m, x, device=0)
            tr = m.trace()
        q.put((rank, how, y, tr["expert"].copy(), tr["hit"].copy()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_fused_peer_reduce_two_processes_cuda_ipc():
    """The multi-process wiring (one process per rank, as under torchrun): exchange buffers
    mapped with CUDA IPC through tp.connect_peers (handles all-gathered over a gloo group),
    both ranks on cuda:0 (their kernels time-slice the GPU). Same bar: bit-identical y on both
    ranks, within 1e-4 of the unsplit oracle, routing equal to the oracle's."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=180) for _ in range(2)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    L, d, ff, n, K, T = 2, 256, 1024, 8, 2, 4
    full = harness.host_model(L, d, ff, n, K)
    x, _ = harness.hidden_states(full, T, "paper")
    ref = oracle.decode(x, full.gates, lambda l, e: inputs.expert_weights(l, e, d, ff), N=L, M=2, K=K)
    assert [r[1] for r in res] == ["fused-peer", "fused-peer"]
    assert np.array_equal(res[0][2].view(np.uint32), res[1][2].view(np.uint32))
    for r in res:
        np.testing.assert_array_equal(r[3].astype(np.int64), ref.records["expert"].astype(np.int64))
        np.testing.assert_array_equal(r[4].astype(np.int64), ref.records["hit"].astype(np.int64))
    worst = max(float(np.abs(res[0][2][t, l] - ref.y[t, l]).max() / np.abs(ref.y[t, l]).max())
                for t in range(T) for l in range(L))
    assert worst <= TIGHT, worst
