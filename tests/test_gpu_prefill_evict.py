"""Prefill (f4) with evictions inside the prompt (ways M < n): moe_layer_prefill must still be
exactly T successive moe_layer_forward calls for the cache (routing, hit / miss / way /
evicted sequence, counters), the expert FFN runs batched on the tensor cores with experts that
are no longer resident at the end of the prompt read from the prefill staging area, and the
cache it leaves behind must serve the following decode calls (their traces and outputs are
checked too). Bar: trace fields bit-exact, y within 1e-2 (h is rounded to bf16 between the two
GEMMs)."""
import numpy as np
import pytest

import harness
import inputs
import oracle
import paper_2512_16473_b200 as moe
from test_gpu_parity import EXACT_FIELDS, STAT_KEYS, TOL

pytestmark = pytest.mark.gpu


def _run(hm, x, M, warm, policy, mode, T_pre):
    """Prefill tokens [0, T_pre) layer by layer, then decode the rest token by token."""
    import torch
    T, L, d = x.shape
    dev = torch.device("cuda", 0)
    y = np.zeros((T, L, d), np.float32)
    with harness.open_moe(hm) as m:
        m.configure(ways=M, indexes=L, warm_start=warm, policy=policy, miss_mode=mode)
        yp = torch.empty((T_pre, d), dtype=torch.float32, device=dev)
        for l in range(L):
            xl = torch.from_numpy(np.ascontiguousarray(x[:T_pre, l, :]).view(np.int16)).to(dev)
            m.prefill(l, xl.data_ptr(), yp.data_ptr(), T_pre)
            torch.cuda.synchronize()
            y[:T_pre, l] = yp.cpu().numpy()
        if T > T_pre:
            y[T_pre:] = harness.run_decode(m, np.ascontiguousarray(x[T_pre:]))
        tr = m.trace()
        st = [m.stats(l) for l in range(L)]
    return y, tr, st


def _check(hm, x, ref, y, tr, st, T_pre):
    T, L, _ = x.shape
    K = hm.K
    # the prompt's records are layer-major, the decode tail's token-major: compare by key
    order = np.lexsort((tr["rank"], tr["layer"], tr["token"]))
    got = tr[order]
    for f in EXACT_FIELDS:
        np.testing.assert_array_equal(got[f].astype(np.int64), ref.records[f].astype(np.int64), err_msg=f)
    np.testing.assert_allclose(got["weight"], ref.records["weight"], rtol=1e-5, atol=1e-6)
    for l in range(L):
        for k in STAT_KEYS:
            assert st[l][k] == ref.stats[l][k], (l, k)
        assert st[l]["fetches"] == st[l]["expert_misses"]
    worst = max(float(np.abs(y[t, l] - ref.y[t, l]).max() / np.abs(ref.y[t, l]).max())
                for t in range(T) for l in range(L))
    assert worst <= TOL, worst
    assert sum(s["evictions"] for s in st) > 0        # the prompt really evicted


@pytest.mark.parametrize("M,warm,policy,mode", [(2, False, moe.POLICY_LRU, moe.MISS_FETCH),
                                                (3, True, moe.POLICY_LRU, moe.MISS_PULL),
                                                (4, False, moe.POLICY_FIFO, moe.MISS_FETCH),
                                                (2, True, moe.POLICY_FIFO, moe.MISS_PULL),
                                                (7, False, moe.POLICY_LRU, moe.MISS_PULL)])
def test_prefill_with_evictions_tiny(M, warm, policy, mode):
    c = inputs.CONFIGS["tiny"]
    hm = harness.host_model(c["L"], c["d"], c["ff"], c["n"], c["K"])
    T, T_pre = 48, 40
    x, _ = harness.hidden_states(hm, T, "paper")
    opol = oracle.LRU if policy == moe.POLICY_LRU else oracle.FIFO
    ref = oracle.decode(x, hm.gates, lambda l, e: inputs.expert_weights(l, e, hm.d, hm.ff), N=hm.L, M=M, K=hm.K,
                        policy=opol, warm_start=warm)
    y, tr, st = _run(hm, x, M, warm, policy, mode, T_pre)
    _check(hm, x, ref, y, tr, st, T_pre)


def test_prefill_with_evictions_long_prompt_multi_tile():
    """600 tokens: several 128-row m-tiles per expert, most experts evicted and re-fetched
    many times inside the prompt."""
    c = inputs.CONFIGS["tiny"]
    hm = harness.host_model(1, c["d"], c["ff"], c["n"], c["K"])
    T = 600
    x, _ = harness.hidden_states(hm, T, "uniform")
    ref = oracle.decode(x, hm.gates, lambda l, e: inputs.expert_weights(l, e, hm.d, hm.ff), N=1, M=3, K=hm.K)
    y, tr, st = _run(hm, x, 3, False, moe.POLICY_LRU, moe.MISS_FETCH, T)
    _check(hm, x, ref, y, tr, st, T)


@pytest.mark.slow
@pytest.mark.parametrize("name,M,T,mode", [("mixtral-8x7b", 2, 192, moe.MISS_FETCH), ("phi-3.5-moe", 4, 256, moe.MISS_PULL)])
def test_prefill_with_evictions_full_shape_sampled(name, M, T, mode):
    """BASELINE expert shapes, cold cache: trace and counters bit-exact for every token, y on
    sampled tokens, then two decode tokens on the cache the prompt left behind."""
    c = inputs.CONFIGS[name]
    hm = harness.host_model(1, c["d"], c["ff"], c["n"], c["K"])
    x, _ = harness.hidden_states(hm, T + 2, "paper")
    sample = [0, 1, 127, T // 2, T - 1, T, T + 1]
    ref = oracle.decode(x, hm.gates, lambda l, e: inputs.expert_weights(l, e, hm.d, hm.ff), N=1, M=M, K=c["K"],
                        tokens=sample)
    y, tr, st = _run(hm, x, M, False, moe.POLICY_LRU, mode, T)
    order = np.lexsort((tr["rank"], tr["layer"], tr["token"]))
    for f in EXACT_FIELDS:
        np.testing.assert_array_equal(tr[order][f].astype(np.int64), ref.records[f].astype(np.int64), err_msg=f)
    for k in STAT_KEYS:
        assert st[0][k] == ref.stats[0][k], k
    worst = max(float(np.abs(y[t, 0] - ref.y[t, 0]).max() / np.abs(ref.y[t, 0]).max()) for t in sample)
    assert worst <= TOL, worst
