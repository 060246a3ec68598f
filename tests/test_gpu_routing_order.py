"""moe.h promises that moe_layer_prefill routes a prompt exactly like T successive
moe_layer_forward calls. With logits a margin apart that is a statement about the method;
with NEAR-TIED logits it is a statement about rounding: every kernel that computes the gate
logits must sum the same products in the same order (gate_gemv.cuh, DESIGN R25).

Construction: gate rows 1 and 2 are permutations of row 0 (reversed; rotated by d/2) and
every hidden state is invariant under both permutations (x_i = g(i mod d/2) with g
reflection-symmetric), so z_0 = z_1 = z_2 in exact arithmetic and only fp32 rounding —
i.e. the summation order — decides which two of the three are selected and in which rank
order. The other gate rows are scaled down so that they never compete. Decode (fused
kernel), decode (split router) and prefill must produce the identical trace and gate-weight
bits on every token — with 8 experts (the FHFMA form of the shared order) and with 12 and 16
(its tensor-core form, gate_mma_form)."""
import numpy as np
import pytest

import harness
import inputs
import paper_2512_16473_b200 as moe

pytestmark = pytest.mark.gpu

T = 96


def _tied_model(n):
    # d = 4096 (Mixtral's and Phi's model width: fp32 rounding of 4096-term sums is common),
    # small experts
    L, d, ff, K = 2, 4096, 128, 2
    hm = harness.host_model(L, d, ff, n, K)
    rng = np.random.default_rng(7)
    for l in range(L):
        g0 = rng.standard_normal(d).astype(np.float32)
        G = np.empty((n, d), np.float32)
        G[0] = g0
        G[1] = g0[::-1]
        G[2] = np.roll(g0, d // 2)
        G[3:] = 0.05 * rng.standard_normal((n - 3, d))
        hm.gates[l] = inputs.f32_to_bf16(G)
    x = np.empty((T, L, d), np.uint16)
    half = d // 2
    for t in range(T):
        for l in range(L):
            G = inputs.bf16_to_f32(hm.gates[l]).astype(np.float64)
            w0 = G[0]
            s0 = w0[:half] + w0[half:]                   # projection of row 0 on period-d/2 vectors
            u = rng.standard_normal(half)
            g = 0.5 * (s0 + s0[::-1]) + 0.5 * (u + u[::-1])   # + reflection-symmetric noise
            xx = np.concatenate([g, g]).astype(np.float32)
            x[t, l] = inputs.f32_to_bf16(xx)
            xf = inputs.bf16_to_f32(x[t, l]).astype(np.float64)
            assert np.array_equal(xf, xf[::-1]) and np.array_equal(xf, np.roll(xf, half))
            z = G @ xf
            if z[0] < 0:                                 # keep the tied three on top
                x[t, l] ^= np.uint16(0x8000)
                z = -z
            assert z[0] == z[1] == z[2] and z[0] > np.max(z[3:]) + 0.1, z
    return hm, x


def _decode(hm, x, monkeypatch, split):
    if split:
        monkeypatch.setenv("MOE_EXPERT_PATH", "split")
    with harness.open_moe(hm) as m:
        m.configure(ways=hm.n, indexes=hm.L, warm_start=True)
        harness.run_decode(m, x)
        tr = m.trace()
    monkeypatch.delenv("MOE_EXPERT_PATH", raising=False)
    return tr


def _prefill(hm, x):
    import torch
    dev = torch.device("cuda", 0)
    y = torch.empty((T, hm.d), dtype=torch.float32, device=dev)
    with harness.open_moe(hm) as m:
        m.configure(ways=hm.n, indexes=hm.L, warm_start=True)
        for l in range(hm.L):
            xl = torch.from_numpy(np.ascontiguousarray(x[:, l, :]).view(np.int16)).to(dev)
            m.prefill(l, xl.data_ptr(), y.data_ptr(), T)
        torch.cuda.synchronize()
        tr = m.trace()
    return tr[np.lexsort((tr["rank"], tr["layer"], tr["token"]))]


@pytest.mark.parametrize("n", [8, 12, 16])
def test_near_tied_logits_route_identically_on_every_path(monkeypatch, n):
    hm, x = _tied_model(n)
    fused = _decode(hm, x, monkeypatch, split=False)
    split = _decode(hm, x, monkeypatch, split=True)
    pre = _prefill(hm, x)
    # the near tie is real: the three tied experts take the top-2 slots, in varying order
    assert set(np.unique(fused["expert"])) <= {0, 1, 2}
    assert len({(int(a), int(b)) for a, b in fused["expert"].reshape(-1, 2)}) >= 2
    for f in ("expert", "hit", "way", "evicted", "rank", "token", "layer"):
        np.testing.assert_array_equal(fused[f], split[f], err_msg=f"split {f}")
        np.testing.assert_array_equal(fused[f], pre[f], err_msg=f"prefill {f}")
    np.testing.assert_array_equal(fused["weight"].view(np.uint32), split["weight"].view(np.uint32))
    np.testing.assert_array_equal(fused["weight"].view(np.uint32), pre["weight"].view(np.uint32))
