"""Pins for the oracle's arithmetic (router, expert FFN, combine) — CPU only.

Each test ties the oracle to something other than itself: float64 NumPy (library
routine), closed forms, special cases, brute force over all experts. A plausible
slip (dropped term, swapped W1/W3, transposed W2, softmax over all n instead of
the K, reversed tie-break, wrong weight index) fails at least one of them.
"""
import numpy as np
import pytest

import inputs
import oracle


def _rand_bf16(rng, shape, scale=1.0):
    return inputs.f32_to_bf16((rng.standard_normal(shape) * scale).astype(np.float32))


def _f64(a):
    return inputs.bf16_to_f32(a).astype(np.float64)


# ----------------------------------------------------------------------------- router
@pytest.mark.parametrize("n,d", [(8, 64), (16, 256), (32, 96)])
def test_gate_logits_match_float64_matmul(n, d):
    rng = np.random.default_rng(0)
    Wg, x = _rand_bf16(rng, (n, d), 0.1), _rand_bf16(rng, (d,))
    z, z64 = oracle.gate_logits(Wg, x)
    ref = _f64(Wg) @ _f64(x)
    np.testing.assert_allclose(z64, ref, rtol=0, atol=1e-12)
    np.testing.assert_allclose(z, ref, rtol=0, atol=1e-5 * (1 + np.abs(ref).max()))


def _brute_topk(z, K):
    order = sorted(range(len(z)), key=lambda e: (-float(z[e]), e))
    return order[:K]


@pytest.mark.parametrize("n,K", [(8, 1), (8, 2), (16, 2), (16, 5), (32, 4), (8, 8)])
def test_topk_softmax_brute_force(n, K):
    rng = np.random.default_rng(n * 100 + K)
    for trial in range(200):
        z = rng.standard_normal(n).astype(np.float32)
        if trial % 5 == 0:  # inject exact ties
            z[rng.integers(n)] = z[rng.integers(n)]
        S, w = oracle.topk_softmax(z, K)
        assert list(S) == _brute_topk(z, K)
        zs = z[S].astype(np.float64)
        ref = np.exp(zs - zs.max()) / np.exp(zs - zs.max()).sum()
        np.testing.assert_allclose(w, ref, rtol=1e-6, atol=1e-7)
        assert abs(float(w.astype(np.float64).sum()) - 1.0) < 1e-6
        assert np.all(np.diff(w) <= 0)  # rank order = descending gate weight


def test_topk_all_experts_when_k_equals_n():
    z = np.array([0.3, -1.0, 2.0, 0.3], np.float32)
    S, w = oracle.topk_softmax(z, 4)
    assert list(S) == [2, 0, 3, 1]  # tie 0.3: lower index first (reading R2)


def test_zero_input_tie_case():
    """x = 0 => z = 0 => S = {0, 1}, w = (1/2, 1/2) (reading R2)."""
    Wg = inputs.gate_weights(0, 8, 64)
    z, _ = oracle.gate_logits(Wg, np.zeros(64, np.uint16))
    S, w = oracle.topk_softmax(z, 2)
    assert list(S) == [0, 1]
    assert list(w) == [0.5, 0.5]


# ----------------------------------------------------------------------------- expert FFN
def _numpy_swiglu(W1, W3, W2, x):
    x = _f64(x)
    g, u = _f64(W1) @ x, _f64(W3) @ x
    h = g / (1.0 + np.exp(-g)) * u
    return _f64(W2) @ h, h


@pytest.mark.parametrize("d,ff", [(64, 128), (128, 64), (96, 160)])
def test_expert_ffn_matches_float64_numpy(d, ff):
    rng = np.random.default_rng(d + ff)
    W1, W3 = _rand_bf16(rng, (ff, d), d ** -0.5), _rand_bf16(rng, (ff, d), d ** -0.5)
    W2, x = _rand_bf16(rng, (d, ff), ff ** -0.5), _rand_bf16(rng, (d,))
    o, h = oracle.expert_ffn(W1, W3, W2, x)
    o_ref, h_ref = _numpy_swiglu(W1, W3, W2, x)
    assert np.abs(h - h_ref).max() <= 1e-5 * np.abs(h_ref).max()
    assert np.abs(o - o_ref).max() <= 1e-5 * np.abs(o_ref).max()
    # W1 / W3 are not interchangeable (silu applies to W1 x only)
    o_swapped, _ = _numpy_swiglu(W3, W1, W2, x)
    assert np.abs(o - o_swapped).max() > 1e-3 * np.abs(o_ref).max()


def test_expert_ffn_special_cases():
    rng = np.random.default_rng(5)
    d = ff = 32
    W1, W3, W2 = (_rand_bf16(rng, (ff, d), 0.2) for _ in range(3))
    zero = np.zeros(d, np.uint16)
    o, _ = oracle.expert_ffn(W1, W3, W2, zero)
    assert np.all(o == 0)                                   # x = 0 => y = 0
    x = _rand_bf16(rng, (d,))
    o, _ = oracle.expert_ffn(W1, np.zeros_like(W3), W2, x)
    assert np.all(o == 0)                                   # W3 = 0 => y = 0
    eye = inputs.f32_to_bf16(np.eye(d, dtype=np.float32))
    o, _ = oracle.expert_ffn(eye, eye, eye, x)              # W = I => y_c = silu(x_c) x_c
    xf = _f64(x)
    np.testing.assert_allclose(o, xf / (1 + np.exp(-xf)) * xf, rtol=1e-6, atol=1e-7)


def test_combine_is_weighted_sum_in_rank_order():
    o = np.array([[1.0, 2.0, -3.0], [4.0, 0.5, 1.0]], np.float32)
    w = np.array([0.75, 0.25], np.float32)
    np.testing.assert_array_equal(oracle.combine(o, w), np.array([1.75, 1.625, -2.0], np.float32))


# ----------------------------------------------------------------------------- full layer
def test_moe_layer_equals_dense_brute_force():
    """Evaluate ALL n experts, weight by g_e = w_r if e = S_r else 0 (north_star's dense check)."""
    cfg = inputs.CONFIGS["tiny"]
    L, d, ff, n, K = cfg["L"], cfg["d"], cfg["ff"], cfg["n"], cfg["K"]
    T = 6
    tr = inputs.generate_trace(L, n, K, T, inputs.PRESETS["paper"](n))
    gates = [inputs.gate_weights(l, n, d) for l in range(L)]
    x, ranked = inputs.make_hidden(tr, gates)
    W = {(l, e): inputs.expert_weights(l, e, d, ff) for l in range(L) for e in range(n)}
    res = oracle.decode(x, gates, lambda l, e: W[(l, e)], N=L, M=2, K=K)
    for t in range(T):
        for l in range(L):
            z = _f64(gates[l]) @ _f64(x[t, l])
            S = _brute_topk(z, K)
            zs = z[S]
            gw = np.exp(zs - zs.max()) / np.exp(zs - zs.max()).sum()
            g = np.zeros(n)
            g[S] = gw
            dense = sum(g[e] * _numpy_swiglu(*W[(l, e)], x[t, l])[0] for e in range(n))
            y = res.y[t, l]
            assert np.abs(y - dense).max() <= 1e-5 * np.abs(dense).max()
            recs = res.records[(t * L + l) * K:(t * L + l + 1) * K]
            assert list(recs["expert"]) == S == list(ranked[t, l])


def test_tp_ff_split_partials_sum_to_full():
    """Distributivity: sum_p W2[:, slice_p] h[slice_p] == W2 h (north_star (4))."""
    d, ff = 64, 256
    rng = np.random.default_rng(9)
    x = _rand_bf16(rng, (d,))
    full, _ = oracle.expert_ffn(*inputs.expert_weights(0, 3, d, ff), x)
    for P in (2, 4, 8):
        parts = [oracle.expert_ffn(*inputs.expert_weights(0, 3, d, ff, p, P), x)[0] for p in range(P)]
        tot = np.sum(np.stack(parts).astype(np.float64), axis=0)
        assert np.abs(tot - full).max() <= 1e-5 * np.abs(full).max()


@pytest.mark.parametrize("name,T", [("tiny", 32), ("mixtral-8x7b", 3), ("phi-3.5-moe", 3)])
def test_generated_hidden_states_realise_routing_with_margin(name, T):
    """The oracle's router recovers the generator's intended ranking with fp64 margin >= 0.1."""
    c = inputs.CONFIGS[name]
    L = min(c["L"], 2)
    tr = inputs.generate_trace(L, c["n"], c["K"], T, inputs.PRESETS["paper"](c["n"]))
    gates = [inputs.gate_weights(l, c["n"], c["d"]) for l in range(L)]
    x, ranked = inputs.make_hidden(tr, gates)
    for t in range(T):
        for l in range(L):
            z, z64 = oracle.gate_logits(gates[l], np.ascontiguousarray(x[t, l]))
            S, _ = oracle.topk_softmax(z, c["K"])
            assert list(S) == list(ranked[t, l])
            srt = np.sort(z64)[::-1]
            assert np.min(srt[:c["K"]] - srt[1:c["K"] + 1]) >= 0.1


def test_expert_ffn_independent_of_thread_count():
    """The oracle's row-parallel loops give bit-identical results at any thread count (each
    output row is one sequential sum): bench.py's cpu_baseline times it at 1 and all threads."""
    import inputs
    d, ff = 256, 512
    W1, W3, W2 = inputs.expert_weights(0, 3, d, ff)
    rng = np.random.default_rng(5)
    x = inputs.f32_to_bf16(rng.standard_normal(d).astype(np.float32))
    n0 = oracle.max_threads()
    try:
        oracle.set_threads(1)
        o1, h1 = oracle.expert_ffn(W1, W3, W2, x)
        oracle.set_threads(4)
        o4, h4 = oracle.expert_ffn(W1, W3, W2, x)
    finally:
        oracle.set_threads(n0)
    assert np.array_equal(o1.view(np.uint32), o4.view(np.uint32))
    assert np.array_equal(h1.view(np.uint32), h4.view(np.uint32))
