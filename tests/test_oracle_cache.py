"""Pins for the oracle's expert cache — CPU only."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import inputs
import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_worked_trace_golden():
    g = _gold("lru_worked_trace.json")
    s = g["setup"]
    c = oracle.Cache(s["layers"], s["covered"], s["M"], s["K"], oracle.LRU, s["warm_start"])
    for a in g["accesses"]:
        hit, way, ev, cov = c.access(0, np.array(a["S"]))
        assert list(hit) == a["hit"] and list(way) == a["way"] and list(ev) == a["evicted"]
        tags, stamps = c.set_state(0)
        assert [[int(t), int(st)] for t, st in zip(tags, stamps)] == a["ways_after"]
    st = c.stats(0)
    for k, v in g["stats"].items():
        assert st[k] == v, k


@pytest.mark.parametrize("case", _gold("spec_cache_examples.json")["cases"], ids=lambda c: c["name"])
def test_spec_examples(case):
    pol = oracle.LRU if case["policy"] == "LRU" else oracle.FIFO
    c = oracle.Cache(1, 1, case["M"], 1, pol)
    ev = None
    for e in case["sequence"]:
        _, _, ev, _ = c.access(0, np.array([e]))
    assert int(ev[0]) == case["final_evicted"]


def test_divergence_example_never_evicts_current_access():
    """Reading R10: set {b older, c}, access (a, b) -> a misses, b hits, c evicted."""
    a, b, cc = 0, 1, 2
    c = oracle.Cache(1, 1, 2, 1)
    c.access(0, np.array([b]))
    c.access(0, np.array([cc]))
    c2 = oracle.Cache(1, 1, 2, 2)
    c2.access(0, np.array([b, cc]))       # b -> way0 (older), c -> way1
    hit, way, ev, _ = c2.access(0, np.array([a, b]))
    assert list(hit) == [0, 1] and int(ev[0]) == cc


# ----------------------------------------------------------------------------- brute-force LRU
class BruteCache:
    """Independent reference: per-set recency LIST (most-recent last) + way map.

    Same semantics (R10, R11), different data structure: no stamps, no clock.
    """

    def __init__(self, M, policy):
        self.M, self.policy = M, policy
        self.ways = [None] * M    # way -> expert
        self.order = []           # experts, least recent first (FIFO: insertion order)

    def access(self, S):
        pre = set(e for e in self.ways if e is not None)
        hit = [e in pre for e in S]
        for e, h in zip(S, hit):
            if h and self.policy == oracle.LRU:
                self.order.remove(e)
                self.order.append(e)
        way, ev = [], []
        for e, h in zip(S, hit):
            if h:
                way.append(self.ways.index(e))
                ev.append(-1)
                continue
            if None in self.ways:
                v = self.ways.index(None)
                ev.append(-1)
            else:
                victim = next(x for x in self.order if x not in S)
                v = self.ways.index(victim)
                self.order.remove(victim)
                ev.append(victim)
            self.ways[v] = e
            self.order.append(e)
            way.append(v)
        return hit, way, ev


@pytest.mark.parametrize("policy", [oracle.LRU, oracle.FIFO])
@pytest.mark.parametrize("n,M,K", [(4, 2, 2), (8, 2, 1), (8, 4, 2), (8, 3, 3), (6, 4, 3), (8, 8, 2)])
def test_replay_equals_brute_force(policy, n, M, K):
    """SPEC S:252 / S:511: replay equivalence vs a brute-force reference cache (T <= 1000)."""
    rng = np.random.default_rng(n * 31 + M * 7 + K + policy)
    T = 1000
    c = oracle.Cache(1, 1, M, K, policy)
    b = BruteCache(M, policy)
    for t in range(T):
        S = rng.choice(n, size=K, replace=False) if rng.random() < 0.6 or t == 0 else S
        hit, way, ev, _ = c.access(0, S)
        bh, bw, be = b.access([int(e) for e in S])
        assert list(hit.astype(bool)) == bh, t
        assert list(way) == bw, t
        assert list(ev) == be, t


# ----------------------------------------------------------------------------- closed forms
@pytest.mark.parametrize("row", _gold("paper_closed_forms.json")["random_policy"],
                         ids=lambda r: f"n{r['n']}M{r['M']}")
def test_closed_form_values(row):
    n, M = row["n"], row["M"]
    p1 = 1 - Fraction(n - M, n) * Fraction(n - M - 1, n - 1)
    p2 = Fraction(M, n) * Fraction(M - 1, n - 1)
    assert p1 == Fraction(*row["at_least_one"]) and p2 == Fraction(*row["both"])


@pytest.mark.parametrize("policy", [oracle.LRU, oracle.FIFO])
@pytest.mark.parametrize("n,M", [(8, 2), (8, 4), (8, 6), (16, 4), (16, 8)])
def test_demand_fill_hit_rates_equal_paper_closed_forms_under_iid_routing(policy, n, M):
    """Under i.i.d. uniform top-2 routing the resident set is always M distinct experts
    independent of the next pair, so LRU/FIFO steady-state rates equal P:361-363's forms."""
    rng = np.random.default_rng(1000 + n + M)
    T = 60000
    c = oracle.Cache(1, 1, M, 2, policy)
    for t in range(T):
        c.access(0, rng.choice(n, size=2, replace=False))
    st = c.stats(0)
    p1 = 1 - (n - M) / n * (n - M - 1) / (n - 1)
    p2 = M / n * (M - 1) / (n - 1)
    assert abs(st["at_least_one_hit"] / T - p1) < 0.01
    assert abs(st["all_k_hit"] / T - p2) < 0.01


def test_lru_beats_random_static_on_reuse_heavy_trace():
    """S:254 / P:364 (directional): LRU >= random-policy closed form when tokens reuse experts."""
    n, M, K, T = 8, 4, 2, 20000
    tr = inputs.generate_trace(1, n, K, T, inputs.RoutingParams(0.45, 0.0))
    c = oracle.Cache(1, 1, M, K)
    for t in range(T):
        c.access(0, tr[t, 0])
    p1 = 1 - (n - M) / n * (n - M - 1) / (n - 1)
    assert c.stats(0)["at_least_one_hit"] / T >= p1


# ----------------------------------------------------------------------------- invariants
@pytest.mark.parametrize("L,N,M,warm", [(4, 4, 2, False), (4, 2, 2, False), (6, 3, 4, True),
                                        (3, 0, 2, False), (5, 9, 3, False)])
def test_counting_invariants(L, N, M, warm):
    n, K, T = 8, 2, 300
    tr = inputs.generate_trace(L, n, K, T, inputs.PRESETS["paper"](n))
    c = oracle.Cache(L, N, M, K, oracle.LRU, warm)
    Ncov = min(N, L)
    for t in range(T):
        for l in range(L):
            c.access(l, tr[t, l])
            if l < Ncov:
                tags, _ = c.set_state(l)
                valid = [int(x) for x in tags if x >= 0]
                assert len(valid) <= M and len(set(valid)) == len(valid)
    tot = c.stats(-1)
    assert tot["expert_hits"] + tot["expert_misses"] == T * L * K
    assert tot["coverage_misses"] == T * (L - Ncov) * K
    for l in range(L):
        s = c.stats(l)
        assert s["all_k_hit"] <= s["at_least_one_hit"] <= s["accesses"] == T
        covered_misses = s["expert_misses"] - s["coverage_misses"]
        if l < Ncov:
            tags, _ = c.set_state(l)
            occ = int((tags >= 0).sum())
            occ0 = M if warm else 0
            assert s["evictions"] == covered_misses - (occ - occ0)
        else:
            assert s["expert_hits"] == 0 and s["evictions"] == 0


def test_full_associativity_warm_start_all_hits():
    """M = n => all hits (warm start preloads experts 0..M-1)."""
    n, K = 8, 2
    c = oracle.Cache(2, 2, n, K, oracle.LRU, True)
    rng = np.random.default_rng(3)
    for _ in range(200):
        for l in range(2):
            hit, _, ev, _ = c.access(l, rng.choice(n, 2, replace=False))
            assert hit.all() and (ev == -1).all()


def test_cold_start_all_misses_first_access():
    c = oracle.Cache(3, 3, 2, 2)
    for l in range(3):
        hit, _, _, _ = c.access(l, np.array([5, 6]))
        assert not hit.any()


# ----------------------------------------------------------------------------- geometry
def test_geometry_paper_example():
    g = _gold("paper_closed_forms.json")["geometry_example"]
    slot = 352_321_536
    S, N_raw, N = oracle.cache_geometry(g["slots"] * slot + slot - 1, slot, g["ways"], 32)
    assert (S, N_raw, N) == (g["slots"], g["indexes"], g["indexes"])
    assert oracle.cache_geometry(0, slot, 4, 32) == (0, 0, 0)        # S = 0
    prev = -1
    for mem in range(0, 20 * slot, slot // 3):                         # monotone, N*M <= S
        S, N_raw, N = oracle.cache_geometry(mem, slot, 4, 32)
        assert S >= prev and N_raw * 4 <= S
        prev = S


# ----------------------------------------------------------------------------- generator stats
def test_generator_uniform_reuse_matches_closed_form():
    """uniform i.i.d. top-2 draws: P(reuse >= 1) = 1 - C(n-2,2)/C(n,2)."""
    import math
    for n in (8, 16):
        tr = inputs.generate_trace(1, n, 2, 40000, inputs.PRESETS["uniform"](n))
        st = inputs.pattern_stats(tr)
        cf = 1 - math.comb(n - 2, 2) / math.comb(n, 2)
        assert abs(st["token_reuse_at_least_one"] - cf) < 0.01


def test_generator_forced_repetition_and_paper_preset_band():
    tr = inputs.generate_trace(3, 8, 2, 50, inputs.RoutingParams(1.0, 0.0))
    assert all(set(tr[t, l]) == set(tr[0, l]) for t in range(50) for l in range(3))
    st = inputs.pattern_stats(inputs.generate_trace(8, 8, 2, 1500, inputs.PRESETS["paper"](8)))
    assert 0.40 <= st["token_reuse_at_least_one"] <= 0.70      # P:180 "between 40% and 60%" band
    assert 0.35 <= st["layer_match_at_least_one"] <= 0.55      # P:177 "approximately 44%"


# ----------------------------------------------------------------------------- random static policy
@pytest.mark.parametrize("n,M", [(8, 2), (8, 4), (8, 6), (16, 4), (16, 8)])
def test_static_random_policy_reaches_paper_closed_forms(n, M):
    """the random policy stores a random expert set statically; under uniform
    top-2 routing its hit rates ARE the closed forms (within 0.01 over 1e5)."""
    rng = np.random.default_rng(77 + n + M)
    T = 100_000
    c = oracle.Cache(1, 1, M, 2, oracle.STATIC, n=n, seed=1234 + M)
    tags0, _ = c.set_state(0)
    assert len(set(int(t) for t in tags0)) == M and all(0 <= t < n for t in tags0)
    for _ in range(T):
        c.access(0, rng.choice(n, size=2, replace=False))
    tags1, _ = c.set_state(0)
    assert np.array_equal(tags0, tags1)                 # never mutated
    st = c.stats(0)
    p1 = 1 - (n - M) / n * (n - M - 1) / (n - 1)
    p2 = M / n * (M - 1) / (n - 1)
    assert abs(st["at_least_one_hit"] / T - p1) < 0.01
    assert abs(st["all_k_hit"] / T - p2) < 0.01
    assert st["evictions"] == 0 and st["expert_hits"] + st["expert_misses"] == 2 * T


def test_static_draw_is_seeded_and_layer_dependent():
    a = oracle.Cache(4, 4, 3, 2, oracle.STATIC, n=8, seed=5)
    b = oracle.Cache(4, 4, 3, 2, oracle.STATIC, n=8, seed=5)
    c = oracle.Cache(4, 4, 3, 2, oracle.STATIC, n=8, seed=6)
    sets_a = [tuple(a.set_state(l)[0]) for l in range(4)]
    assert sets_a == [tuple(b.set_state(l)[0]) for l in range(4)]
    assert sets_a != [tuple(c.set_state(l)[0]) for l in range(4)]
    assert len(set(sets_a)) > 1


def test_lru_beats_static_random_on_paper_pattern_routing():
    """P:364 (directional): 'LRU improves the probability by around 5~15%' over random."""
    n, M, K, T = 8, 4, 2, 20000
    tr = inputs.generate_trace(1, n, K, T, inputs.PRESETS["paper"](n))
    lru = oracle.Cache(1, 1, M, K)
    st = oracle.Cache(1, 1, M, K, oracle.STATIC, n=n, seed=3)
    for t in range(T):
        lru.access(0, tr[t, 0])
        st.access(0, tr[t, 0])
    assert lru.stats(0)["at_least_one_hit"] > st.stats(0)["at_least_one_hit"]
