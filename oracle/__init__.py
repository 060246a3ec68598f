"""THE ORACLE — test infrastructure only.

Plain CPU implementation (``oracle.c``) of the per-layer MoE block of arXiv
2512.16473 at single-request decode, plus the decode loop that composes it.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package. It shares no code with the
CUDA path (``paper_2512_16473_b200``) and never imports it.

Every function cites the passage it follows (P:<line> = PAPER.md, S:<line> =
SPEC.md, R<k> = the reading listed in DESIGN.md). The pins that tie it to the
paper and to mathematics live in ``tests/test_oracle_*.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

LRU, FIFO, STATIC = 0, 1, 2
STAT_FIELDS = ("accesses", "at_least_one_hit", "all_k_hit", "expert_hits", "expert_misses",
               "coverage_misses", "evictions")


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-ffp-contract=off",
                               "-fno-fast-math", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        p, i32 = ctypes.c_void_p, ctypes.c_int
        lib.oracle_gate_logits.argtypes = [p, p, i32, i32, p, p]
        lib.oracle_topk_softmax.argtypes = [p, i32, i32, p, p]
        lib.oracle_expert_ffn.argtypes = [p, p, p, p, i32, i32, p, p]
        lib.oracle_combine.argtypes = [p, p, i32, i32, p]
        lib.oracle_cache_new.argtypes = [i32, i32, i32, i32, i32, i32]
        lib.oracle_cache_new.restype = p
        lib.oracle_cache_new_seeded.argtypes = [i32, i32, i32, i32, i32, i32, i32, ctypes.c_uint64]
        lib.oracle_cache_new_seeded.restype = p
        lib.oracle_cache_free.argtypes = [p]
        lib.oracle_cache_access.argtypes = [p, i32, p, p, p, p, p]
        lib.oracle_cache_stats.argtypes = [p, i32, p]
        lib.oracle_cache_set.argtypes = [p, i32, p, p]
        lib.oracle_set_threads.argtypes = [i32]
        lib.oracle_max_threads.restype = i32
        _lib = lib
    return _lib


def set_threads(n: int) -> None:
    """OpenMP threads of the row-parallel loops (results do not depend on it)."""
    _load().oracle_set_threads(int(n))


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def _p(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"], "oracle inputs must be C-contiguous"
    return a.ctypes.data


# ----------------------------------------------------------------------------- router
def gate_logits(Wg: np.ndarray, x: np.ndarray):
    """z = Wg x in fp32 (sequential) and fp64 (R1). Wg [n][d], x [d] bf16 bits."""
    n, d = Wg.shape
    z = np.empty(n, np.float32)
    z64 = np.empty(n, np.float64)
    _load().oracle_gate_logits(_p(Wg), _p(x), n, d, _p(z), _p(z64))
    return z, z64


def topk_softmax(z: np.ndarray, K: int):
    """Top-K by (z desc, index asc), softmax over the K in rank order (R1, R2)."""
    z = np.ascontiguousarray(z, np.float32)
    S = np.empty(K, np.int32)
    w = np.empty(K, np.float32)
    _load().oracle_topk_softmax(_p(z), z.size, K, _p(S), _p(w))
    return S, w


# ----------------------------------------------------------------------------- expert FFN
def expert_ffn(W1: np.ndarray, W3: np.ndarray, W2: np.ndarray, x: np.ndarray):
    """o = W2 (silu(W1 x) * (W3 x)) in fp32 (R4). Returns (o [d], h [ff])."""
    ff, d = W1.shape
    assert W3.shape == (ff, d) and W2.shape == (d, ff) and x.shape == (d,)
    h = np.empty(ff, np.float32)
    o = np.empty(d, np.float32)
    _load().oracle_expert_ffn(_p(W1), _p(W3), _p(W2), _p(x), d, ff, _p(h), _p(o))
    return o, h


def combine(o: np.ndarray, w: np.ndarray):
    """y = sum_r w[r] o_r in rank order (Fig.1)."""
    o = np.ascontiguousarray(o, np.float32)
    K, d = o.shape
    w = np.ascontiguousarray(w, np.float32)
    y = np.empty(d, np.float32)
    _load().oracle_combine(_p(o), _p(w), K, d, _p(y))
    return y


# ----------------------------------------------------------------------------- expert cache
class Cache:
    """N-index x M-way set-associative expert cache over layers 0..N-1."""

    def __init__(self, L: int, N: int, M: int, K: int, policy: int = LRU, warm_start: bool = False,
                 n: int = 0, seed: int = 0):
        self.L, self.N, self.M, self.K = L, min(N, L), M, K
        if policy == STATIC and n < M:
            raise ValueError("STATIC policy needs n >= M")
        self._h = _load().oracle_cache_new_seeded(L, N, M, K, policy, int(warm_start), n, seed)

    def __del__(self):
        if getattr(self, "_h", None):
            _load().oracle_cache_free(self._h)
            self._h = None

    def access(self, layer: int, S: np.ndarray):
        S = np.ascontiguousarray(S, np.int32)
        K = self.K
        hit = np.empty(K, np.int8)
        way = np.empty(K, np.int8)
        ev = np.empty(K, np.int16)
        cov = np.empty(K, np.int8)
        _load().oracle_cache_access(self._h, layer, _p(S), _p(hit), _p(way), _p(ev), _p(cov))
        return hit, way, ev, cov

    def stats(self, layer: int = -1) -> dict:
        out = np.empty(7, np.uint64)
        _load().oracle_cache_stats(self._h, layer, _p(out))
        return dict(zip(STAT_FIELDS, (int(v) for v in out)))

    def set_state(self, layer: int):
        tags = np.empty(self.M, np.int32)
        stamps = np.empty(self.M, np.uint64)
        _load().oracle_cache_set(self._h, layer, _p(tags), _p(stamps))
        return tags, stamps


def cache_geometry(cache_bytes: int, slot_bytes: int, M: int, L: int):
    """S = floor(avail / per-expert), N = floor(S / M); coverage min(N, L) (R7)."""
    S = cache_bytes // slot_bytes
    N_raw = S // M
    return S, N_raw, min(N_raw, L)


# ----------------------------------------------------------------------------- decode loop
@dataclass
class DecodeResult:
    y: np.ndarray                 # [T][L][d] fp32
    records: np.ndarray           # structured [T*L*K]: token, layer, rank, hit, expert, way, evicted, cov, weight
    logits64: np.ndarray          # [T][L][n] fp64 router logits (margin checks)
    stats: list = field(default_factory=list)  # per layer dicts
    total: dict = field(default_factory=dict)


RECORD_DTYPE = np.dtype([("token", np.uint32), ("layer", np.uint16), ("rank", np.uint8),
                         ("hit", np.uint8), ("expert", np.int16), ("evicted", np.int16),
                         ("way", np.int8), ("coverage", np.uint8), ("weight", np.float32)])


def decode(x: np.ndarray, gates, experts, N: int, M: int, K: int, policy: int = LRU,
           warm_start: bool = False, tokens=None, compute: bool = True, seed: int = 0) -> DecodeResult:
    """Token-major, layer-ascending decode of decoupled hidden states x[t][l] (R17).

    gates[l]  : Wg [n][d] bf16 bits.   experts(l, e) -> (W1, W3, W2) bf16 bits.
    For each (t, l): router -> cache check / LRU update ->
    expert FFNs of the K routed experts (the cache changes where weights are read,
    never the math, so the result is the plain MoE layer) -> gate-weighted combine.
    `tokens` restricts the FFN evaluation to a subset (routing/cache still run for all).
    """
    T, L, d = x.shape
    n = gates[0].shape[0]
    cache = Cache(L, N, M, K, policy, warm_start, n=n, seed=seed)
    y = np.zeros((T, L, d), np.float32)
    recs = np.zeros(T * L * K, RECORD_DTYPE)
    z64s = np.zeros((T, L, n), np.float64)
    want = set(range(T)) if tokens is None else set(tokens)
    i = 0
    for t in range(T):
        for l in range(L):
            xl = np.ascontiguousarray(x[t, l])
            z, z64 = gate_logits(gates[l], xl)
            z64s[t, l] = z64
            S, w = topk_softmax(z, K)
            hit, way, ev, cov = cache.access(l, S)
            for r in range(K):
                recs[i] = (t, l, r, hit[r], S[r], ev[r], way[r], cov[r], w[r])
                i += 1
            if compute and t in want:
                o = np.stack([expert_ffn(*experts(l, int(S[r])), xl)[0] for r in range(K)])
                y[t, l] = combine(o, w)
    return DecodeResult(y=y, records=recs, logits64=z64s,
                        stats=[cache.stats(l) for l in range(L)], total=cache.stats(-1))
