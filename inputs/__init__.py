"""Seeded synthetic input generators shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no gate GEMV, no top-k, no
cache, no FFN). It produces:

* expert weights (bf16 bit patterns) from a counter-based hash (``gen.c``),
  regenerable per row / column slice;
* gate weights: seeded Gaussian rows orthonormalised in fp64 (QR), rounded to bf16;
* routing traces with the paper's expert-reuse patterns (SPEC ``generate_trace``
  semantics, SPEC.md:146-154 / S:172-173; patterns from PAPER.md:177-181);
* hidden states x[t][l] whose router logits realise a chosen routing with a
  margin (target logits z*, then x = Wg^T (Wg Wg^T)^-1 z* + null-space noise).

The recipe is stated in DESIGN.md ("Input recipe").
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB = os.path.join(_HERE, "libinputs.so")
_lib = None

KIND_GATE, KIND_W1, KIND_W3, KIND_W2 = 0, 1, 2, 3
SEED_WEIGHTS, SEED_ROUTING, SEED_NOISE = 1, 2, 3


def build(force: bool = False) -> str:
    """Compile gen.c into libinputs.so (gcc, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-ffp-contract=off",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        u64, i32, i64, f32, p = (ctypes.c_uint64, ctypes.c_int, ctypes.c_int64, ctypes.c_float,
                                 ctypes.c_void_p)
        lib.gen_rows.argtypes = [u64, i32, i32, i32, i64, f32, i64, i64, p]
        lib.gen_cols.argtypes = [u64, i32, i32, i32, i64, i64, f32, i64, i64, p]
        lib.f32_to_bf16_array.argtypes = [p, p, i64]
        _lib = lib
    return _lib


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


# ----------------------------------------------------------------------------- bf16 helpers
def bf16_to_f32(a: np.ndarray) -> np.ndarray:
    return (a.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    out = np.empty(a.shape, dtype=np.uint16)
    _load().f32_to_bf16_array(_ptr(a), _ptr(out), a.size)
    return out


# ----------------------------------------------------------------------------- expert weights
def expert_weights_into(w1: np.ndarray, w3: np.ndarray, w2: np.ndarray, layer: int, expert: int,
                        d: int, ff: int, tp_rank: int = 0, tp_size: int = 1,
                        seed: int = SEED_WEIGHTS) -> None:
    """Fill caller buffers with this rank's ff-slice of expert (layer, expert).

    w1, w3: [ff/P][d] rows [p*ff/P, (p+1)*ff/P) of W1 / W3 (nn.Linear layout, row j = d contiguous)
    w2    : [d][ff/P] columns of W2 ([d][ff] nn.Linear layout), repacked contiguous.
    Buffers may be views into a pinned host blob (any C-contiguous uint16 memory).
    """
    ffr = ff // tp_size
    r0, r1 = tp_rank * ffr, (tp_rank + 1) * ffr
    assert w1.shape == (ffr, d) and w3.shape == (ffr, d) and w2.shape == (d, ffr)
    lib = _load()
    lib.gen_rows(seed, KIND_W1, layer, expert, d, float(d), r0, r1, _ptr(w1))
    lib.gen_rows(seed, KIND_W3, layer, expert, d, float(d), r0, r1, _ptr(w3))
    lib.gen_cols(seed, KIND_W2, layer, expert, d, ff, float(ff), r0, r1, _ptr(w2))


def expert_weights(layer: int, expert: int, d: int, ff: int, tp_rank: int = 0, tp_size: int = 1,
                   seed: int = SEED_WEIGHTS):
    ffr = ff // tp_size
    w1 = np.empty((ffr, d), np.uint16)
    w3 = np.empty((ffr, d), np.uint16)
    w2 = np.empty((d, ffr), np.uint16)
    expert_weights_into(w1, w3, w2, layer, expert, d, ff, tp_rank, tp_size, seed)
    return w1, w3, w2


# ----------------------------------------------------------------------------- gate weights
def gate_weights(layer: int, n: int, d: int, seed: int = SEED_WEIGHTS) -> np.ndarray:
    """Wg [n][d] bf16: seeded Gaussian, rows orthonormalised in fp64 (QR), rounded to bf16."""
    rng = np.random.default_rng([seed, KIND_GATE, layer])
    g = rng.standard_normal((d, n))
    q, _ = np.linalg.qr(g)  # d x n, orthonormal columns
    return f32_to_bf16(q.T.astype(np.float32))


# ----------------------------------------------------------------------------- routing traces
@dataclass(frozen=True)
class RoutingParams:
    p_token_reuse: float
    p_layer_follow: float


PRESETS = {
    # (n) -> params; "uniform" drives the closed-form pins, "paper" the reuse patterns.
    "uniform": lambda n: RoutingParams(0.0, 0.0),
    "paper": lambda n: RoutingParams(0.15 if n <= 8 else 0.20, 0.0),
}


def generate_trace(L: int, n: int, K: int, T: int, params: RoutingParams,
                   seed: int = SEED_ROUTING) -> np.ndarray:
    """Expert sets e[t][l][0..K-1] (draw order), SPEC generate_trace semantics.

    Per (t, l, slot): with p_token_reuse copy a not-yet-chosen expert of layer l at t-1
    (token rule first); else with p_layer_follow copy a not-yet-chosen expert of
    layer l-1 at t; else draw uniformly among experts not yet chosen.
    """
    assert 1 <= K <= n
    rng = np.random.default_rng(seed)
    out = np.empty((T, L, K), np.int32)
    for t in range(T):
        for l in range(L):
            chosen: list[int] = []
            for _ in range(K):
                if t > 0 and params.p_token_reuse > 0 and rng.random() < params.p_token_reuse:
                    cand = [e for e in out[t - 1, l] if e not in chosen]
                    if cand:
                        chosen.append(int(cand[rng.integers(len(cand))]))
                        continue
                if l > 0 and params.p_layer_follow > 0 and rng.random() < params.p_layer_follow:
                    cand = [e for e in out[t, l - 1] if e not in chosen]
                    if cand:
                        chosen.append(int(cand[rng.integers(len(cand))]))
                        continue
                rem = [e for e in range(n) if e not in chosen]
                chosen.append(rem[int(rng.integers(len(rem)))])
            out[t, l] = chosen
    return out


def pattern_stats(trace: np.ndarray) -> dict:
    """Consecutive-token / consecutive-layer reuse rates of a trace."""
    T, L, K = trace.shape
    tok = [len(set(trace[t, l]) & set(trace[t - 1, l])) for t in range(1, T) for l in range(L)]
    lay = [len(set(trace[t, l]) & set(trace[t, l - 1])) > 0 for t in range(T) for l in range(1, L)]
    tok = np.array(tok)
    return {
        "token_reuse_at_least_one": float((tok > 0).mean()) if tok.size else float("nan"),
        "token_reuse_per_expert": float(tok.mean() / K) if tok.size else float("nan"),
        "layer_match_at_least_one": float(np.mean(lay)) if lay else float("nan"),
    }


# ----------------------------------------------------------------------------- hidden states
def target_logits(trace: np.ndarray, n: int, seed: int = SEED_NOISE):
    """z*[t][l][n] realising each set with a rank order and margins; returns (z*, ranked sets).

    Chosen experts get distinct values on a 0.3-spaced grid inside [0.5, 2.5] (random
    assignment = the rank order); the others uniform in [-2, 0]. Margins >= 0.3 / 0.5.
    """
    T, L, K = trace.shape
    rng = np.random.default_rng([seed, 7])
    z = rng.uniform(-2.0, 0.0, size=(T, L, n))
    step = 0.3 if K <= 7 else 2.0 / (K - 1)
    grid = 0.5 + step * np.arange(max(K, 7 if K <= 7 else K))
    grid = grid[grid <= 2.5 + 1e-12]
    ranked = np.empty_like(trace)
    for t in range(T):
        for l in range(L):
            vals = np.sort(rng.choice(grid, size=K, replace=False))[::-1]
            order = rng.permutation(trace[t, l])
            z[t, l, order] = vals
            ranked[t, l] = order
    return z, ranked


def make_hidden(trace: np.ndarray, gates: list[np.ndarray], seed: int = SEED_NOISE):
    """x[t][l][d] (bf16) with Wg_l x ~= z*[t][l] and ranked sets (intended top-K order)."""
    T, L, K = trace.shape
    n, d = gates[0].shape
    z, ranked = target_logits(trace, n, seed)
    rng = np.random.default_rng([seed, 11])
    x = np.empty((T, L, d), np.uint16)
    for l in range(L):
        G = bf16_to_f32(gates[l]).astype(np.float64)          # n x d
        B = np.linalg.inv(G @ G.T)                            # n x n
        noise = rng.standard_normal((T, d))
        noise -= (noise @ G.T) @ B @ G                        # project onto null(G)
        xl = z[:, l, :] @ B @ G + noise                       # G x = z*
        x[:, l, :] = f32_to_bf16(xl.astype(np.float32))
    return x, ranked


@dataclass
class Workload:
    """A seeded synthetic decode workload (shapes of BASELINE.json configs)."""
    name: str
    L: int
    d: int
    ff: int
    n: int
    K: int
    T: int
    preset: str = "paper"

    def trace(self) -> np.ndarray:
        return generate_trace(self.L, self.n, self.K, self.T, PRESETS[self.preset](self.n))

    def gates(self) -> list[np.ndarray]:
        return [gate_weights(l, self.n, self.d) for l in range(self.L)]


CONFIGS = {
    "tiny": dict(L=4, d=64, ff=128, n=8, K=2),
    "mixtral-8x7b": dict(L=32, d=4096, ff=14336, n=8, K=2),
    "phi-3.5-moe": dict(L=32, d=4096, ff=6400, n=16, K=2),
    "mixtral-8x22b": dict(L=56, d=6144, ff=16384, n=8, K=2),
}

