#!/usr/bin/env python
"""Fig.6-style hit-rate table from bench_sweep.py JSON lines: per (model, M,
policy) the paper's "expert(s) hit" (>= 1 of the K routed experts resident) and "2 experts
hit" (all K), measured by the GPU's cache counters (timed tokens), the oracle's replay of the
same routing beside them (must be equal), the closed forms of the random static policy
 and the LRU - random gap (the paper reports +5-15 % for Mixtral).

    python tools/fig6_table.py profiles/r02_fig6_*.jsonl
"""
from __future__ import annotations

import json
import sys


def closed_forms(n: int, M: int):
    """P(>=1 hit) = 1 - (n-M)/n * (n-M-1)/(n-1); P(2 hit) = M/n * (M-1)/(n-1)."""
    return 1.0 - (n - M) / n * (n - M - 1) / (n - 1), M / n * (M - 1) / (n - 1)


def main(paths):
    rows = []
    for p in paths:
        for line in open(p):
            line = line.strip()
            if line.startswith("{"):
                rows.append(json.loads(line))
    N_EXP = {"mixtral-8x7b": 8, "phi-3.5-moe": 16, "tiny": 8}
    by = {}
    for r in rows:
        by[(r["config"], r["ways"], r["policy"])] = r
    print(f"{'model':14s} {'M':>2s} {'policy':7s} {'>=1 hit':>8s} {'2 hit':>7s} {'per-exp':>7s} "
          f"{'closed >=1':>10s} {'closed 2':>8s} {'GPU==oracle':>11s} {'LRU-rand >=1':>12s} {'LRU-rand 2':>10s}")
    for (cfg, M, pol) in sorted(by):
        r = by[(cfg, M, pol)]
        n = N_EXP[cfg]
        h = r["hit_rate"]
        o = r.get("oracle_hit_rate", h)
        c1, c2 = closed_forms(n, M)
        eq = r["trace_bit_exact_vs_oracle"] and r["stats_equal_oracle"] and all(
            abs(h[k] - o[k]) < 1e-12 for k in h)
        gap = ""
        if pol == "lru" and (cfg, M, "static") in by:
            s = by[(cfg, M, "static")]["hit_rate"]
            gap = f"{h['expert(s)_hit'] - s['expert(s)_hit']:+12.3f} {h['all_k_hit'] - s['all_k_hit']:+10.3f}"
        print(f"{cfg:14s} {M:2d} {pol:7s} {h['expert(s)_hit']:8.3f} {h['all_k_hit']:7.3f} {h['per_expert']:7.3f} "
              f"{c1 if pol == 'static' else float('nan'):10.3f} {c2 if pol == 'static' else float('nan'):8.3f} "
              f"{str(eq):>11s} {gap}")


if __name__ == "__main__":
    main(sys.argv[1:])
