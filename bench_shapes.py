#!/usr/bin/env python
"""Decode-step roofline across the BASELINE shapes on one B200 (fused one-kernel step,
warm cache: every routed expert resident, so the step is the HBM stream plus the fixed
routing prologue):

  mixtral-8x7b   configs[1]/[2] layer   d 4096, ff 14336, n 8   704.7 MB / step
  phi-3.5-moe    configs[3] layer       d 4096, ff  6400, n 16  314.7 MB / step
  8x22b/P        configs[4] per-rank    d 6144, ff 16384/P, n 8 (P = 1, 2, 4, 8): the work one
                 rank of the ff-split does per layer (its slice as a tp_size 1 model; the
                 fused peer reduction adds its exchange on top, see bench_tp_emul.py)

    python bench_shapes.py [--shapes ...] [--steps 3000] [--warmup 100]

One JSON line per shape: us per step (CUDA events over K back-to-back steps on the launch
stream), algorithmic bytes, GB/s and the fraction of the measured copy peak. The smaller
the step, the larger the share of the fixed prologue (PDL wait -> x -> gate GEMV ->
routing -> first weight bytes, ~5 us) in it.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import harness  # noqa: E402
import inputs  # noqa: E402

SHAPES = {
    "tiny": (64, 128, 8, 2),            # configs[0] expert shape: the step's fixed-cost floor
    "mixtral-8x7b": (4096, 14336, 8, 2),
    "phi-3.5-moe": (4096, 6400, 16, 2),
    "8x22b-P1": (6144, 16384, 8, 2),
    "8x22b-P2": (6144, 8192, 8, 2),
    "8x22b-P4": (6144, 4096, 8, 2),
    "8x22b-P8": (6144, 2048, 8, 2),
    "mixtral-8x7b-P8": (4096, 1792, 8, 2),   # configs[1]'s layer split 8 ways: one rank's work
}


def _peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"])
    return 6650.0


def run(name: str, steps: int, warmup: int, tokens: int) -> dict:
    import torch
    d, ff, n, K = SHAPES[name]
    hm = harness.host_model(1, d, ff, n, K)
    x, _ = harness.hidden_states(hm, tokens, "uniform")
    xd = torch.from_numpy(x.view(np.int16)).cuda()
    yd = torch.empty((tokens, d), dtype=torch.float32, device="cuda")
    with harness.open_moe(hm) as m:
        m.configure(ways=n, indexes=1, warm_start=True)
        s = torch.cuda.Stream()
        for i in range(warmup):
            m.forward(0, xd[i % tokens, 0].data_ptr(), yd[i % tokens].data_ptr(), s.cuda_stream)
        s.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(s)
        for i in range(steps):
            t = (warmup + i) % tokens
            m.forward(0, xd[t, 0].data_ptr(), yd[t].data_ptr(), s.cuda_stream)
        ev1.record(s)
        ev1.synchronize()
        info = m.runtime_info()
    us = ev0.elapsed_time(ev1) / steps * 1e3
    nbytes = K * 3 * d * ff * 2 + n * d * 2 + d * 2
    gbs = nbytes / (us * 1e-6) / 1e9
    return {"shape": name, "d": d, "ff_r": ff, "n": n, "K": K, "us_per_step": us, "bytes_per_step": nbytes,
            "gbs": gbs, "frac_of_measured_copy_peak": gbs / _peak(), "stream_floor_us_at_peak": nbytes / _peak() / 1e3,
            "runtime": info, "steps": steps, "routing": "uniform preset (rotating expert pairs)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default=",".join(SHAPES))
    ap.add_argument("--steps", type=int, default=3000)
    ap.add_argument("--warmup", type=int, default=100)
    ap.add_argument("--tokens", type=int, default=64)
    args = ap.parse_args()
    for name in args.shapes.split(","):
        print(json.dumps(run(name, args.steps, args.warmup, args.tokens)), flush=True)


if __name__ == "__main__":
    main()
