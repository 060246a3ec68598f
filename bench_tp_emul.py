#!/usr/bin/env python
"""f3 on one GPU: the ff-split TP group of BASELINE configs[4] (Mixtral-8x22B-shaped layer:
d = 6144, ff = 16384, 8 experts, top-2) emulated by P contexts on ONE B200, each holding
its ff/P slice of every expert, wired with moe_tp_connect_local: the P decode kernels of a
layer run co-resident (#SMs / P CTAs each) and sum y inside their epilogues through the
exchange buffers (the same kernel code that stores to the peers over NVLink on P GPUs).

What this measures: the cost of the fused reduction and of the grid split at a fixed total
HBM stream (P ranks share one GPU's HBM, so the whole layer's bytes stream once per step
whatever P is). What it does not: NVLink latency / bandwidth between GPUs (1-GPU boxes).

    python bench_tp_emul.py [--P 1,2,4,8] [--steps 2000] [--warmup 50]

One JSON line per P (P = 1: one context, full grid, no reduction, PDL as in bench.py).
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


def epilogue_breakdown(P: int, tokens: int = 16, steps: int = 40) -> dict:
    """Median per-CTA durations (us) of the fused reduction epilogue in the last call
    (MOE_DEBUG_TS marks 18, 21): wait for every rank's terms of the slice + fixed-order sum.
    The marks exist only in the debug build: run with MOE_LIB_PATH=.../lib/libmoe_debug.so."""
    import ctypes
    import statistics
    import torch
    import paper_2512_16473_b200 as moe
    os.environ["MOE_DEBUG_TS"] = "1"
    c = inputs.CONFIGS["mixtral-8x22b"]
    d, ff, n, K = c["d"], c["ff"], c["n"], c["K"]
    hps = [harness.host_model(1, d, ff, n, K, tp_size=P, tp_rank=p) for p in range(P)]
    x, _ = harness.hidden_states(hps[0], tokens, "paper")
    xd = torch.from_numpy(x.view(np.int16)).cuda()
    yd = torch.empty((P, tokens, d), dtype=torch.float32, device="cuda")
    ms = [harness.open_moe(hp) for hp in hps]
    os.environ.pop("MOE_DEBUG_TS", None)
    lib = moe.lib()
    lib.moe_debug_timestamps.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong]
    try:
        for m in ms:
            m.configure(ways=n, indexes=1, warm_start=True)
        moe.tp_connect_local(ms)
        streams = [torch.cuda.Stream() for _ in range(P)]
        for i in range(steps):
            for p in range(P):
                ms[p].forward(0, xd[i % tokens, 0].data_ptr(), yd[p, i % tokens].data_ptr(), streams[p].cuda_stream)
        torch.cuda.synchronize()
        marks = []
        for m in ms:
            G = m.runtime_info()["grid"]
            ts = np.zeros(G * 64, np.uint64)
            stride = lib.moe_debug_timestamps(m._h.value, ts.ctypes.data, ts.size)
            assert stride > 0, "per-CTA marks need the debug build (MOE_LIB_PATH=.../libmoe_debug.so)"
            marks.append(ts[:G * stride].reshape(G, stride).astype(np.int64))
    finally:
        for m in ms:
            m.close()
    t = np.concatenate(marks)
    if not (t[:, 18] > 0).any():   # the production build carries no marks
        return {"note": "epilogue marks need the debug build: MOE_LIB_PATH=paper_2512_16473_b200/lib/libmoe_debug.so"}
    med = lambda a: statistics.median(a.tolist()) / 1e3  # noqa: E731
    # the rank that arrives last waits only for its own slices to land everywhere: its wait is
    # the exchange latency; the other ranks' waits add the skew between the ranks' kernels
    per_rank = [med(mk[:, 21] - mk[:, 18]) for mk in marks]
    return {"epilogue_us_last_rank": min(per_rank), "epilogue_us_per_rank": per_rank,
            "epilogue_us_median": med(t[:, 21] - t[:, 18]),
            "note": "medians over CTAs, last call, from the CTA's last own term to all ranks' terms of its column "
                    "slice landed; the ranks share one GPU (no NVLink hop), so waits beyond the last rank's are "
                    "skew between the co-resident rank kernels, not exchange cost"}


def run(P: int, steps: int, warmup: int, tokens: int, pdl1: bool) -> dict:
    import torch
    import paper_2512_16473_b200 as moe
    c = inputs.CONFIGS["mixtral-8x22b"]
    d, ff, n, K = c["d"], c["ff"], c["n"], c["K"]
    hps = [harness.host_model(1, d, ff, n, K, tp_size=P, tp_rank=p) for p in range(P)]
    x, _ = harness.hidden_states(hps[0], tokens, "paper")
    xd = torch.from_numpy(x.view(np.int16)).cuda()
    yd = torch.empty((P, tokens, d), dtype=torch.float32, device="cuda")
    env_pdl = os.environ.get("MOE_PDL")
    if P == 1 and not pdl1:
        os.environ["MOE_PDL"] = "0"
    ms = [harness.open_moe(hp) for hp in hps]
    if env_pdl is None:
        os.environ.pop("MOE_PDL", None)
    else:
        os.environ["MOE_PDL"] = env_pdl
    try:
        for m in ms:
            m.configure(ways=n, indexes=1, warm_start=True)
        if P > 1:
            moe.tp_connect_local(ms)
        info = ms[0].runtime_info()
        streams = [torch.cuda.Stream() for _ in range(P)]

        def steps_on(first: int, count: int):
            for i in range(first, first + count):
                t = i % tokens
                for p in range(P):
                    ms[p].forward(0, xd[t, 0].data_ptr(), yd[p, t].data_ptr(), streams[p].cuda_stream)

        steps_on(0, warmup)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(streams[0])
        for s in streams[1:]:
            s.wait_event(ev0)
        steps_on(warmup, steps)
        for s in streams[1:]:
            e = torch.cuda.Event()
            e.record(s)
            streams[0].wait_event(e)
        ev1.record(streams[0])
        ev1.synchronize()
        ms_step = ev0.elapsed_time(ev1) / steps
        y = yd.cpu().numpy()
        same = all(np.array_equal(y[p].view(np.uint32), y[0].view(np.uint32)) for p in range(P))
        tr = [m.trace() for m in ms]
        same_tr = all(np.array_equal(tr[p]["expert"], tr[0]["expert"]) for p in range(P))
    finally:
        for m in ms:
            m.close()
    layer_bytes = K * 3 * d * ff * 2 + P * (n * d * 2 + d * 2)
    return {"P": P, "workload": "configs[4] Mixtral-8x22B-shaped layer (d=6144, ff=16384, 8 experts top-2), "
                                "decode batch 1, M=8 warm, ff-split over P contexts on ONE GPU",
            "us_per_layer_step": ms_step * 1e3, "layer_steps_per_s": 1e3 / ms_step,
            "stream_gbs": layer_bytes / (ms_step * 1e-3) / 1e9, "bytes_per_step": layer_bytes,
            "runtime": info, "ranks_bit_identical_y": bool(same), "ranks_identical_routing": bool(same_tr),
            "steps": steps, "warmup": warmup}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--P", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--tokens", type=int, default=64)
    args = ap.parse_args()
    for P in [int(v) for v in args.P.split(",")]:
        if P == 1:
            for pdl in (True, False):
                r = run(1, args.steps, args.warmup, args.tokens, pdl)
                print(json.dumps(r), flush=True)
        else:
            r = run(P, args.steps, args.warmup, args.tokens, False)
            r["fused_reduction_epilogue"] = epilogue_breakdown(P)
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
