#!/usr/bin/env python
"""Prefill (f4) benchmark: one MoE layer of a BASELINE shape (default Mixtral-8x7B) over a
prompt of T tokens, expert FFN as two tcgen05 tensor-core GEMMs per distinct routed expert.

    python bench_prefill.py [--shape mixtral-8x7b|phi-3.5-moe|mixtral-8x22b] [--tokens 128,512,2048,4096] [--reps 20]

Prints one JSON line per T: tokens/s, the two GEMMs' TFLOP/s against the measured bf16
dense peak (MEASURED_PEAKS.json), the weight-byte roofline (each expert's weights are read
once per 128-token tile row of the GEMM grid; L2 absorbs the re-reads), and the max relative
error of sampled tokens against the oracle.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="mixtral-8x7b", choices=["mixtral-8x7b", "phi-3.5-moe", "mixtral-8x22b"])
    ap.add_argument("--tokens", default="128,512,2048,4096")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--check", type=int, default=4, help="tokens checked against the oracle per T")
    ap.add_argument("--ways", type=int, default=0, help="cache ways M (default n: nothing evicted; M < n: "
                    "evictions inside the prompt, the cache pass replays the accesses in order)")
    args = ap.parse_args()
    import torch

    import harness
    import oracle

    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        peaks = json.load(f)
    c = inputs.CONFIGS[args.shape]
    d, ff, n, K = c["d"], c["ff"], c["n"], c["K"]
    hm = harness.host_model(1, d, ff, n, K)
    M = args.ways or n
    dev = torch.device("cuda", 0)
    W = {}
    for T in [int(v) for v in args.tokens.split(",")]:
        x, _ = harness.hidden_states(hm, T, "paper")
        xd = torch.from_numpy(np.ascontiguousarray(x[:, 0, :]).view(np.int16)).to(dev)
        yd = torch.empty((T, d), dtype=torch.float32, device=dev)
        with harness.open_moe(hm) as m:
            m.configure(ways=M, indexes=1, warm_start=True)
            s = torch.cuda.Stream(dev)
            for _ in range(3):
                m.prefill(0, xd.data_ptr(), yd.data_ptr(), T, s.cuda_stream)
            s.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(args.reps):
                m.prefill(0, xd.data_ptr(), yd.data_ptr(), T, s.cuda_stream)
            e1.record(s)
            e1.synchronize()
            ms = e0.elapsed_time(e1) / args.reps
            m.profile(True)
            m.profile_read()
            for _ in range(args.reps):
                m.prefill(0, xd.data_ptr(), yd.data_ptr(), T, s.cuda_stream)
            s.synchronize()
            prof = m.profile_read()
            tr = m.trace()
        ybuf = yd.cpu().numpy()
        distinct = len(set(int(e) for e in tr["expert"][: T * K]))
        flops_g1 = 2.0 * T * K * 2 * d * ff
        flops_g2 = 2.0 * T * K * d * ff
        g1 = prof["expert_ffn"]["ms"] / max(prof["expert_ffn"]["launches"], 1)
        g2 = prof["expert_down"]["ms"] / max(prof["expert_down"]["launches"], 1)
        rt = prof["route_probe"]["ms"] / max(prof["route_probe"]["launches"], 1)
        # oracle on a few tokens (y does not depend on the cache state)
        chk = np.linspace(0, T - 1, num=min(args.check, T)).astype(int)

        def experts(l, e):
            if (l, e) not in W:
                W[(l, e)] = inputs.expert_weights(l, e, d, ff)
            return W[(l, e)]
        errs = []
        for t in chk:
            r = oracle.decode(x[t:t + 1], hm.gates, experts, N=1, M=n, K=K, warm_start=True)
            errs.append(float(np.abs(ybuf[t] - r.y[0, 0]).max() / np.abs(r.y[0, 0]).max()))
        peak = float(peaks["bf16_tflops"])
        line = {"workload": f"prefill: one {args.shape}-shaped MoE layer (d={d}, ff={ff}, {n} experts top-{K}), M={M} warm",
                "T": T, "ms": ms, "tokens_per_s": T / (ms * 1e-3), "distinct_experts": distinct,
                "tflops_total": (flops_g1 + flops_g2) / (ms * 1e-3) / 1e12,
                "gemm_swiglu": {"ms": g1, "tflops": flops_g1 / (g1 * 1e-3) / 1e12,
                                "frac_of_measured_bf16": flops_g1 / (g1 * 1e-3) / 1e12 / peak},
                "gemm_down": {"ms": g2, "tflops": flops_g2 / (g2 * 1e-3) / 1e12,
                              "frac_of_measured_bf16": flops_g2 / (g2 * 1e-3) / 1e12 / peak},
                "router_cache_ms": rt,
                "weight_bytes": distinct * 3 * d * ff * 2,
                "weight_gbs": distinct * 3 * d * ff * 2 / (ms * 1e-3) / 1e9,
                "peak_bf16_tflops_measured": peak, "hbm_gbs_measured": peaks["hbm_gbs"],
                "max_rel_err_vs_oracle": max(errs), "checked_tokens": [int(t) for t in chk]}
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
