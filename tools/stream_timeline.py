#!/usr/bin/env python
"""Overlap of the miss traffic with compute, read from the library's own stream timeline
(MOE_STREAM_TIMELINE=1: CUDA events around every kernel on the caller's stream, every weight
copy on the fetch stream and every host-result copy on the activation stream — the two
streams of P:226). No system profiler is needed (nsys is not in this image).

Runs a miss-heavy cold decode (default: Mixtral-8x7B shape, 32 layers, M=4 ways, 8 tokens)
in the FETCH and HOST_COMPUTE miss modes and prints, per mode, one JSON line:
  fetch copies: count, bytes, link GB/s over the union of copy intervals (PCIe Gen5 x16:
    ~64 GB/s nominal), busy fraction of the decode;
  overlap: share of the fetch-stream busy time during which a kernel of ANOTHER call ran
    (FETCH: a call waits for its own fill, so its copy overlaps only earlier/later calls;
    HOST_COMPUTE: the post-fetch of call s runs under the following calls' kernels);
  activation copies (HOST_COMPUTE): count, mean latency.

    python tools/stream_timeline.py [--config mixtral-8x7b] [--layers 32] [--ways 4] [--tokens 8]
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("MOE_STREAM_TIMELINE", "1")

import numpy as np  # noqa: E402

import harness  # noqa: E402
import inputs  # noqa: E402
import paper_2512_16473_b200 as moe  # noqa: E402


def union_len(iv):
    """Total length of the union of intervals [(a, b)]."""
    tot, end = 0.0, -1e300
    for a, b in sorted(iv):
        if b <= end:
            continue
        tot += b - max(a, end)
        end = b
    return tot


def overlap_len(a_iv, b_iv):
    """Length of (union of a_iv) intersected with (union of b_iv)."""
    def merged(iv):
        out = []
        for a, b in sorted(iv):
            if out and a <= out[-1][1]:
                out[-1][1] = max(out[-1][1], b)
            else:
                out.append([a, b])
        return out
    A, B = merged(a_iv), merged(b_iv)
    i = j = 0
    tot = 0.0
    while i < len(A) and j < len(B):
        lo, hi = max(A[i][0], B[j][0]), min(A[i][1], B[j][1])
        if hi > lo:
            tot += hi - lo
        if A[i][1] < B[j][1]:
            i += 1
        else:
            j += 1
    return tot


def run(cfg_name, L, M, T, mode_name):
    import torch
    c = inputs.CONFIGS[cfg_name]
    tr = inputs.generate_trace(L, c["n"], c["K"], T, inputs.PRESETS["paper"](c["n"]))
    hm = harness.host_model(L, c["d"], c["ff"], c["n"], c["K"], touched=harness.routed_experts(tr))
    x, _ = inputs.make_hidden(tr, hm.gates)
    mode = {"fetch": moe.MISS_FETCH, "host": moe.MISS_HOST_COMPUTE, "pull": moe.MISS_PULL}[mode_name]
    lib = moe.lib()
    lib.moe_debug_stream_timeline.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
    lib.moe_debug_stream_timeline.restype = ctypes.c_int64
    with harness.open_moe(hm) as m:
        m.configure(ways=M, indexes=L, miss_mode=mode)
        lib.moe_debug_stream_timeline(m._h.value, None, 0)  # drop anything recorded so far
        y = harness.run_decode(m, x)
        cap = 1 << 20
        buf = np.zeros((cap, 5), np.float64)
        n = lib.moe_debug_stream_timeline(m._h.value, buf.ctypes.data, cap)
        st = m.stats(-1)
    rec = buf[:max(n, 0)]
    ker = rec[rec[:, 0] == 0]
    fet = rec[rec[:, 0] == 1]
    act = rec[rec[:, 0] == 2]
    t0 = float(ker[:, 2].min())
    t1 = float(ker[:, 3].max())
    fetch_iv = [(a, b) for a, b in fet[:, 2:4]]
    fetch_busy = union_len(fetch_iv)
    # overlap of each copy with kernels of OTHER calls
    other = 0.0
    for s_, a, b in fet[:, 1:4]:
        other += overlap_len([(a, b)], [(ka, kb) for ks, ka, kb in ker[:, 1:4] if ks != s_])
    out = {"config": cfg_name, "layers": L, "ways": M, "tokens": T, "miss_mode": mode_name,
           "decode_ms": t1 - t0, "tokens_per_s": T / ((t1 - t0) * 1e-3), "calls": int(len(ker)),
           "misses": st["expert_misses"], "fetches": st["fetches"], "host_computed": st["host_computed"],
           "fetch_copies": int(len(fet)), "fetch_bytes": float(fet[:, 4].sum()),
           "link_gbs_busy": float(fet[:, 4].sum()) / (fetch_busy * 1e-3) / 1e9 if fetch_busy > 0 else None,
           "fetch_busy_frac_of_decode": fetch_busy / (t1 - t0),
           "per_copy_gbs_median": float(np.median(fet[:, 4] / ((fet[:, 3] - fet[:, 2]) * 1e-3) / 1e9)) if len(fet) else None,
           "fetch_time_overlapped_by_other_calls_kernels": other / fetch_busy if fetch_busy > 0 else None,
           "activation_copies": int(len(act)),
           "activation_copy_us_mean": float(np.mean(act[:, 3] - act[:, 2]) * 1e3) if len(act) else None,
           "y_finite": bool(np.isfinite(y).all())}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mixtral-8x7b")
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--ways", type=int, default=4)
    ap.add_argument("--tokens", type=int, default=8)
    ap.add_argument("--modes", default="fetch,host")
    args = ap.parse_args()
    for mode in args.modes.split(","):
        print(json.dumps(run(args.config, args.layers, args.ways, args.tokens, mode)), flush=True)


if __name__ == "__main__":
    main()
