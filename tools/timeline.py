#!/usr/bin/env python
"""Per-CTA timeline of the fused decode kernel (MOE_DEBUG_TS=1, globaltimer ns).

Runs `--steps` warm decode steps of one shape (bench_shapes.SHAPES) back to back, then
reads the per-CTA phase marks of the LAST call (moe_debug_timestamps) and prints, for
each mark, the median / min / max over CTAs relative to the END of the previous call
(the latest CTA end of call seq-1, from moe_debug_step_ts): what the one-kernel step
spends between the previous step's last byte and this step's first / last byte.

    python tools/timeline.py --shape mixtral-8x7b    (loads lib/libmoe_debug.so)
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("MOE_DEBUG_TS", "1")
# the marks exist only in the debug build of the library
os.environ.setdefault("MOE_LIB_PATH", os.path.join(ROOT, "paper_2512_16473_b200", "lib", "libmoe_debug.so"))

import numpy as np  # noqa: E402

import bench_shapes  # noqa: E402
import harness  # noqa: E402
import paper_2512_16473_b200 as moe  # noqa: E402

# per-CTA slots written by expert_fused_kernel (kTsPerCta = 48)
MARKS = {0: "cta_start", 8: "pdl_wait_done", 9: "x_landed", 10: "router_has_logits", 1: "route_published",
         11: "route_decided", 2: "first_row_consumed", 3: "phase_A_done", 4: "phase_B_first_h", 6: "phase_B_second_h",
         5: "cta_end", 12: "prod_last_A_issued", 13: "prod_last_Bo0_issued", 14: "prod_last_B_issued",
         15: "first_B_row_seen", 16: "cta_out_of_phase_A", 17: "h_first_published",
         19: "merged_h0_published", 20: "merged_h1_published", 22: "merged_h1_landed_warp0",
         23: "warp0_last_B_chunk_done", 38: "prod_first_row_issued", 39: "st0_pub_h0_before", 40: "st0_pub_h0_after",
         41: "st0_end_pub_seg0_before", 42: "st0_end_pub_seg0_after", 43: "st0_end_pub_seg1_before",
         44: "st0_end_pub_seg1_after", 46: "router_h1_copy_landed", 47: "router_h1_settled"}
KSTS_RING, KSTS_HEAD = 64, 8


def main():
    import torch
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="mixtral-8x7b")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--tokens", type=int, default=64)
    args = ap.parse_args()
    d, ff, n, K = bench_shapes.SHAPES[args.shape]
    hm = harness.host_model(1, d, ff, n, K)
    x, _ = harness.hidden_states(hm, args.tokens, "uniform")
    xd = torch.from_numpy(x.view(np.int16)).cuda()
    yd = torch.empty((args.tokens, d), dtype=torch.float32, device="cuda")
    lib = moe.lib()
    lib.moe_debug_timestamps.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong]
    lib.moe_debug_step_ts.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    with harness.open_moe(hm) as m:
        m.configure(ways=n, indexes=1, warm_start=True)
        s = torch.cuda.Stream()
        for i in range(args.steps):
            m.forward(0, xd[i % args.tokens, 0].data_ptr(), yd[i % args.tokens].data_ptr(), s.cuda_stream)
        s.synchronize()
        G = m.runtime_info()["grid"]
        ts = np.zeros(G * 64, np.uint64)
        tstride = lib.moe_debug_timestamps(m._h.value, ts.ctypes.data, ts.size)
        assert tstride > 0, "per-CTA marks need the debug build"
        ts = ts[:G * tstride]
        stride = KSTS_HEAD + 2 * G
        sts = np.zeros(KSTS_RING * stride, np.uint64)
        lib.moe_debug_step_ts(m._h.value, sts.ctypes.data)
        lib.moe_debug_events.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        ev = np.zeros(G * 512 * 2, np.uint64)
        lib.moe_debug_events(m._h.value, ev.ctypes.data)
    ts = ts.reshape(G, tstride).astype(np.int64)
    sts = sts.reshape(KSTS_RING, stride).astype(np.int64)
    last = args.steps  # seq of the last call (seqs start at 1)
    prev = sts[(last - 1) % KSTS_RING]
    prev_end = int(prev[KSTS_HEAD + G:KSTS_HEAD + 2 * G].max())
    cur = sts[last % KSTS_RING]
    cur_end = int(cur[KSTS_HEAD + G:KSTS_HEAD + 2 * G].max())
    out = {"shape": args.shape, "grid": G, "step_us_prev_end_to_end": (cur_end - prev_end) / 1e3, "marks_us": {}}
    for slot, name in MARKS.items():
        v = ts[:, slot]
        v = v[v > 0] - prev_end
        if v.size:
            out["marks_us"][name] = {"median": statistics.median(v.tolist()) / 1e3, "min": float(v.min()) / 1e3,
                                     "max": float(v.max()) / 1e3}
    # SM-clock marks inside the routing prologue (clock64, same CTA): 24 gate rows in smem
    # (consumer warp 0, after x), 25 x landed (consumer
    # warp 0), 26 its gate GEMV done, 27 router warp past the logits barrier, 28 top-K done,
    # 29 probe done (all-hit publish), 30 LRU bookkeeping done, 31 decision returned
    names = {24: "gate_rows_landed", 25: "x_landed", 26: "gemv_done", 27: "router_has_logits", 28: "topk_done", 29: "probe_published",
             30: "lru_done", 31: "decided", 32: "fast_path_published", 35: "fast_z_summed", 36: "fast_ranked",
             37: "fast_all_resident"}
    base = ts[:, 27]
    cyc = {}
    for slot, name in names.items():
        v = ts[:, slot]
        ok = (v > 0) & (base > 0)
        if ok.any():
            cyc[name] = statistics.median((v[ok] - base[ok]).tolist())
    out["router_cycles_rel_logits"] = cyc
    # the CTAs that end last (the next call's PDL wait follows the LAST one)
    end = ts[:, 5] - prev_end
    last = np.argsort(-end)[:6]
    out["latest_ctas"] = [dict({"cta": int(c)}, **{nm: round(float(ts[c, sl] - prev_end) / 1e3, 2)
                                                    for sl, nm in MARKS.items() if ts[c, sl] > 0})
                          for c in last[:3]]
    out["end_us_quantiles"] = {q: float(np.quantile(end, q)) / 1e3 for q in (0.1, 0.5, 0.9, 0.97, 1.0)}
    # effective SM clock of each CTA over the kernel: clock64 / globaltimer between its start
    # (slot 33 / 0) and its end (slot 34 / 5)
    ok = (ts[:, 34] > 0) & (ts[:, 33] > 0) & (ts[:, 5] > ts[:, 0])
    if ok.any():
        mhz = (ts[ok, 34] - ts[ok, 33]) / ((ts[ok, 5] - ts[ok, 0]) / 1e3)
        out["sm_mhz_effective"] = {"median": float(np.median(mhz)), "min": float(mhz.min()), "max": float(mhz.max())}
    # stage-data arrival curve: bytes the consumers took per 0.5 us bin (upper bound on the
    # landing time: a consumer still busy sees its stage later), from the per-CTA events
    ev = ev.reshape(G * 512, 2).astype(np.int64)
    t = ev[:, 0] - prev_end
    ok = (ev[:, 0] > prev_end) & (ev[:, 0] <= cur_end)
    if ok.any():
        tb = t[ok]
        by = ev[ok, 1] & 0xffffffff
        ph = ev[ok, 1] >> 32
        binw = 500
        nb = int(tb.max() // binw) + 1
        curve = []
        for k in range(nb):
            sel = (tb >= k * binw) & (tb < (k + 1) * binw)
            curve.append(round(float(by[sel].sum()) / binw / 1e3, 2))  # TB/s (bytes/ns / 1e3)
        out["arrival_TBs_per_0.5us"] = curve
        out["phase_bytes_first_last_us"] = {int(p): [round(float(tb[ph == p].min()) / 1e3, 2),
                                                    round(float(tb[ph == p].max()) / 1e3, 2),
                                                    int(by[ph == p].sum())] for p in np.unique(ph)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
