#!/usr/bin/env python
"""Is the decode step host-bound? For each shape: (a) host microseconds per moe_layer_forward
call (Python binding + C++ runtime + launch), and (b) the device time per step twice —
back to back as the host enqueues them, and with the launch queue pre-filled (the K steps
are enqueued behind torch.cuda._sleep, so the GPU never waits for the host).

    python tools/host_overhead.py [--shapes phi-3.5-moe,8x22b-P8] [--steps 400]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench_shapes  # noqa: E402
import harness  # noqa: E402


def main():
    import torch
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="tiny,8x22b-P8,phi-3.5-moe,mixtral-8x7b")
    ap.add_argument("--steps", type=int, default=400)
    args = ap.parse_args()
    shapes = dict(bench_shapes.SHAPES, tiny=(64, 128, 8, 2))
    for name in args.shapes.split(","):
        d, ff, n, K = shapes[name]
        hm = harness.host_model(1, d, ff, n, K)
        x, _ = harness.hidden_states(hm, 64, "uniform")
        xd = torch.from_numpy(x.view(np.int16)).cuda()
        yd = torch.empty((64, d), dtype=torch.float32, device="cuda")
        xs = [xd[t, 0].data_ptr() for t in range(64)]
        ys = [yd[t].data_ptr() for t in range(64)]
        with harness.open_moe(hm) as m:
            m.configure(ways=n, indexes=1, warm_start=True)
            s = torch.cuda.Stream()
            sp = s.cuda_stream
            for i in range(50):
                m.forward(0, xs[i % 64], ys[i % 64], sp)
            s.synchronize()
            out = {"shape": name}
            # (b1) back to back, as enqueued
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            h0 = time.perf_counter()
            for i in range(args.steps):
                m.forward(0, xs[i % 64], ys[i % 64], sp)
            h1 = time.perf_counter()
            e1.record(s)
            e1.synchronize()
            out["host_us_per_call_live"] = (h1 - h0) * 1e6 / args.steps
            out["device_us_per_step_live"] = e0.elapsed_time(e1) * 1e3 / args.steps
            # (b2) queue pre-filled behind a GPU sleep
            with torch.cuda.stream(s):
                torch.cuda._sleep(int(2e9 * max(0.05, args.steps * 60e-6)))
            e0.record(s)
            h0 = time.perf_counter()
            for i in range(args.steps):
                m.forward(0, xs[i % 64], ys[i % 64], sp)
            h1 = time.perf_counter()
            e1.record(s)
            e1.synchronize()
            out["host_us_per_call_queued"] = (h1 - h0) * 1e6 / args.steps
            out["device_us_per_step_prefilled"] = e0.elapsed_time(e1) * 1e3 / args.steps
            # (a) the binding alone vs the raw ctypes call
            lib = m._h
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
