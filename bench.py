#!/usr/bin/env python
"""Benchmark of the hot path: one MoE-block decode step (router + cache probe/LRU +
expert SwiGLU GEMVs + combine) per token, through the C-ABI.

N=1 workload = BASELINE.json configs[1]: a single Mixtral-8x7B-shaped MoE layer
(d=4096, ff=14336, 8 experts, top-2), decode batch 1, 8-way cache warm (all experts
resident), routing from the paper-pattern generator. N>1 (torchrun): the same layer with
each expert's ff dimension split across the N ranks, y summed inside the decode kernel
over peer memory (f3; NCCL all-reduce fallback) (north_star (4)); total work fixed
("strong"). The N>1 line also carries a `configs4` record: BASELINE configs[4]'s
Mixtral-8x22B-shaped layer (d=6144, ff=16384) split the same N ways.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0. torch.distributed (gloo)
carries only the barriers, the IPC-handle exchange and the max-over-ranks reduction of the
device-timed region; an NCCL communicator is created only if the fused peer reduction
cannot be wired. When the ranks outnumber the visible GPUs (e.g. the N=2 arm on a one-GPU
box) the run is a REHEARSAL: ranks share GPUs (time-sliced), the line says so and its
numbers are not a measurement of N GPUs.
"""
from __future__ import annotations

import argparse
import datetime
import json
import os
import platform
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import inputs  # noqa: E402

METRIC = "single-request decode tokens/sec; expert-GEMV HBM GB/s vs peak; cache hit rate"
WORKLOAD = "configs[1]: single Mixtral-8x7B-shaped MoE layer (d=4096, ff=14336, 8 experts top-2), decode batch 1"
CFG = inputs.CONFIGS["mixtral-8x7b"]
CFG4 = inputs.CONFIGS["mixtral-8x22b"]
TRACE_TOKENS = 256
# Table III: CPU expert computation time per expert, Mixtral 8x7B, Threadripper 7960X
PAPER_TABLE3_MS = {"1": 44.12, "24": 7.34}


def step_bytes(cfg: dict, world: int) -> int:
    """Algorithmic bytes of one decode step on one rank: the K routed experts' W1+W3+W2
    slices, the gate rows and x."""
    ffr = cfg["ff"] // world
    return cfg["K"] * 3 * cfg["d"] * ffr * 2 + cfg["n"] * cfg["d"] * 2 + cfg["d"] * 2


def workload_config(world: int) -> dict:
    """The `config` object — identical in both arms (the driver compares them)."""
    return {"workload": WORKLOAD, "cache": f"N=1 index, M={CFG['n']} ways, warm (all hits)",
            "parallelism": f"tp{world} (expert ff-split)" if world > 1 else "single GPU",
            "trace_tokens": TRACE_TOKENS, "routing": "paper preset (p_token_reuse=0.15)",
            "l2": f"inputs larger than L2: {step_bytes(CFG, world) / 1e6:.1f} MB of expert weights per step and rank "
                  f"vs 126 MB L2"}


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _ncu_traffic():
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu --set full summary."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_full_*.json")))
    if not files:
        return None
    with open(files[-1]) as f:
        j = json.load(f)
    return j.get("dram_bytes_per_launch", {}).get("expert_ffn")


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.p is not None:
            time.sleep(0.25)
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU oracle legs
def _oracle_layer_inputs(T: int):
    gates = [inputs.gate_weights(0, CFG["n"], CFG["d"])]
    tr = inputs.generate_trace(1, CFG["n"], CFG["K"], max(T, 1), inputs.PRESETS["paper"](CFG["n"]))
    x, _ = inputs.make_hidden(tr, gates)
    return gates, tr, x


def _time_oracle(x, gates, W, tokens: int, budget_s: float):
    """Decode `tokens` steps of the configs[1] layer through the oracle (at least 1, stop
    early past the budget). Returns (steps, seconds)."""
    import oracle
    done = 0
    t0 = time.perf_counter()
    while done < tokens and (done < 1 or time.perf_counter() - t0 < budget_s):
        t = done % x.shape[0]
        oracle.decode(x[t:t + 1], gates, lambda l, e: W[(l, e)], N=1, M=8, K=CFG["K"], warm_start=True)
        done += 1
    return done, time.perf_counter() - t0


def cpu_baseline_sample(budget_s: float = 12.0) -> dict:
    """The oracle (as it stands) timed on a bounded sample of the same workload on this
    box's host cores, at one thread and at all threads (rank 0, N=1 only), next to the
    paper's own CPU expert times (Table III)."""
    import oracle
    cores = len(os.sched_getaffinity(0))
    gates, tr, x = _oracle_layer_inputs(8)
    W = {}
    for t in range(8):  # only the experts the sample touches, generated before timing
        for e in tr[t, 0]:
            if (0, int(e)) not in W:
                W[(0, int(e))] = inputs.expert_weights(0, int(e), CFG["d"], CFG["ff"])
    legs = {}
    for threads, tokens, budget in ((1, 4, budget_s / 3), (cores, 8, budget_s)):
        oracle.set_threads(threads)
        n, dt = _time_oracle(x, gates, W, tokens, budget)
        legs[threads] = {"threads": threads, "tokens": n, "tokens_per_s": n / dt,
                         "ms_per_layer_step": 1000.0 * dt / n, "ms_per_expert": 1000.0 * dt / n / CFG["K"]}
    oracle.set_threads(cores)
    allc = legs[cores]
    return {"value": allc["tokens_per_s"], "unit": "tokens/s", "cores": cores, "kind": "oracle",
            "cpu_model": _cpu_model(),
            "sample": f"{allc['tokens']} decode tokens of the configs[1] layer (gate GEMV + top-2 + LRU + 2 SwiGLU "
                      f"experts) at {cores} threads, {legs[1]['tokens']} at 1 thread; plain fp32 C oracle, OpenMP "
                      f"row-parallel",
            "threads_1": legs[1], "threads_all": allc,
            "paper_table3": {"ms_per_expert_by_threads": PAPER_TABLE3_MS, "cpu": "AMD Threadripper 7960X (24 cores)",
                             "cite": "PAPER.md:296-299 (Table III, Mixtral 8x7B expert computation time)"}}


def run_reference(args, rank: int, world: int) -> None:
    """The oracle, as it stands, on this box's host cores (the reference arm for this tier)."""
    if rank != 0:
        return
    import oracle
    cores = len(os.sched_getaffinity(0))
    oracle.set_threads(cores)
    gates, tr, x = _oracle_layer_inputs(TRACE_TOKENS)
    W = {}
    for e in range(CFG["n"]):  # weight generation is input preparation, outside the timed region
        W[(0, e)] = inputs.expert_weights(0, e, CFG["d"], CFG["ff"])
    budget = float(os.environ.get("BENCH_REF_BUDGET_S", "90"))
    _time_oracle(x, gates, W, args.warmup, budget)
    steps, dt = _time_oracle(x, gates, W, args.steps, budget)
    v = steps / dt
    sample = (f"{steps} of {args.steps} requested decode tokens through the oracle (time-bounded at {budget:.0f} s), "
              f"{cores} OpenMP threads on a {_cpu_model()}")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": steps, "warmup": args.warmup, "ms_per_step": 1000.0 * dt / steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded counter-based bf16 weights, paper-pattern routing)",
            "config": workload_config(world),
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": cores, "kind": "oracle", "sample": sample,
                             "cpu_model": _cpu_model()},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
class Group:
    """torch.distributed over gloo: barriers, object exchange, max over ranks (CPU tensors)."""

    def __init__(self, world: int):
        self.world = world
        self.dist = None
        if world > 1:
            import torch.distributed as dist
            dist.init_process_group("gloo", timeout=datetime.timedelta(minutes=10))
            self.dist = dist

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def max(self, v: float) -> float:
        if not self.dist:
            return v
        import torch
        t = torch.tensor([v], dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.dist:
            self.dist.destroy_process_group()


def open_layer(cfg: dict, group: Group, rank: int, dev_index: int):
    """One decode context over a 1-layer model of `cfg`'s shape (this rank's ff slice),
    8 ways warm, with the y reduction wired for N>1: fused peer memory first; an NCCL
    communicator only if that fails (or MOE_TP_REDUCE=nccl). Returns (hm, m, tp_reduce)."""
    import harness
    world = group.world
    hm = harness.host_model(1, cfg["d"], cfg["ff"], cfg["n"], cfg["K"], tp_size=world, tp_rank=rank)
    tp_reduce = "none"
    m = None
    if world > 1 and os.environ.get("MOE_TP_REDUCE", "fused") != "nccl":
        from paper_2512_16473_b200 import tp
        m = harness.open_moe(hm, device=dev_index)
        r = tp.connect_peers(m)
        if r == "fused-peer":
            tp_reduce = "fused peer-memory reduction in the decode kernel's epilogue"
        else:
            m.close()
            m = None
            tp_reduce = f"nccl all-reduce after the kernel (fused peer reduction unavailable: {r})"
    if world > 1 and m is None:
        from paper_2512_16473_b200 import tp
        nccl_id = tp.broadcast_nccl_id()
        m = harness.open_moe(hm, device=dev_index, nccl_id=nccl_id)
        if tp_reduce == "none":
            tp_reduce = "nccl all-reduce after the kernel (MOE_TP_REDUCE=nccl)"
    if m is None:
        m = harness.open_moe(hm, device=dev_index)
    m.configure(ways=cfg["n"], indexes=1, warm_start=True)
    group.barrier()
    return hm, m, tp_reduce


def timed_steps(m, group: Group, dev, stream, xs, ys, first: int, n_steps: int):
    """K back-to-back decode steps bracketed by barrier + synchronize, CUDA events on the
    launch stream; returns (device ms max over ranks, host enqueue us per step)."""
    import torch
    group.barrier()
    torch.cuda.synchronize(dev)
    sp = stream.cuda_stream
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    h0 = time.perf_counter()
    T = len(xs)
    for i in range(n_steps):
        t = (first + i) % T
        m.forward(0, xs[t], ys[t], sp)
    h1 = time.perf_counter()
    ev1.record(stream)
    ev1.synchronize()
    group.barrier()
    torch.cuda.synchronize(dev)
    return group.max(ev0.elapsed_time(ev1)), (h1 - h0) * 1e6 / max(n_steps, 1)


def run_ours(args, rank: int, world: int, local_rank: int) -> None:
    import torch
    import harness

    ngpu = torch.cuda.device_count()
    rehearsal = world > ngpu
    dev = torch.device("cuda", local_rank % ngpu)
    torch.cuda.set_device(dev)
    group = Group(world)
    hm, m, tp_reduce = open_layer(CFG, group, rank, dev.index)
    x, _ = harness.hidden_states(hm, TRACE_TOKENS, "paper")
    xd = torch.from_numpy(x.view(np.int16)).to(dev)          # [T][1][d] resident in HBM
    yd = torch.empty((TRACE_TOKENS, CFG["d"]), dtype=torch.float32, device=dev)
    xs = [xd[t, 0].data_ptr() for t in range(TRACE_TOKENS)]
    ys = [yd[t].data_ptr() for t in range(TRACE_TOKENS)]
    stream = torch.cuda.Stream(dev)
    for i in range(args.warmup):
        m.forward(0, xs[i % TRACE_TOKENS], ys[i % TRACE_TOKENS], stream.cuda_stream)
    stream.synchronize()
    m.stats(-1)

    # (1) headline: the K timed steps exactly as a user runs them (no profiling events)
    with ClockSampler(dev.index) as clk:
        ms, host_us = timed_steps(m, group, dev, stream, xs, ys, args.warmup, args.steps)
    # (2) roofline: the same steps again with CUDA events around every kernel on the stream
    m.profile(True)
    m.profile_read()
    ms_prof, _ = timed_steps(m, group, dev, stream, xs, ys, args.warmup, args.steps)
    prof = m.profile_read()
    m.profile(False)
    st = m.stats(-1)
    rinfo = m.runtime_info()

    # end-to-end: host buffers through moe_layer_forward_host (H2D x, D2H y, sync per step)
    xh = torch.from_numpy(x.view(np.int16)[:, 0, :].copy()).pin_memory()
    yh = torch.empty((CFG["d"],), dtype=torch.float32).pin_memory()
    e2e_steps = 0 if args.skip_e2e else max(1, min(args.steps, 20 if rehearsal else 2000))
    for i in range(min(args.warmup, 20)):
        m.forward_host(0, xh[i % TRACE_TOKENS].data_ptr(), yh.data_ptr())
    group.barrier()
    t0 = time.perf_counter()
    for i in range(e2e_steps):
        m.forward_host(0, xh[i % TRACE_TOKENS].data_ptr(), yh.data_ptr())
    e2e_s = group.max(max(time.perf_counter() - t0, 1e-9))
    m.close()

    cfg4 = run_configs4(args, group, rank, dev, rehearsal) if world > 1 and not args.no_configs4 else None

    if rank != 0:
        group.close()
        return
    ms_step = ms / args.steps
    ffr = CFG["ff"] // world
    d, K = CFG["d"], CFG["K"]
    bytes_gateup = K * 2 * ffr * d * 2          # W1 + W3 rows of the K routed experts (per rank)
    sbytes = step_bytes(CFG, world)
    peak, peak_src = _peaks()
    ffn, dn, rt = prof["expert_ffn"], prof["expert_down"], prof["route_probe"]
    fused = dn["launches"] == 0 and rt["launches"] == 0   # one kernel per step: router inside
    ffn_ms = ffn["ms"] / max(ffn["launches"], 1)
    dn_ms = dn["ms"] / max(dn["launches"], 1)
    rt_ms = rt["ms"] / max(rt["launches"], 1)
    kname = "expert_fused (router + cache probe + gate/up + down + combine)" if fused else "expert_gateup"
    kbytes = sbytes if fused else bytes_gateup
    if fused and (world == 1 or rinfo.get("tp_reduce") == "fused-peer"):
        # the timed region holds exactly K back-to-back launches of this one kernel and
        # nothing else: its average launch duration is the region's event time / K
        launch_ms = ms_step
        launch_src = "CUDA events over the timed region / K (one kernel per step, launch stream)"
    else:
        launch_ms = ffn_ms
        launch_src = "CUDA events around every kernel (second pass over the same steps)"
    achieved = kbytes / (launch_ms * 1e-3) / 1e9
    launches_per_step = 1 if fused else 3      # our kernels (an NCCL all-reduce is not counted)
    line = {
        "metric": METRIC, "value": 1000.0 / ms_step, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded counter-based bf16 weights of Mixtral-8x7B expert shape, paper-pattern routing, "
                "margin-guaranteed hidden states)",
        "config": workload_config(world),
        "runtime": rinfo, "tp_reduce": tp_reduce if world > 1 else None,
        "roofline": {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": _ncu_traffic() if world == 1 else None,
                     "algorithmic_bytes_per_launch": kbytes, "avg_launch_us": launch_ms * 1e3,
                     "avg_launch_src": launch_src, "isolated_launch_us": ffn_ms * 1e3,
                     "peak_source": peak_src,
                     "step": {"bytes": sbytes, "gbs": sbytes / (ms_step * 1e-3) / 1e9,
                              "frac": sbytes / (ms_step * 1e-3) / 1e9 / peak},
                     "kernels_us": {"route_probe": rt_ms * 1e3 if not fused else None, "expert_ffn": ffn_ms * 1e3,
                                    "expert_down": dn_ms * 1e3 if not fused else None},
                     "profiled_ms_per_step": ms_prof / args.steps, "host_enqueue_us_per_step": host_us},
        "e2e": {"value": e2e_steps / e2e_s, "unit": "tokens/s", "h2d_bytes_per_step": d * 2,
                "d2h_bytes_per_step": d * 4, "steps": e2e_steps,
                "path": "moe_layer_forward_host (pinned host x/y, zero-copy: the kernel reads x from and writes y "
                        "to host memory), host wall clock incl. the per-step synchronisation"},
        "gpu_launches": args.steps * launches_per_step,
        "hit_rate": {"expert(s)_hit": st["at_least_one_hit"] / max(st["accesses"], 1),
                     "all_k_hit": st["all_k_hit"] / max(st["accesses"], 1),
                     "per_expert": st["expert_hits"] / max(st["expert_hits"] + st["expert_misses"], 1),
                     "note": "M = n = 8 warm: every expert resident by construction (the miss-path rates are in "
                             "profiles/*fig6*)"},
        "clocks": clk.summary(),
    }
    if rehearsal:
        line["rehearsal"] = {"physical_gpus": ngpu, "note": f"{world} ranks time-sliced on {ngpu} GPU(s): a check of "
                             "the N>1 code path and JSON line, not a measurement of N GPUs"}
    if cfg4 is not None:
        line["configs4"] = cfg4
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_sample()
    print(json.dumps(line), flush=True)
    group.close()


def run_configs4(args, group: Group, rank: int, dev, rehearsal: bool) -> dict:
    """BASELINE configs[4]: one Mixtral-8x22B-shaped layer (d=6144, ff=16384, 8 experts
    top-2) ff-split across the same N ranks, warm, fused peer reduction: per-rank step time
    and its HBM roofline fraction (the tp-N decode step of that model, layer by layer)."""
    import torch
    import harness
    world = group.world
    hm, m, tp_reduce = open_layer(CFG4, group, rank, dev.index)
    x, _ = harness.hidden_states(hm, 64, "paper")
    xd = torch.from_numpy(x.view(np.int16)).to(dev)
    yd = torch.empty((64, CFG4["d"]), dtype=torch.float32, device=dev)
    xs = [xd[t, 0].data_ptr() for t in range(64)]
    ys = [yd[t].data_ptr() for t in range(64)]
    stream = torch.cuda.Stream(dev)
    for i in range(args.warmup):
        m.forward(0, xs[i % 64], ys[i % 64], stream.cuda_stream)
    stream.synchronize()
    steps = min(args.steps, 20 if rehearsal else 2000)
    ms, host_us = timed_steps(m, group, dev, stream, xs, ys, args.warmup, steps)
    rinfo = m.runtime_info()
    m.close()
    us = ms / steps * 1e3
    nbytes = step_bytes(CFG4, world)
    peak, _ = _peaks()
    return {"workload": f"configs[4]: Mixtral-8x22B-shaped layer (d=6144, ff=16384, 8 experts top-2), ff-split tp{world} "
                        f"(ff_r={CFG4['ff'] // world}), M=8 warm",
            "tokens_per_s_per_layer": 1e6 / us, "us_per_layer_step": us, "steps": steps,
            "bytes_per_rank_step": nbytes, "per_rank_gbs": nbytes / (us * 1e-6) / 1e9,
            "per_rank_frac_of_peak": nbytes / (us * 1e-6) / 1e9 / peak,
            "tokens_per_s_56_layers": 1e6 / us / CFG4["L"], "tp_reduce": tp_reduce, "runtime": rinfo,
            "host_enqueue_us_per_step": host_us}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=6000)
    ap.add_argument("--warmup", type=int, default=200)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs4", action="store_true", help="(N>1) skip the configs[4] record")
    ap.add_argument("--skip-e2e", action="store_true", help="(profiling runs) skip the host-buffer e2e leg")
    args = ap.parse_args()
    if args.warmup < 3:   # (profiling passes run 1-2 steps; such a line is not a bench value)
        print(f"bench.py: warning: --warmup {args.warmup} < 3, the timing rules need W >= 3", file=sys.stderr)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N>1 must be launched with torchrun (one process per GPU)")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
