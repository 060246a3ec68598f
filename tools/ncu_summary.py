#!/usr/bin/env python
"""Summarise ncu captures into profiles/ (run here, on the CPU box, after gpurun).

    python tools/ncu_summary.py --round 1 --full gpurun_out/prof_fused.ncu-rep [more.ncu-rep] \
        --launches gpurun_out/launches.csv

Writes profiles/ncu_full_rNN.json (per-kernel DRAM bytes per launch, duration, throughput,
stall summary), profiles/rNN_ncu_full.txt (human-readable) and profiles/rNN_launches.txt
(per-kernel share of the launch list).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "launch__shared_mem_per_block_dynamic": "dyn_smem",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1024, "MB": 1024 ** 2, "ms": 1e3, "us": 1.0, "ns": 1e-3, "nsecond": 1e-3, "usecond": 1.0,
              "msecond": 1e3, "%": 1, "": 1}


def short(name: str) -> str:
    for k in ("expert_fused", "route_probe", "expert_gateup", "expert_down", "write_ready"):
        if k in name:
            return {"expert_fused": "expert_ffn", "expert_gateup": "expert_ffn"}.get(k, k)
    return name[:40]


def raw(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = {"kernel": row[head.index("Kernel Name")]}
        for k, nm in KEYS.items():
            if k in head:
                i = head.index(k)
                try:
                    v = float(row[i].replace(",", ""))
                except ValueError:
                    continue
                sc = UNIT_SCALE.get(units[i], 1)
                d[nm] = v * sc
        res.append(d)
    return res


def stalls(rep: str, kernel: str, top: int = 8):
    fn = kernel.split("(")[0].split("::")[-1]
    out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{fn}", "--page", "source", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    h = rows[1]
    if "Warp Stall Sampling (All Samples)" not in h:
        return []
    si = h.index("Warp Stall Sampling (All Samples)")
    body = [r for r in rows[2:] if len(r) > si and r[si].isdigit()]
    tot = sum(int(r[si]) for r in body) or 1
    body.sort(key=lambda r: -int(r[si]))
    return [{"sass": r[1].strip(), "share": round(int(r[si]) / tot, 4)} for r in body[:top]]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", type=int, required=True)
    ap.add_argument("--full", nargs="*", default=[])
    ap.add_argument("--launches")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    tag = f"r{a.round:02d}"
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    summary = {"round": a.round, "note": a.note, "kernels": {}, "dram_bytes_per_launch": {}}
    lines = []
    for rep in a.full:
        for d in raw(rep):
            k = short(d["kernel"])
            d["top_stall_sass"] = stalls(rep, d["kernel"])
            summary["kernels"][k] = d
            if "dram_read" in d:
                summary["dram_bytes_per_launch"][k] = d["dram_read"] + d.get("dram_write", 0.0)
            lines.append(f"== {k}  ({d['kernel']})  from {os.path.basename(rep)}")
            for nm in ("duration", "dram_read", "dram_write", "dram_pct_of_peak", "warps_active_pct", "registers",
                       "dyn_smem", "grid", "block", "smem_bank_conflicts", "tensor_pipe_pct"):
                if nm in d:
                    unit = {"duration": "us", "dram_read": "B", "dram_write": "B"}.get(nm, "")
                    lines.append(f"   {nm:22s} {d[nm]:,.3f} {unit}")
            if "duration" in d and "dram_read" in d:
                gbs = (d["dram_read"] + d.get("dram_write", 0)) / (d["duration"] * 1e-6) / 1e9
                lines.append(f"   {'dram GB/s (ncu)':22s} {gbs:,.1f}")
            for s in d["top_stall_sass"]:
                lines.append(f"   stall {100 * s['share']:5.1f}%  {s['sass']}")
    if a.launches:
        rows = list(csv.reader(open(a.launches)))
        hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        h = rows[hi]
        ki, vi = h.index("Kernel Name"), h.index("Metric Value")
        ui = h.index("Metric Unit") if "Metric Unit" in h else None
        per = defaultdict(list)
        for r in rows[hi + 1:]:
            try:
                sc = {"usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(r[ui], 1.0) if ui is not None else 1.0
                per[short(r[ki])].append(float(r[vi].replace(",", "")) * sc)
            except (ValueError, IndexError):
                continue
        tot = sum(sum(v) for v in per.values()) or 1
        ll = [f"launch list {os.path.basename(a.launches)} (ncu gpu__time_duration.sum, serialised, cold-cache):"]
        summary["launch_share"] = {}
        for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            share = sum(v) / tot
            summary["launch_share"][k] = {"launches": len(v), "avg_ns": sum(v) / len(v), "share": share}
            ll.append(f"   {k:16s} launches {len(v):5d}  avg {sum(v) / len(v) / 1e3:9.2f} us  share {100 * share:5.1f}%")
        with open(os.path.join(prof, f"{tag}_launches.txt"), "w") as f:
            f.write("\n".join(ll) + "\n")
        lines += [""] + ll
    with open(os.path.join(prof, f"ncu_full_{tag}.json"), "w") as f:
        json.dump(summary, f, indent=1)
    with open(os.path.join(prof, f"{tag}_ncu_full.txt"), "w") as f:
        f.write((a.note + "\n" if a.note else "") + "\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
