"""Rehearsal of bench.py's N>1 arm on the GPU(s) at hand (the driver's scaling run launches
`torchrun --nproc-per-node N bench.py --gpus N`): 2 ranks, fused peer reduction wired over
CUDA IPC with no NCCL communicator, one JSON line from rank 0 carrying the headline record,
the roofline object and the configs[4] (Mixtral-8x22B-shaped, tp2) record. On a one-GPU box
both ranks time-slice cuda:0 and the line says it is a rehearsal."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_json_line():
    import torch
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, PYTHONPATH=ROOT)
    env.pop("MOE_TP_REDUCE", None)
    res = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
                          "--steps", "20", "--warmup", "5"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    lines = [l for l in res.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, res.stdout
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and j["steps"] == 20 and j["value"] > 0
    assert j["config"]["parallelism"].startswith("tp2")
    assert j["tp_reduce"].startswith("fused peer-memory"), j["tp_reduce"]
    assert j["runtime"]["tp_reduce"] == "fused-peer" and j["runtime"]["expert_path"] == "fused"
    r = j["roofline"]
    assert r["bound"] == "hbm" and r["achieved"] > 0 and r["unit"] == "GB/s"
    assert r["algorithmic_bytes_per_launch"] == 2 * 3 * 4096 * 7168 * 2 + 8 * 4096 * 2 + 4096 * 2
    c4 = j["configs4"]
    assert c4["workload"].startswith("configs[4]") and c4["us_per_layer_step"] > 0
    assert c4["tp_reduce"].startswith("fused peer-memory")
    assert j["e2e"]["value"] > 0 and j["gpu_launches"] == 20
    if torch.cuda.device_count() < 2:
        assert j["rehearsal"]["physical_gpus"] == torch.cuda.device_count()
