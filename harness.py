"""Workload harness shared by tests/, bench.py and __graft_entry__.smoke().

Builds the seeded synthetic workload of a BASELINE.json config (inputs/) as HOST
buffers in the library's blob layout (pinned through torch when CUDA is present) and
opens a ``paper_2512_16473_b200.Moe`` context over them. It performs none of the
method's arithmetic and never imports ``oracle``.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

import inputs
import paper_2512_16473_b200 as moe


def _cuda():
    try:
        import torch
        return torch if torch.cuda.is_available() else None
    except Exception:  # pragma: no cover
        return None


@dataclass
class HostModel:
    L: int
    d: int
    ff: int
    n: int
    K: int
    tp_size: int = 1
    tp_rank: int = 0
    gates: list = field(default_factory=list)
    blobs: list = field(default_factory=list)
    pinned: bool = False
    _keep: object = None

    @property
    def ffr(self) -> int:
        return self.ff // self.tp_size

    @property
    def slot_bytes(self) -> int:
        return moe.slot_bytes(self.d, self.ff, self.tp_size)

    def weights(self, l: int, e: int):
        """(W1, W3, W2) numpy views of this rank's blob of expert (l, e)."""
        return moe.blob_views(self.blobs[l * self.n + e], self.d, self.ffr)


def host_model(L: int, d: int, ff: int, n: int, K: int, tp_size: int = 1, tp_rank: int = 0,
               pinned: bool | None = None, touched=None) -> HostModel:
    """Host backing store of an (L, d, ff, n, K) model. `touched`: optional set of (layer,
    expert) pairs a workload will route to (known in advance: the hidden states are built for
    a generated routing, harness.hidden_states); only those get their seeded weights, every
    other blob pointer aliases one all-zero blob — a full-depth model then needs host memory
    for the experts it uses only (a mis-routed call would read zeros and fail the parity
    checks)."""
    torch = _cuda()
    if pinned is None:
        pinned = torch is not None
    sb = moe.slot_bytes(d, ff, tp_size)
    keys = [(l, e) for l in range(L) for e in range(n)]
    tset = None if touched is None else set(touched)
    real = keys if tset is None else [k for k in keys if k in tset]
    nblob = len(real) + (0 if touched is None else 1)
    total = nblob * sb
    if pinned and torch is not None:
        buf = moe.PinnedBuffer(total)     # cudaHostAlloc, exact size (torch rounds to 2^k)
        arr = buf.array
    else:
        buf = arr = np.empty(total, np.uint8)
        pinned = False
    hm = HostModel(L, d, ff, n, K, tp_size, tp_rank, pinned=pinned, _keep=buf)
    hm.gates = [inputs.gate_weights(l, n, d) for l in range(L)]
    where = {k: i for i, k in enumerate(real)}
    if touched is not None:
        arr[len(real) * sb:(len(real) + 1) * sb] = 0
    for (l, e) in keys:
        i = where.get((l, e), len(real))
        blob = arr[i * sb:(i + 1) * sb]
        hm.blobs.append(blob)
        if (l, e) in where:
            w1, w3, w2 = moe.blob_views(blob, d, ff // tp_size)
            inputs.expert_weights_into(w1, w3, w2, l, e, d, ff, tp_rank, tp_size)
    return hm


def routed_experts(trace) -> set:
    """(layer, expert) pairs of a routing trace [T][L][K] (inputs.generate_trace)."""
    T, L, K = trace.shape
    return {(l, int(trace[t, l, r])) for t in range(T) for l in range(L) for r in range(K)}


def open_moe(hm: HostModel, device: int = 0, nccl_id: bytes | None = None) -> moe.Moe:
    return moe.Moe(hm.L, hm.d, hm.ff, hm.n, hm.K, hm.gates, hm.blobs, device=device,
                   tp_size=hm.tp_size, tp_rank=hm.tp_rank, nccl_id=nccl_id, already_pinned=hm.pinned)


def hidden_states(hm: HostModel, T: int, preset: str = "paper"):
    """(x [T][L][d] bf16 bits, intended ranked routing [T][L][K])."""
    tr = inputs.generate_trace(hm.L, hm.n, hm.K, T, inputs.PRESETS[preset](hm.n))
    return inputs.make_hidden(tr, hm.gates)


def run_decode(m: moe.Moe, x: np.ndarray, device: int = 0, stream=None):
    """Device decode of x[t][l] in token-major / layer order; returns y [T][L][d] fp32 (host)."""
    import torch
    T, L, d = x.shape
    dev = torch.device("cuda", device)
    xd = torch.from_numpy(x.view(np.int16)).to(dev)
    yd = torch.empty((T, L, d), dtype=torch.float32, device=dev)
    s = stream or torch.cuda.current_stream(dev)
    for t in range(T):
        for l in range(L):
            m.forward(l, xd[t, l].data_ptr(), yd[t, l].data_ptr(), s.cuda_stream)
    s.synchronize()
    return yd.cpu().numpy()
