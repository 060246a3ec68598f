"""CPU-only checks of the C-ABI library: it loads, exports every symbol include/moe.h
declares, and rejects invalid arguments before touching the GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2512_16473_b200 as moe
from paper_2512_16473_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "moe.h")).read()
    return sorted(set(re.findall(r"MOE_API\s+[\w\s\*]+?\b(\w+)\s*\(", src)))


def test_header_and_binding_agree():
    declared = _declared_symbols()
    assert set(declared) == set(_abi.EXPORTS), declared


def test_library_exports_every_declared_symbol():
    lib = moe.lib()
    for name in _declared_symbols():
        assert hasattr(lib, name), name
    assert lib.moe_abi_version() == 1


def test_struct_layouts_match_header():
    assert ctypes.sizeof(_abi.LayerStats) == 88
    assert _abi.RECORD_DTYPE.itemsize == 20
    assert ctypes.sizeof(_abi.CacheConfig) == 56
    assert ctypes.sizeof(_abi.ModelDesc) == 40
    assert ctypes.sizeof(_abi.RuntimeInfo) == 32
    assert ctypes.sizeof(_abi.TpExchange) == 80   # {void*, int64, uint8[64]}


@pytest.mark.parametrize("shape,msg", [((0, 64, 128, 8, 2), "bad shape"), ((4, 60, 128, 8, 2), "bad shape"),
                                       ((4, 64, 128, 40, 2), "bad shape"), ((4, 64, 128, 8, 9), "bad shape"),
                                       ((4, 64, 100, 8, 2), None)])
def test_moe_init_rejects_bad_shapes_without_gpu(shape, msg):
    L, d, ff, n, K = shape
    tp = 4 if msg is None else 1  # ff=100 with P=4: ff % (8P) != 0
    gates = [np.zeros((max(n, 1), d), np.uint16) for _ in range(max(L, 1))]
    blobs = [np.zeros(8, np.uint16) for _ in range(max(L, 1) * max(n, 1))]
    with pytest.raises(moe.MoeError) as ei:
        moe.Moe(L, d, ff, n, K, gates, blobs, tp_size=tp, tp_rank=0,
                nccl_id=b"\0" * 128 if tp > 1 else None)
    assert ei.value.status == 1
    assert ("tensor-parallel" if msg is None else msg) in str(ei.value)


def test_nccl_id_must_match_tp_size():
    gates = [np.zeros((8, 64), np.uint16)]
    blobs = [np.zeros(8, np.uint16)] * 8
    with pytest.raises(moe.MoeError, match="nccl_unique_id"):
        moe.Moe(1, 64, 128, 8, 2, gates, blobs, tp_size=1, nccl_id=b"\0" * 128)


def test_slot_layout_helpers():
    d, ffr = 16, 24
    blob = np.arange(3 * d * ffr, dtype=np.uint16).view(np.uint8)
    w1, w3, w2 = moe.blob_views(blob, d, ffr)
    assert w1.shape == (ffr, d) and w3.shape == (ffr, d) and w2.shape == (d, ffr)
    assert w1[0, 0] == 0 and w3[0, 0] == ffr * d and w2[0, 0] == 2 * ffr * d
    assert moe.slot_bytes(4096, 14336) == 352_321_536                 # Mixtral expert ("340 MB")
    assert moe.slot_bytes(4096, 6400) == 157_286_400                  # Phi-3.5-MoE expert ("152 MB")
    assert moe.slot_bytes(6144, 16384, 8) == 603_979_776 // 8


@pytest.mark.parametrize("d,ff", [(64, 128), (200, 136), (1024, 512), (4096, 256)])
def test_host_expert_ffn_matches_oracle(d, ff):
    """The library's host-CPU expert (MOE_MISS_HOST_COMPUTE) vs the oracle, on CPU."""
    import inputs
    import oracle
    blob = np.empty(3 * d * ff, np.uint16)
    w1, w3, w2 = moe.blob_views(blob.view(np.uint8), d, ff)
    inputs.expert_weights_into(w1, w3, w2, 0, 3, d, ff)
    x = inputs.f32_to_bf16(np.random.default_rng(d).standard_normal(d).astype(np.float32))
    ref, _ = oracle.expert_ffn(*inputs.expert_weights(0, 3, d, ff), x)
    for thr in (1, 3):
        out = moe.host_expert_ffn(blob, x, d, ff, threads=thr)
        assert np.abs(out - ref).max() <= 1e-5 * np.abs(ref).max()
    assert np.array_equal(moe.host_expert_ffn(blob, x, d, ff, 1), moe.host_expert_ffn(blob, x, d, ff, 4))


def test_tp_connect_validation_without_gpu():
    """moe_tp_connect_local rejects bad arguments before touching any context."""
    lib = moe.lib()
    assert lib.moe_tp_connect_local(None, 2) == 1
    arr = (ctypes.c_void_p * 1)(None)
    assert lib.moe_tp_connect_local(arr, 1) == 1      # P < 2
    assert lib.moe_tp_connect_local(arr, 9) == 1      # P > 8
    assert lib.moe_tp_connect_ipc(None, None) == 1
    assert lib.moe_tp_exchange_buffer(None, None) == 1
    assert lib.moe_tp_disconnect(None) == 1
