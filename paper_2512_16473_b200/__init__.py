"""B200-native expert-cached MoE decode block (arXiv 2512.16473) — Python binding.

Thin ctypes binding over libmoe.so (include/moe.h): argument marshalling only. The
router, cache probe / LRU update, miss fetch and expert GEMVs all run in the library's
sm_100a kernels and C++ runtime. PyTorch is used by callers only for device memory,
streams and process groups.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _abi
from ._abi import (MISS_FETCH, MISS_HOST_COMPUTE, MISS_PULL, POLICY_FIFO, POLICY_LRU, POLICY_STATIC_RANDOM, PROF_KINDS,
                   RECORD_DTYPE, STAT_FIELDS)

__all__ = ["Moe", "MoeError", "PinnedBuffer", "MISS_FETCH", "MISS_HOST_COMPUTE", "MISS_PULL", "host_expert_ffn", "POLICY_LRU", "POLICY_FIFO", "POLICY_STATIC_RANDOM", "RECORD_DTYPE",
           "STAT_FIELDS", "slot_bytes", "blob_views", "lib", "nccl_unique_id", "PROF_KINDS", "tp_connect_local"]

_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        _lib = _abi.load()
    return _lib


class MoeError(RuntimeError):
    def __init__(self, fn: str, status: int):
        msg = lib().moe_last_error().decode(errors="replace")
        super().__init__(f"{fn} -> {_abi.STATUS.get(status, status)}: {msg}")
        self.status = status


def _check(fn: str, st: int) -> None:
    if st != _abi.MOE_OK:
        raise MoeError(fn, st)


def slot_bytes(d: int, ff: int, tp_size: int = 1) -> int:
    """Bytes of one expert blob / cache slot: 3 * d * (ff / P) * 2 (moe.h)."""
    return 3 * d * (ff // tp_size) * 2


def blob_views(blob: np.ndarray, d: int, ffr: int):
    """(W1 [ffr][d], W3 [ffr][d], W2 [d][ffr]) uint16 views of one expert blob (moe.h layout)."""
    u16 = blob.view(np.uint16)
    assert u16.size == 3 * d * ffr
    n = ffr * d
    return u16[:n].reshape(ffr, d), u16[n:2 * n].reshape(ffr, d), u16[2 * n:].reshape(d, ffr)


class PinnedBuffer:
    """Page-locked host buffer from moe_host_alloc (exact size), exposed as a numpy uint8 array."""

    def __init__(self, nbytes: int):
        p = ctypes.c_void_p()
        _check("moe_host_alloc", lib().moe_host_alloc(nbytes, ctypes.byref(p)))
        self._p = p
        self.nbytes = nbytes
        self.array = np.ctypeslib.as_array((ctypes.c_uint8 * nbytes).from_address(p.value))

    def free(self) -> None:
        if getattr(self, "_p", None):
            self.array = None
            lib().moe_host_free(self._p)
            self._p = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def host_expert_ffn(blob: np.ndarray, x: np.ndarray, d: int, ffr: int, threads: int = 0) -> np.ndarray:
    """The library's host-CPU expert FFN (MOE_MISS_HOST_COMPUTE path) on one blob."""
    out = np.empty(d, np.float32)
    _check("moe_host_expert_ffn", lib().moe_host_expert_ffn(_addr(blob), _addr(x), d, ffr, out.ctypes.data, threads))
    return out


def nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check("moe_nccl_unique_id", lib().moe_nccl_unique_id(buf))
    return bytes(buf)


def tp_connect_local(moes) -> None:
    """Connect the P contexts of one TP group living in this process (moe_tp_connect_local);
    contexts on one GPU then split its SMs (ranks emulated on one device)."""
    arr = (ctypes.c_void_p * len(moes))(*[m._h.value for m in moes])
    _check("moe_tp_connect_local", lib().moe_tp_connect_local(arr, len(moes)))


def _addr(a) -> int:
    if isinstance(a, int):
        return a
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"]
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    raise TypeError(f"cannot take the address of {type(a)}")


class Moe:
    """One MoE decode context (moe_init ... moe_destroy).

    gates: L host arrays, each Wg [n][d] uint16 (bf16 bits).
    blobs: L*n host buffers (numpy / pinned torch tensors / raw addresses), blob[l*n+e] in
           the moe.h slot layout for this rank's ff slice. Caller keeps them alive.
    """

    def __init__(self, L: int, d: int, ff: int, n: int, K: int, gates, blobs, device: int = 0,
                 tp_size: int = 1, tp_rank: int = 0, nccl_id: bytes | None = None,
                 already_pinned: bool = False):
        self.L, self.d, self.ff, self.n, self.K = L, d, ff, n, K
        self.tp_size, self.tp_rank = tp_size, tp_rank
        self.ffr = ff // tp_size
        self._keep = (gates, blobs)
        self._gate_ptrs = (ctypes.c_void_p * max(len(gates), 1))(*[_addr(g) for g in gates])
        self._blob_ptrs = (ctypes.c_void_p * max(len(blobs), 1))(*[_addr(b) for b in blobs])
        if L >= 1 and n >= 1 and (len(gates) < L or len(blobs) < L * n):
            raise ValueError("need L gate arrays and L*n expert blobs")
        self._nccl = (ctypes.c_uint8 * 128)(*nccl_id) if nccl_id is not None else None
        desc = _abi.ModelDesc(L, d, ff, n, K, device, tp_size, tp_rank,
                              ctypes.cast(self._nccl, ctypes.c_void_p) if self._nccl is not None else None)
        w = _abi.Weights(self._gate_ptrs, self._blob_ptrs, int(already_pinned))
        h = ctypes.c_void_p()
        _check("moe_init", lib().moe_init(ctypes.byref(desc), ctypes.byref(w), ctypes.byref(h)))
        self._h = h
        self.geometry = None

    # ------------------------------------------------------------------ lifecycle
    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().moe_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ------------------------------------------------------------------ cache
    def configure(self, ways: int, indexes: int | None = None, cache_bytes: int | None = None,
                  policy: int = POLICY_LRU, warm_start: bool = False, seed: int = 0,
                  pool=None, pool_bytes: int = 0, miss_mode: int = MISS_FETCH, host_threads: int = 0) -> dict:
        if cache_bytes is None:
            cache_bytes = -1
            indexes = self.L if indexes is None else indexes
        cfg = _abi.CacheConfig(cache_bytes, ways, indexes or 0, policy, int(warm_start), seed,
                               _addr(pool) if pool is not None else None, pool_bytes, miss_mode, host_threads)
        geo = _abi.CacheGeometry()
        _check("cache_configure", lib().cache_configure(self._h, ctypes.byref(cfg), ctypes.byref(geo)))
        self.geometry = {f: getattr(geo, f) for f, _ in _abi.CacheGeometry._fields_ if f != "reserved"}
        return self.geometry

    # ------------------------------------------------------------------ forward
    def forward(self, layer: int, x, y, stream=None) -> None:
        """x: device bf16 [d] (torch uint16/bfloat16 tensor or address); y: device fp32 [d]."""
        s = stream if isinstance(stream, int) or stream is None else getattr(stream, "cuda_stream", stream)
        _check("moe_layer_forward", lib().moe_layer_forward(self._h, layer, _addr(x), _addr(y), s))

    def prefill(self, layer: int, x, y, T: int, stream=None) -> None:
        """x: device bf16 [T][d]; y: device fp32 [T][d] (tensor-core batched expert FFN)."""
        s = stream if isinstance(stream, int) or stream is None else getattr(stream, "cuda_stream", stream)
        _check("moe_layer_prefill", lib().moe_layer_prefill(self._h, layer, _addr(x), _addr(y), T, s))

    def forward_host(self, layer: int, x_host, y_host) -> None:
        _check("moe_layer_forward_host", lib().moe_layer_forward_host(self._h, layer, _addr(x_host), _addr(y_host)))

    # ------------------------------------------------------------------ introspection
    def stats(self, layer: int = -1) -> dict:
        s = _abi.LayerStats()
        _check("cache_stats", lib().cache_stats(self._h, layer, ctypes.byref(s)))
        return {f: int(getattr(s, f)) for f in STAT_FIELDS}

    def trace(self, cap: int | None = None) -> np.ndarray:
        n = ctypes.c_int64()
        _check("cache_trace", lib().cache_trace(self._h, None, 0, ctypes.byref(n)))
        m = n.value if cap is None else min(cap, n.value)
        out = np.zeros(m, RECORD_DTYPE)
        _check("cache_trace", lib().cache_trace(self._h, out.ctypes.data if m else None, m, ctypes.byref(n)))
        return out

    def runtime_info(self) -> dict:
        r = _abi.RuntimeInfo()
        _check("moe_get_runtime_info", lib().moe_get_runtime_info(self._h, ctypes.byref(r)))
        return {"expert_path": "fused" if r.expert_path else "split", "pdl": bool(r.pdl),
                "ring_stages": r.ring_stages, "stage_bytes": r.stage_bytes, "grid": r.grid,
                "tp_reduce": {0: "none", 1: "nccl", 2: "fused-peer"}.get(r.tp_reduce, r.tp_reduce)}

    # ------------------------------------------------------------------ fused TP reduction (f3)
    def tp_exchange_buffer(self) -> dict:
        """This rank's exchange buffer: {"dev_ptr", "bytes", "ipc_handle" (64 bytes)}."""
        e = _abi.TpExchange()
        _check("moe_tp_exchange_buffer", lib().moe_tp_exchange_buffer(self._h, ctypes.byref(e)))
        return {"dev_ptr": e.dev_ptr, "bytes": e.bytes, "ipc_handle": bytes(e.ipc_handle)}

    def tp_connect_ipc(self, handles) -> None:
        """handles: the P ranks' 64-byte IPC handles in rank order (all-gathered by the caller)."""
        if len(handles) != self.tp_size or any(len(h) != 64 for h in handles):
            raise ValueError("need tp_size 64-byte IPC handles")
        buf = (ctypes.c_uint8 * (64 * self.tp_size))(*b"".join(handles))
        _check("moe_tp_connect_ipc", lib().moe_tp_connect_ipc(self._h, buf))

    def tp_disconnect(self) -> None:
        _check("moe_tp_disconnect", lib().moe_tp_disconnect(self._h))

    def profile(self, enable: bool = True) -> None:
        _check("moe_profile_enable", lib().moe_profile_enable(self._h, int(enable)))

    def profile_read(self) -> dict:
        p = _abi.Profile()
        _check("moe_profile_read", lib().moe_profile_read(self._h, ctypes.byref(p)))
        return {k: {"ms": p.ms[i], "launches": int(p.launches[i])} for i, k in enumerate(PROF_KINDS)}
