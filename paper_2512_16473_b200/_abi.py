"""ctypes mirror of include/moe.h — argument marshalling only.

Every step of the hot path runs inside libmoe.so (sm_100a kernels + C++ runtime).
There is no Python or CPU fallback: if the library is missing, importing this module
raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MOE_LIB_PATH") or os.path.join(_PKG, "lib", "libmoe.so")  # override: A/B runs

MOE_OK = 0
STATUS = {0: "MOE_OK", 1: "MOE_ERR_INVALID_ARG", 2: "MOE_ERR_OUT_OF_MEMORY", 3: "MOE_ERR_CUDA",
          4: "MOE_ERR_NCCL", 5: "MOE_ERR_STATE", 6: "MOE_ERR_UNSUPPORTED"}
POLICY_LRU, POLICY_FIFO, POLICY_STATIC_RANDOM = 0, 1, 2
PROF_KINDS = ("route_probe", "expert_ffn", "expert_down", "allreduce")
EXPORTS = ("moe_init", "moe_destroy", "cache_configure", "moe_layer_forward",
           "moe_layer_forward_host", "cache_stats", "cache_trace", "moe_profile_enable",
           "moe_profile_read", "moe_nccl_unique_id", "moe_last_error", "moe_abi_version",
           "moe_get_runtime_info", "moe_host_alloc", "moe_host_free", "moe_host_expert_ffn",
           "moe_layer_prefill", "moe_tp_exchange_buffer", "moe_tp_connect_ipc", "moe_tp_connect_local",
           "moe_tp_disconnect")


class ModelDesc(ctypes.Structure):
    _fields_ = [("num_layers", ctypes.c_int32), ("d_model", ctypes.c_int32), ("d_ff", ctypes.c_int32),
                ("num_experts", ctypes.c_int32), ("top_k", ctypes.c_int32), ("device", ctypes.c_int32),
                ("tp_size", ctypes.c_int32), ("tp_rank", ctypes.c_int32),
                ("nccl_unique_id", ctypes.c_void_p)]


class Weights(ctypes.Structure):
    _fields_ = [("gate", ctypes.POINTER(ctypes.c_void_p)), ("expert_blob", ctypes.POINTER(ctypes.c_void_p)),
                ("already_pinned", ctypes.c_int32)]


class CacheConfig(ctypes.Structure):
    _fields_ = [("cache_bytes", ctypes.c_int64), ("ways", ctypes.c_int32), ("indexes", ctypes.c_int32),
                ("policy", ctypes.c_int32), ("warm_start", ctypes.c_int32), ("seed", ctypes.c_uint64),
                ("pool", ctypes.c_void_p), ("pool_bytes", ctypes.c_int64),
                ("miss_mode", ctypes.c_int32), ("host_threads", ctypes.c_int32)]


class CacheGeometry(ctypes.Structure):
    _fields_ = [("slots_S", ctypes.c_int64), ("slot_bytes", ctypes.c_int64), ("pool_bytes", ctypes.c_int64),
                ("ways_M", ctypes.c_int32), ("indexes_N_raw", ctypes.c_int32),
                ("covered_layers", ctypes.c_int32), ("reserved", ctypes.c_int32)]


STAT_FIELDS = ("accesses", "at_least_one_hit", "all_k_hit", "expert_hits", "expert_misses",
               "coverage_misses", "evictions", "fetches", "fetch_bytes", "hit_under_fill", "host_computed")
MISS_FETCH, MISS_HOST_COMPUTE, MISS_PULL = 0, 1, 2


class LayerStats(ctypes.Structure):
    _fields_ = [(f, ctypes.c_uint64) for f in STAT_FIELDS]


class RuntimeInfo(ctypes.Structure):
    _fields_ = [("expert_path", ctypes.c_int32), ("pdl", ctypes.c_int32), ("ring_stages", ctypes.c_int32),
                ("stage_bytes", ctypes.c_int32), ("grid", ctypes.c_int32), ("tp_reduce", ctypes.c_int32),
                ("reserved", ctypes.c_int32 * 2)]


class TpExchange(ctypes.Structure):
    _fields_ = [("dev_ptr", ctypes.c_void_p), ("bytes", ctypes.c_int64), ("ipc_handle", ctypes.c_uint8 * 64)]


class Profile(ctypes.Structure):
    _fields_ = [("ms", ctypes.c_double * 4), ("launches", ctypes.c_uint64 * 4)]


# numpy view of moe_access_record (20 bytes, C layout)
RECORD_DTYPE = np.dtype({"names": ["token", "layer", "rank", "hit", "expert", "evicted", "way",
                                   "coverage", "reserved", "weight"],
                         "formats": [np.uint32, np.uint16, np.uint8, np.uint8, np.int16, np.int16,
                                     np.int8, np.uint8, np.uint16, np.float32],
                         "offsets": [0, 4, 6, 7, 8, 10, 12, 13, 14, 16], "itemsize": 20})


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    if not os.path.exists(path):
        raise ImportError(f"libmoe.so not built at {path}: run `python -c 'import __graft_entry__ as g; g.build()'`"
                          " (there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    p, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    lib.moe_init.argtypes = [ctypes.POINTER(ModelDesc), ctypes.POINTER(Weights), ctypes.POINTER(p)]
    lib.moe_destroy.argtypes = [p]
    lib.cache_configure.argtypes = [p, ctypes.POINTER(CacheConfig), ctypes.POINTER(CacheGeometry)]
    lib.moe_layer_forward.argtypes = [p, i32, p, p, p]
    lib.moe_layer_forward_host.argtypes = [p, i32, p, p]
    lib.cache_stats.argtypes = [p, i32, ctypes.POINTER(LayerStats)]
    lib.cache_trace.argtypes = [p, p, i64, ctypes.POINTER(i64)]
    lib.moe_profile_enable.argtypes = [p, i32]
    lib.moe_profile_read.argtypes = [p, ctypes.POINTER(Profile)]
    lib.moe_nccl_unique_id.argtypes = [p]
    lib.moe_get_runtime_info.argtypes = [p, ctypes.POINTER(RuntimeInfo)]
    lib.moe_host_alloc.argtypes = [i64, ctypes.POINTER(p)]
    lib.moe_host_free.argtypes = [p]
    lib.moe_host_expert_ffn.argtypes = [p, p, i32, i32, p, i32]
    lib.moe_layer_prefill.argtypes = [p, i32, p, p, i32, p]
    lib.moe_tp_exchange_buffer.argtypes = [p, ctypes.POINTER(TpExchange)]
    lib.moe_tp_connect_ipc.argtypes = [p, p]
    lib.moe_tp_connect_local.argtypes = [p, i32]
    lib.moe_tp_disconnect.argtypes = [p]
    lib.moe_last_error.restype = ctypes.c_char_p
    lib.moe_abi_version.restype = i32
    for name in EXPORTS:
        if name not in ("moe_last_error", "moe_abi_version"):
            getattr(lib, name).restype = i32
    return lib
