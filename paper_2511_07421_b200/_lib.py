"""ctypes binding of the C-ABI (include/a3g.h) in liba3g_b200.so.

The product path has no CPU fallback: if the library is missing or no CUDA
device is present, device entry points raise (loudly) instead of computing
anything on the host.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

LIB_PATH = os.environ.get("A3G_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "liba3g_b200.so")

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
i32p = C.POINTER(C.c_int32)
u64p = C.POINTER(C.c_uint64)
f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)
vp = C.c_void_p


# ---------------------------------------------------------------- errors ----
class A3gError(RuntimeError):
    status = -1


class ParameterError(A3gError, ValueError):
    """a3gnn::ParameterError (common.hpp:14)."""
    status = 1


class LookupError_(A3gError, LookupError):
    """a3gnn::LookupError (common.hpp:20)."""
    status = 2


class ConfigError(A3gError):
    """a3gnn::ConfigError (common.hpp:26)."""
    status = 3


class IoError(A3gError, IOError):
    """a3gnn::IoError (common.hpp:37)."""
    status = 4


class CudaError(A3gError):
    status = 5


class NcclError(A3gError):
    status = 6


class OutOfMemory(A3gError, MemoryError):
    status = 7


_BY_STATUS = {c.status: c for c in (ParameterError, LookupError_, ConfigError, IoError, CudaError, NcclError,
                                    OutOfMemory)}


class HostGraph(C.Structure):
    _fields_ = [("num_nodes", C.c_uint64), ("num_edges", C.c_uint64), ("feat_dim", C.c_uint32),
                ("row_offsets", u64p), ("col_indices", u32p), ("features", f32p), ("labels", u32p),
                ("train_mask", u8p), ("test_mask", u8p)]


# name: (restype, argtypes)  -- status-returning calls use C.c_int
_SIGS = {
    "a3g_last_error": (C.c_char_p, []),
    "a3g_version": (C.c_char_p, []),
    "a3g_host_graph_power_law": (C.c_int, [C.c_uint64, C.c_uint32, C.c_double, C.c_uint32, C.c_uint64, C.c_int,
                                           C.POINTER(C.POINTER(HostGraph))]),
    "a3g_host_graph_load": (C.c_int, [C.c_char_p, C.POINTER(C.POINTER(HostGraph))]),
    "a3g_host_graph_save": (C.c_int, [C.POINTER(HostGraph), C.c_char_p]),
    "a3g_host_graph_from_edges": (C.c_int, [C.c_uint64, u32p, u32p, C.c_uint64, C.c_uint32,
                                            C.POINTER(C.POINTER(HostGraph))]),
    "a3g_host_graph_free": (None, [C.POINTER(HostGraph)]),
    "a3g_sampling_seed": (C.c_uint64, [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32]),
    "a3g_plan_epoch_order": (None, [u32p, C.c_uint64, C.c_uint32, C.c_uint64, u32p]),
    "a3g_graph_create": (C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.c_uint32, u64p, u32p, f32p, C.c_int, u32p,
                                   C.POINTER(vp)]),
    "a3g_graph_destroy": (None, [vp]),
    "a3g_graph_synthesize_features": (C.c_int, [vp, C.c_uint32, C.c_int, C.c_uint64]),
    "a3g_graph_synth_patched": (C.c_uint64, [vp]),
    "a3g_store_create": (C.c_int, [vp, f32p, i32p, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]),
    "a3g_store_info": (C.c_int, [vp, u64p, u64p, u64p]),
    "a3g_store_local_ptr": (C.c_int, [vp, C.POINTER(vp)]),
    "a3g_store_set_peer": (C.c_int, [vp, C.c_int, vp]),
    "a3g_store_ipc_handle": (C.c_int, [vp, u8p]),
    "a3g_store_open_peer": (C.c_int, [vp, C.c_int, u8p]),
    "a3g_store_destroy": (None, [vp]),
    "a3g_cache_build": (C.c_int, [vp, C.c_uint64, C.c_uint32, i32p, C.POINTER(vp)]),
    "a3g_cache_from_map": (C.c_int, [vp, i32p, C.c_uint32, C.POINTER(vp)]),
    "a3g_cache_total_cached": (C.c_uint64, [vp]),
    "a3g_cache_hot_order": (C.c_int, [vp, u32p]),
    "a3g_cache_lookup": (C.c_int, [vp, u32p, C.c_uint64, i32p, u64p, u64p, u64p]),
    "a3g_cache_destroy": (None, [vp]),
    "a3g_sampler_create": (C.c_int, [vp, vp, C.c_uint32, u32p, C.c_uint32, C.POINTER(vp)]),
    "a3g_sampler_destroy": (None, [vp]),
    "a3g_sample_khop": (C.c_int, [vp, u32p, C.c_uint32, C.c_int, C.c_double, C.c_int, C.c_uint64, vp]),
    "a3g_batch_sizes": (C.c_int, [vp, u64p, u64p, u64p, u64p]),
    "a3g_batch_copy": (C.c_int, [vp, u32p, C.POINTER(u32p), C.POINTER(u32p)]),
    "a3g_retrieve_features": (C.c_int, [vp, f32p, C.c_int, u64p, u64p, u64p, vp]),
    "a3g_gather_rows": (C.c_int, [vp, vp, u32p, C.c_uint64, f32p, u64p, u64p]),
    "a3g_weighted_reservoir": (C.c_int, [u32p, f64p, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, u32p, u64p]),
    "a3g_uniform_reservoir": (C.c_int, [u32p, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, u32p, u64p]),
    "a3g_init_model": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, f64p, f64p]),
    "a3g_trainer_create": (C.c_int, [vp, vp, C.c_uint32, u32p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_double,
                                     C.c_uint64, C.POINTER(vp)]),
    "a3g_trainer_destroy": (None, [vp]),
    "a3g_trainer_set_weights": (C.c_int, [vp, f64p, f64p]),
    "a3g_trainer_get_weights": (C.c_int, [vp, f64p, f64p]),
    "a3g_trainer_set_comm": (C.c_int, [vp, vp]),
    "a3g_trainer_set_pipeline": (C.c_int, [vp, C.c_int]),
    "a3g_train_step": (C.c_int, [vp, u32p, C.c_uint32, C.c_int, C.c_double, C.c_int, C.c_uint64, C.c_double,
                                 f64p]),
    "a3g_train_steps": (C.c_int, [vp, u32p, C.c_uint32, C.c_uint32, u64p, C.c_double, C.c_int, C.c_int, f64p]),
    "a3g_train_steps_v": (C.c_int, [vp, u32p, u64p, C.c_uint32, u64p, C.c_double, C.c_int, C.c_int, f64p]),
    "a3g_trainer_step_stats": (C.c_int, [vp, u64p, C.c_uint32]),
    "a3g_evaluate_full_graph": (C.c_int, [vp, u8p, f64p]),
    "a3g_trainer_last_grads": (C.c_int, [vp, f64p, f64p]),
    "a3g_trainer_last_forward": (C.c_int, [vp, u64p, f64p, f64p, f64p, f64p]),
    "a3g_trainer_sampler": (vp, [vp, C.c_int]),
    "a3g_trainer_set_tier_accounting": (C.c_int, [vp, C.c_int]),
    "a3g_trainer_tier_rows": (C.c_int, [vp, u64p]),
    "a3g_trainer_profile_step": (C.c_int, [vp, u32p, C.c_uint32, C.c_double, C.c_int, C.c_uint64, f64p]),
    "a3g_trainer_timing": (C.c_int, [vp, f64p, f64p, f64p, u64p]),
    "a3g_trainer_gemm_timing": (C.c_int, [vp, f64p, f64p, u64p]),
    "a3g_batch_model_create": (C.c_int, [C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(vp)]),
    "a3g_batch_model_destroy": (None, [vp]),
    "a3g_batch_model_load": (C.c_int, [vp, C.c_uint64, C.c_uint64, C.c_uint32, u64p, C.POINTER(u32p),
                                       C.POINTER(u32p), f32p, u32p, u64p]),
    "a3g_batch_model_run": (C.c_int, [vp, f64p, f64p, f64p, f64p, f64p]),
    "a3g_batch_model_forward": (C.c_int, [vp, u32p, i32p, u32p, u32p, f64p, f64p, f64p, f64p]),
    "a3g_sgd_step": (C.c_int, [C.c_int, f64p, f64p, C.c_uint64, C.c_uint64, C.c_double]),
    "a3g_mean_gradients": (C.c_int, [C.c_int, C.POINTER(f64p), C.c_uint32, C.c_uint64, f64p]),
    "a3g_comm_unique_id": (C.c_int, [u8p]),
    "a3g_comm_create": (C.c_int, [u8p, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]),
    "a3g_comm_create_host": (C.c_int, [C.c_int, C.c_int, vp, vp, C.POINTER(vp)]),
    "a3g_comm_destroy": (None, [vp]),
}

_lib = None


def lib() -> C.CDLL:
    """Load liba3g_b200.so (raises if it was not built: no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() (the CUDA path is mandatory)")
        L = C.CDLL(LIB_PATH)
        for name, (rt, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = rt
            fn.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS)


def check(status: int) -> None:
    if status != 0:
        msg = lib().a3g_last_error().decode(errors="replace")
        raise _BY_STATUS.get(status, A3gError)(msg)


def ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def cuda_device_count() -> int:
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:  # pragma: no cover
        return 0
