"""ctypes binding of the engine's C-ABI (include/plnmf_gpu.h).

Loads ``libplnmf_gpu.so`` from this package directory and fails loudly when it
is missing — there is no CPU fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libplnmf_gpu.so"

i32, i64, u64, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double
P_i64, P_f64, P_u32 = C.POINTER(C.c_int64), C.POINTER(C.c_double), C.POINTER(C.c_uint32)


class Config(C.Structure):
    """plnmf_config — mirrors SolverConfig (proj/include/plnmf/config.hpp:11-22)."""
    _fields_ = [("rank", i64), ("epsilon", f64), ("max_iters", i64), ("rel_tol", f64),
                ("seed", u64), ("error_every", i64), ("deterministic", i32), ("tile_size", i64)]


class PhaseTimesC(C.Structure):
    _fields_ = [(n, f64) for n in ("precompute_h", "update_h", "precompute_w", "update_w",
                                   "phase1", "phase2", "phase3", "normalize", "error_eval")]


class TraceRecordC(C.Structure):
    _fields_ = [("iteration", i64), ("rel_error", f64), ("elapsed_s", f64), ("phases", PhaseTimesC)]


class TraceC(C.Structure):
    _fields_ = [("initial_error", f64), ("total_seconds", f64), ("update_macs", u64),
                ("totals", PhaseTimesC), ("n_records", i64), ("capacity", i64),
                ("records", C.POINTER(TraceRecordC))]


class StatsC(C.Structure):
    _fields_ = [("kernel_launches", u64), ("persistent_ctas", i32), ("sm_count", i32),
                ("device_bytes", i64), ("w_plan", i32), ("h_plan", i32)]


Engine_p = C.c_void_p
P_cfg = C.POINTER(Config)

# name: (restype, argtypes) — every symbol declared in include/plnmf_gpu.h
SIGNATURES = {
    "plnmf_last_error": (C.c_char_p, []),
    "plnmf_gpu_abi_version": (i32, []),
    "plnmf_config_default": (None, [P_cfg]),
    "plnmf_config_validate": (C.c_int, [P_cfg]),
    "plnmf_plan_tiles": (C.c_int, [i64, i64, P_i64, P_i64, P_i64]),
    "plnmf_init_factors": (C.c_int, [i64, i64, P_cfg, P_f64, P_f64]),
    "plnmf_synth_csr": (C.c_int, [i64, i64, f64, u64, P_i64, P_i64, P_f64, P_i64]),
    "plnmf_mm_read": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "plnmf_mm_read_string": (C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]),
    "plnmf_mm_info": (C.c_int, [C.c_void_p, P_i64, P_i64, P_i64, C.POINTER(C.c_int32)]),
    "plnmf_mm_free": (C.c_int, [C.c_void_p]),
    "plnmf_gpu_create_mm": (C.c_int, [i32, C.c_void_p, i64, C.POINTER(Engine_p)]),
    "plnmf_gpu_create_synthetic": (C.c_int, [i32, i64, i64, f64, u64, i64, C.POINTER(Engine_p)]),
    "plnmf_gpu_get_csr": (C.c_int, [Engine_p, P_i64, P_i64, P_f64]),
    "plnmf_gpu_get_csr_rows": (C.c_int, [Engine_p, i32, P_i64, i64, P_i64, P_i64, P_f64]),
    "plnmf_gpu_get_rows": (C.c_int, [Engine_p, C.c_int, P_i64, i64, P_f64]),
    "plnmf_gpu_device_count": (i32, []),
    "plnmf_gpu_device_name": (C.c_int, [i32, C.c_char_p, i32]),
    "plnmf_gpu_create_csr": (C.c_int, [i32, i64, i64, i64, P_i64, P_i64, P_f64, i64, C.POINTER(Engine_p)]),
    "plnmf_gpu_create_dense": (C.c_int, [i32, i64, i64, P_f64, i64, C.POINTER(Engine_p)]),
    "plnmf_gpu_destroy": (C.c_int, [Engine_p]),
    "plnmf_gpu_input_info": (C.c_int, [Engine_p, P_i64, P_i64, P_i64, P_f64]),
    "plnmf_gpu_set_math": (C.c_int, [Engine_p, C.c_int]),
    "plnmf_gpu_set_reference_threads": (C.c_int, [Engine_p, i32]),
    "plnmf_gpu_force_streaming": (C.c_int, [Engine_p, i32]),
    "plnmf_gpu_force_spmm_blocks": (C.c_int, [Engine_p, i64]),
    "plnmf_gpu_set_factors": (C.c_int, [Engine_p, P_f64, P_f64]),
    "plnmf_gpu_get_factors": (C.c_int, [Engine_p, P_f64, P_f64]),
    "plnmf_gpu_init_factors": (C.c_int, [Engine_p, P_cfg]),
    "plnmf_gpu_iterate": (C.c_int, [Engine_p, P_cfg, C.c_int, C.POINTER(TraceC)]),
    "plnmf_gpu_iterate_host": (C.c_int, [Engine_p, P_cfg, C.c_int, P_f64, P_f64, C.POINTER(TraceC)]),
    "plnmf_gpu_precompute_h_products": (C.c_int, [Engine_p]),
    "plnmf_gpu_precompute_w_products": (C.c_int, [Engine_p]),
    "plnmf_gpu_update_h": (C.c_int, [Engine_p, P_cfg, C.c_int]),
    "plnmf_gpu_update_w": (C.c_int, [Engine_p, P_cfg, C.c_int]),
    "plnmf_gpu_evaluate_error": (C.c_int, [Engine_p, P_f64]),
    "plnmf_gpu_relative_error_direct": (C.c_int, [Engine_p, P_f64]),
    "plnmf_gpu_get_product": (C.c_int, [Engine_p, C.c_int, P_f64]),
    "plnmf_gpu_set_product": (C.c_int, [Engine_p, C.c_int, P_f64]),
    "plnmf_gpu_create_shard": (C.c_int, [i32, i32, i32, i64, i64, i64, P_i64, P_i64, P_f64, i64, P_i64, P_i64,
                                         P_f64, f64, i64, C.POINTER(Engine_p)]),
    "plnmf_gpu_create_shard_synthetic": (C.c_int, [i32, i32, i32, i64, i64, f64, u64, i64, C.POINTER(Engine_p)]),
    "plnmf_gpu_shard_info": (C.c_int, [Engine_p, C.POINTER(i32), C.POINTER(i32), P_i64, P_i64, P_i64, P_i64]),
    "plnmf_gpu_shard_norm_sq": (C.c_int, [Engine_p, f64, P_f64]),
    "plnmf_gpu_shard_set_norm_sq": (C.c_int, [Engine_p, f64]),
    "plnmf_gpu_shard_ipc_handle": (C.c_int, [Engine_p, C.c_void_p]),
    "plnmf_gpu_shard_connect": (C.c_int, [Engine_p, C.c_void_p]),
    "plnmf_gpu_shard_connect_local": (C.c_int, [C.POINTER(Engine_p), i32]),
    "plnmf_gpu_shard_set_timeout": (C.c_int, [Engine_p, f64]),
    "plnmf_gpu_run_iterations": (C.c_int, [Engine_p, P_cfg, C.c_int, i64, P_f64]),
    "plnmf_gpu_phase_ms": (C.c_int, [Engine_p, P_f64]),
    "plnmf_gpu_time_kernel": (C.c_int, [Engine_p, P_cfg, i32, i32, P_f64]),
    "plnmf_gpu_best_integer_tile": (C.c_int, [Engine_p, P_cfg, C.POINTER(C.c_int32), i32, C.POINTER(C.c_int32),
                                              P_f64]),
    "plnmf_gpu_get_stats": (C.c_int, [Engine_p, C.POINTER(StatsC)]),
    "plnmf_gpu_synchronize": (C.c_int, [Engine_p]),
}

_lib = None


def lib() -> C.CDLL:
    """The loaded C-ABI library (raises if the extension has not been built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -m paper_1904_07935_b200.build). The engine has no CPU fallback.")
        handle = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib
