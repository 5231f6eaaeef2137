"""ctypes binding of the C-ABI in include/ntc_b200.h (libntcb.so).

This is the same binding a maintainer would add to call the CUDA path from
Python.  There is no fallback: if libntcb.so is missing
or no CUDA device is present, loading fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libntcb.so")

u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)
f64p = C.POINTER(C.c_double)
f32p = C.POINTER(C.c_float)

NTCB_OK, NTCB_EINVAL, NTCB_ERUNTIME, NTCB_ERANGE, NTCB_EDOMAIN, NTCB_ECUDA = range(6)


class InvalidArgument(ValueError):
    """std::invalid_argument"""


class NtcRuntimeError(RuntimeError):
    """std::runtime_error"""


class OutOfRange(IndexError):
    """std::out_of_range"""


class DomainError(ArithmeticError):
    """std::domain_error"""


class CudaError(RuntimeError):
    """CUDA / device failure."""


_EXC = {NTCB_EINVAL: InvalidArgument, NTCB_ERUNTIME: NtcRuntimeError, NTCB_ERANGE: OutOfRange,
        NTCB_EDOMAIN: DomainError, NTCB_ECUDA: CudaError}


class NmcConfigC(C.Structure):
    _fields_ = [("lambda_", C.c_double), ("c", C.c_double), ("max_inner", C.c_int32),
                ("power_iters", C.c_int32), ("power_tol", C.c_double), ("threads", C.c_int32),
                ("chunk", C.c_int32)]


class AoConfigC(C.Structure):
    _fields_ = [("rank", C.c_uint64), ("lambda_", C.c_double), ("c", C.c_double),
                ("max_inner", C.c_int32), ("power_iters", C.c_int32), ("max_epochs", C.c_double),
                ("term_tol", C.c_double), ("seed", C.c_uint64), ("threads", C.c_int32),
                ("chunk", C.c_int32), ("power_tol", C.c_double), ("eval_metrics", C.c_int32),
                ("metrics_every", C.c_int32)]


class MetricsRecordC(C.Structure):
    _fields_ = [("epoch", C.c_double), ("objective", C.c_double), ("rel_error", C.c_double),
                ("wall_seconds", C.c_double), ("entries_accessed", C.c_uint64)]


class TuningC(C.Structure):
    _fields_ = [("no_tc", C.c_int32), ("no_nat", C.c_int32), ("tc_p", C.c_int32),
                ("update_wpc", C.c_int32), ("short_row", C.c_int64),
                ("side_sampler_ctas", C.c_int32), ("heavy_per", C.c_int32),
                ("heavy_win_log2", C.c_int32), ("heavy_big_log2", C.c_int32),
                ("host_threads", C.c_int32), ("update_ctas_per_sm", C.c_int32), ("update_carveout", C.c_int32), ("graph", C.c_int32), ("peer_fence", C.c_int32),
                ("nat_pad", C.c_int32), ("tiny_sampler", C.c_int32), ("item_order", C.c_int32)]


OBSERVER = C.CFUNCTYPE(None, C.POINTER(MetricsRecordC), C.c_void_p, C.c_void_p)

# name -> (restype, argtypes); every symbol declared in include/ntc_b200.h
SIGNATURES = {
    "ntcb_last_error": (C.c_char_p, []),
    "ntcb_version": (C.c_int, []),
    "ntcb_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "ntcb_destroy": (C.c_int, [C.c_void_p]),
    "ntcb_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "ntcb_synchronize": (C.c_int, [C.c_void_p]),
    "ntcb_host_alloc": (C.c_int, [C.c_uint64, C.POINTER(C.c_void_p)]),
    "ntcb_host_free": (C.c_int, [C.c_void_p]),
    "ntcb_tuning_defaults": (None, [C.POINTER(TuningC)]),
    "ntcb_set_tuning": (C.c_int, [C.c_void_p, C.POINTER(TuningC)]),
    "ntcb_get_tuning": (C.c_int, [C.c_void_p, C.POINTER(TuningC)]),
    "ntcb_rng_fork": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "ntcb_sweep_stream_state": (C.c_uint64, [C.c_uint64, C.c_uint64, C.c_int]),
    "ntcb_tensor_load": (C.c_int, [C.c_void_p, C.c_int, u64p, C.c_uint64, u32p, f64p]),
    "ntcb_tensor_load_f32": (C.c_int, [C.c_void_p, C.c_int, u64p, C.c_uint64, u32p, f32p]),
    "ntcb_tensor_load_device": (C.c_int, [C.c_void_p, C.c_int, u64p, C.c_uint64, C.c_void_p,
                                          C.c_void_p]),
    "ntcb_tensor_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), u64p, u64p]),
    "ntcb_view_export": (C.c_int, [C.c_void_p, C.c_int, u64p, u32p, f32p]),
    "ntcb_view_export_rows": (C.c_int, [C.c_void_p, C.c_int, C.c_uint64, C.c_uint64, u64p, u32p,
                                        f32p]),
    "ntcb_tensor_export": (C.c_int, [C.c_void_p, u32p, f32p]),
    "ntcb_view_keep_rows": (C.c_int, [C.c_void_p, C.c_int, C.c_uint64, C.c_uint64]),
    "ntcb_view_resident": (C.c_int, [C.c_void_p, C.c_int, u64p, u64p, u64p]),
    "ntcb_tns_parse": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), u64p, u64p, C.POINTER(u32p),
                                 C.POINTER(f64p)]),
    "ntcb_tns_last_error": (C.c_char_p, []),
    "ntcb_free": (None, [C.c_void_p]),
    "ntcb_tns_write": (C.c_int, [C.c_char_p, C.c_int, u64p, C.c_uint64, u32p, f64p]),
    "ntcb_tensor_read_tns": (C.c_int, [C.c_void_p, C.c_char_p]),
    "ntcb_factors_init": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(f64p), C.POINTER(f64p)]),
    "ntcb_factors_random": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64]),
    "ntcb_factor_set": (C.c_int, [C.c_void_p, C.c_int, f64p, f64p]),
    "ntcb_factor_get": (C.c_int, [C.c_void_p, C.c_int, f64p, f64p]),
    "ntcb_factor_device_ptr": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p),
                                         u64p]),
    "ntcb_factor_ipc_handle": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "ntcb_ipc_open": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
    "ntcb_factor_set_peers": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "ntcb_s_nmc": (C.c_int, [C.c_void_p, C.c_int, f64p, C.POINTER(NmcConfigC), C.c_uint64, u64p]),
    "ntcb_sample_prefetch": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(NmcConfigC), C.c_uint64]),
    "ntcb_s_nmc_host": (C.c_int, [C.c_void_p, C.c_int, f64p, f64p, f64p, C.POINTER(NmcConfigC),
                                  C.c_uint64, u64p]),
    "ntcb_s_nmc_rows_async": (C.c_int, [C.c_void_p, C.c_int, C.c_uint64, C.c_uint64,
                                        C.POINTER(NmcConfigC), C.c_uint64]),
    "ntcb_collect": (C.c_int, [C.c_void_p, u64p]),
    "ntcb_segment_length": (C.c_int, [C.c_void_p, C.c_int, u64p]),
    "ntcb_s_nmc_chunks_async": (C.c_int, [C.c_void_p, C.c_int, C.c_uint64, C.c_uint32, C.c_uint32,
                                          C.POINTER(NmcConfigC), C.c_uint64, C.c_void_p]),
    "ntcb_finalize_row_async": (C.c_int, [C.c_void_p, C.c_int, C.c_uint64, C.c_void_p, C.c_uint32,
                                          C.POINTER(NmcConfigC)]),
    "ntcb_sample_rows": (C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_uint64, C.c_uint64,
                                   C.c_uint64, C.c_uint64, u64p, u32p]),
    "ntcb_sample_mask": (C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_uint64, C.c_uint64,
                                   C.c_uint64, C.c_uint64, u32p]),
    "ntcb_sample_row": (C.c_int, [C.c_void_p, C.c_int, C.c_uint64, C.c_double, C.c_uint64, u32p,
                                  u64p]),
    "ntcb_sweep_async": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(NmcConfigC), C.c_uint64]),
    "ntcb_ao_ntc": (C.c_int, [C.c_void_p, C.POINTER(AoConfigC), C.POINTER(MetricsRecordC),
                              C.c_uint64, u64p, OBSERVER, C.c_void_p]),
    "ntcb_metrics": (C.c_int, [C.c_void_p, f64p, f64p, f64p]),
    "ntcb_objective": (C.c_int, [C.c_void_p, C.c_double, f64p]),
    "ntcb_relative_error": (C.c_int, [C.c_void_p, f64p]),
    "ntcb_rmse": (C.c_int, [C.c_void_p, f64p]),
    "ntcb_synth_uniform": (C.c_int, [C.c_void_p, C.c_int, u64p, C.c_uint64, C.c_uint64, C.c_double,
                                     C.c_uint64]),
    "ntcb_synth": (C.c_int, [C.c_void_p, C.c_int, u64p, C.c_uint64, C.c_uint64, C.c_double,
                             C.c_uint64, f64p, C.c_int]),
    "ntcb_render_model": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint8)]),
    "ntcb_profile_enable": (C.c_int, [C.c_void_p, C.c_int]),
    "ntcb_profile_read": (C.c_int, [C.c_void_p, f64p, f64p, u64p, u64p]),
    "ntcb_profile_read_kernel": (C.c_int, [C.c_void_p, f64p, u64p]),
}

_L = None


def load(path: str = LIB_PATH):
    """Load libntcb.so (build it first with paper_2109_09534_b200.build)."""
    global _L
    if _L is not None:
        return _L
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run `python -m paper_2109_09534_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _L = L
    return L


def check(rc: int) -> None:
    if rc != NTCB_OK:
        msg = _L.ntcb_last_error().decode()
        raise _EXC.get(rc, CudaError)(msg)
