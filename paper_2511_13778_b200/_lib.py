"""ctypes binding of the adpb200 C ABI (include/adpb200.h).

Loads the in-tree libadpb200.so and fails loudly when it is missing: there is
no CPU or library fallback behind this package.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# ADPB200_LIB: an alternative build of the same library (tuning experiments only)
LIB_PATH = os.environ.get("ADPB200_LIB") or os.path.join(PKG, "libadpb200.so")

OK, ERR_RUNTIME, ERR_CONTRACT = 0, 2, 3
MODE_AUTO, MODE_EMULATE, MODE_NATIVE = 0, 1, 2
PATH_EMULATED, PATH_NATIVE = 0, 1
PAIRS_FULL, PAIRS_TARGET = -1, -2
REASONS = ("ok", "forced", "exceptional_values", "esc_too_large", "too_small", "cost_model")
PATHS = ("emulated", "native_fallback")


class Options(C.Structure):
    _fields_ = [
        ("target_bits", C.c_int32),
        ("max_slices", C.c_int32),
        ("esc_block_len", C.c_int64),
        ("min_dim", C.c_int64),
        ("mode", C.c_int32),
        ("forced_slices", C.c_int32),
        ("cost_ratio", C.c_double),
        ("chunk_len", C.c_int64),
        ("pair_limit", C.c_int32),
        ("guardrails_forced", C.c_int32),
        ("fallback", C.c_int32),
        ("esc_method", C.c_int32),
        ("rounding", C.c_int32),
        ("reserved", C.c_int32 * 3),
    ]


class Trace(C.Structure):
    _fields_ = [
        ("path", C.c_int32),
        ("reason", C.c_int32),
        ("esc_bits", C.c_int32),
        ("slices", C.c_int32),
        ("pair_limit", C.c_int32),
        ("pairs", C.c_int32),
        ("modeled_cost_ratio", C.c_double),
        ("nan_a", C.c_uint64),
        ("inf_a", C.c_uint64),
        ("negzero_a", C.c_uint64),
        ("nan_b", C.c_uint64),
        ("inf_b", C.c_uint64),
        ("negzero_b", C.c_uint64),
        ("m", C.c_int64),
        ("n", C.c_int64),
        ("k", C.c_int64),
        ("gemm_variant", C.c_int32),
        ("k_chunks", C.c_int32),
        ("rounding_deferred", C.c_int32),
        ("reserved_t", C.c_int32),
    ]


TRACE_BYTES = C.sizeof(Trace)

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2511_13778_b200.build` "
            "(there is no fallback implementation)"
        )
    L = C.CDLL(LIB_PATH)
    i64, i32, f64, vp = C.c_int64, C.c_int32, C.c_double, C.c_void_p
    popt = C.POINTER(Options)
    sig = {
        "adpb200_version": (C.c_char_p, []),
        "adpb200_last_error": (C.c_char_p, []),
        "adpb200_status_string": (C.c_char_p, [C.c_int]),
        "adpb200_default_options": (None, [popt]),
        "adpb200_validate_options": (C.c_int, [popt]),
        "adpb200_create": (C.c_int, [C.POINTER(vp), C.c_int]),
        "adpb200_destroy": (C.c_int, [vp]),
        "adpb200_launch_count": (C.c_uint64, [vp]),
        "adpb200_workspace_bytes": (C.c_uint64, [vp]),
        "adpb200_decide_host": (C.c_int, [C.c_int, C.c_int, i64, i64, i64, C.c_int, popt, C.POINTER(i32),
                                          C.POINTER(f64)]),
        "adpb200_dgemm": (C.c_int, [vp, C.c_char, C.c_char, i64, i64, i64, f64, vp, i64, vp, i64, f64, vp, i64,
                                    popt, vp, vp]),
        "adpb200_adp_gemm": (C.c_int, [vp, i64, i64, i64, f64, vp, vp, f64, vp, vp, popt, vp, vp]),
        "adpb200_dgemm_host": (C.c_int, [vp, C.c_char, C.c_char, i64, i64, i64, f64, vp, i64, vp, i64, f64, vp, i64,
                                         popt, vp, vp]),
        "adpb200_adp_gemm_host": (C.c_int, [vp, i64, i64, i64, f64, vp, vp, f64, vp, vp, popt, vp, vp]),
        "adpb200_dgemm_rows": (C.c_int, [vp, C.c_int, i64, C.c_char, C.c_char, i64, i64, i64, f64, vp, i64, vp,
                                         i64, f64, vp, i64, popt, vp, vp, vp]),
        "adpb200_scan": (C.c_int, [vp, vp, i64, vp, vp]),
        "adpb200_block_stats": (C.c_int, [vp, vp, i64, i64, C.c_int, i64, vp, vp, vp, vp, vp]),
        "adpb200_esc_coarsened": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, i64, i64, i64, C.c_int, vp, vp]),
        "adpb200_decompose": (C.c_int, [vp, vp, i64, i64, C.c_int, C.c_int, vp, vp, vp]),
        "adpb200_slice_pair_mm": (C.c_int, [vp, vp, vp, i64, i64, i64, C.c_int, C.c_int, vp, vp]),
        "adpb200_emulated_gemm": (C.c_int, [vp, vp, vp, i64, i64, i64, f64, f64, vp, vp, C.c_int, C.c_int, vp]),
        "adpb200_recompose": (C.c_int, [vp, vp, i64, i64, C.c_int, vp, vp, f64, f64, vp, vp, vp]),
        "adpb200_esc_exact": (C.c_int, [vp, vp, vp, i64, i64, i64, C.c_int, vp, vp, vp]),
        "adpb200_native_gemm": (C.c_int, [vp, vp, vp, i64, i64, i64, f64, f64, vp, vp, vp]),
        "adpb200_dist_sizes": (C.c_int, [i64, i64, C.c_int, popt, C.POINTER(i64)]),
        "adpb200_dist_decision": (C.c_int, [popt, C.POINTER(i32), i64, i64, i64, C.POINTER(i32)]),
        "adpb200_dgemm_dist": (C.c_int, [vp, C.c_int, i64, C.c_int, C.c_int, C.c_char, i64, i64, i64, f64, vp, i64,
                                         vp, f64, vp, i64, popt, vp, vp, vp, vp, vp, vp, C.c_int, vp]),
        "adpb200_ipc_alloc": (C.c_int, [C.c_int, i64, C.POINTER(vp), C.POINTER(C.c_uint8)]),
        "adpb200_ipc_open": (C.c_int, [C.c_int, C.POINTER(C.c_uint8), C.POINTER(vp)]),
        "adpb200_ipc_close": (C.c_int, [vp]),
        "adpb200_ipc_free": (C.c_int, [vp]),
        "adpb200_copy_async": (C.c_int, [vp, vp, i64, vp]),
        "adpb200_dist_flag_offset": (i64, [i64, C.c_int]),
        "adpb200_stream_wait_geq": (C.c_int, [vp, C.c_uint32, vp]),
        "adpb200_stream_write_flag": (C.c_int, [vp, C.c_uint32, vp]),
        "adpb200_geqrf_blocked": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, popt, vp]),
        "adpb200_qr_materialize_q": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, vp]),
        "adpb200_qr_residual": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, vp, vp]),
        "adpb200_dd_gemm": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, vp, vp]),
        "adpb200_error_report": (C.c_int, [vp, i64, i64, vp, vp, vp, f64, C.c_int, vp, vp]),
        "adpb200_gen_uniform_rect": (C.c_int, [vp, i64, i64, C.c_uint64, f64, f64, vp, vp]),
        "adpb200_gen_test2": (C.c_int, [vp, i64, C.c_int, C.c_uint64, vp, vp, vp, vp, vp]),
        "adpb200_profile_enable": (C.c_int, [vp, C.c_int]),
        "adpb200_profile_read": (C.c_int, [vp, C.POINTER(C.c_float), C.POINTER(C.c_int)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


EXPORTED = (
    "adpb200_version", "adpb200_last_error", "adpb200_status_string", "adpb200_default_options",
    "adpb200_validate_options", "adpb200_create", "adpb200_destroy", "adpb200_launch_count", "adpb200_workspace_bytes",
    "adpb200_decide_host", "adpb200_dgemm", "adpb200_adp_gemm", "adpb200_dgemm_rows", "adpb200_dgemm_host",
    "adpb200_adp_gemm_host", "adpb200_scan", "adpb200_block_stats",
    "adpb200_esc_coarsened", "adpb200_decompose", "adpb200_slice_pair_mm", "adpb200_emulated_gemm",
    "adpb200_native_gemm", "adpb200_profile_enable", "adpb200_profile_read", "adpb200_recompose", "adpb200_esc_exact",
    "adpb200_dist_sizes", "adpb200_dist_decision", "adpb200_dgemm_dist", "adpb200_ipc_alloc",
    "adpb200_ipc_open", "adpb200_ipc_close", "adpb200_ipc_free", "adpb200_copy_async",
    "adpb200_dist_flag_offset", "adpb200_stream_wait_geq", "adpb200_stream_write_flag",
    "adpb200_geqrf_blocked", "adpb200_qr_materialize_q", "adpb200_qr_residual",
    "adpb200_dd_gemm", "adpb200_error_report", "adpb200_gen_uniform_rect", "adpb200_gen_test2",
)
PROFILE_STAGES = ("stats", "esc", "decide", "slice", "gemm", "native")


class AdpError(RuntimeError):
    pass


def check(rc: int) -> None:
    """Map C-ABI status codes onto the reference's exception classes."""
    if rc == OK:
        return
    msg = lib().adpb200_last_error().decode()
    if rc == ERR_CONTRACT:
        raise ValueError(msg)  # std::invalid_argument in the reference
    raise AdpError(msg or f"adpb200 error {rc}")


def default_options() -> Options:
    o = Options()
    lib().adpb200_default_options(C.byref(o))
    return o
