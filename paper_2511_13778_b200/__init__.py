"""paper_2511_13778_b200 — B200-native (sm_100a) ADP emulated DGEMM.

A from-scratch implementation of the Automatic Dynamic Precision emulated
DGEMM of arXiv 2511.13778 (reference: ozadp::adp_gemm). All arithmetic runs
in the CUDA kernels of libadpb200.so (C ABI: include/adpb200.h); this Python
package mirrors the reference's host interface on top of it.
"""
from ._lib import LIB_PATH, PAIRS_FULL, PAIRS_TARGET, TRACE_BYTES, lib  # noqa: F401
from .adp import (  # noqa: F401
    AdpConfig,
    AdpMode,
    AdpTrace,
    GraphedDgemm,
    Handle,
    adp_gemm,
    block_exponent_stats,
    decide,
    decompose,
    dgemm,
    dgemm_host,
    emulated_gemm,
    esc_coarsened,
    esc_exact,
    native_gemm,
    parse_mode,
    recompose,
    required_slices,
    scan_matrix,
    slice_pair_mm,
)

__version__ = "0.1.0"
