"""Row-block partition of one large DGEMM across the GPUs of a node.

One process per GPU (torch.distributed, NCCL over NVLink). Rank r owns the
rows rows_of(r) of op(A) and C and a full copy of op(B). The only exchange
on the data path is the ADP decision input: a max-allreduce of
{exceptional, esc_bits} (two int32) between the guardrail phase and the
compute phase of adpb200_dgemm_rows, so every rank decides identically and
uses the same slice count — C is bit-identical to the single-GPU result.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Tuple

import torch
import torch.distributed as dist

from . import _lib
from ._lib import check, lib
from .adp import AdpConfig, Handle, _ptr, _stream


def rows_of(rank: int, world: int, m: int, align: int = 128) -> Tuple[int, int]:
    """[start, stop) of rank's row block: contiguous, multiples of `align`
    rows (the GEMM's M tile) except possibly the last, as even as possible."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    tiles = (m + align - 1) // align
    base, extra = divmod(tiles, world)
    t0 = rank * base + min(rank, extra)
    t1 = t0 + base + (1 if rank < extra else 0)
    return min(m, t0 * align), min(m, t1 * align)


def reduce_xchg(xchg: torch.Tensor, group=None) -> None:
    """Max-reduce the guardrail exchange block over the ranks (in place)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(xchg, op=dist.ReduceOp.MAX, group=group)


def dgemm_rows(transa: str, transb: str, m_global: int, m: int, n: int, k: int, alpha: float, A: torch.Tensor,
               lda: int, B: torch.Tensor, ldb: int, beta: float, C_: torch.Tensor, ldc: int,
               config: Optional[AdpConfig] = None, handle: Optional[Handle] = None, group=None,
               trace: Optional[torch.Tensor] = None, xchg: Optional[torch.Tensor] = None) -> None:
    """This rank's share of a row-partitioned ADP DGEMM (column-major storage
    of the local block: C_ is m x n with leading dimension ldc). Stream
    ordered end to end; the allreduce runs on NCCL's stream, ordered against
    the current stream by torch."""
    config = config or AdpConfig()
    dev = C_.device
    handle = handle or Handle.default(dev.index)
    if xchg is None:
        xchg = torch.zeros(2, dtype=torch.int32, device=dev)
    o = config.to_c()
    args = (m_global, transa.encode()[:1], transb.encode()[:1], m, n, k, float(alpha), _ptr(A), lda, _ptr(B), ldb,
            float(beta), _ptr(C_), ldc, C.byref(o), None if trace is None else C.c_void_p(trace.data_ptr()),
            C.c_void_p(xchg.data_ptr()), _stream(dev))
    check(lib().adpb200_dgemm_rows(handle.h, 1, *args))
    reduce_xchg(xchg, group)
    check(lib().adpb200_dgemm_rows(handle.h, 2, *args))
