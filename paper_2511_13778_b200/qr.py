"""The reference's application caller on the GPU: blocked Householder QR with
ADP trailing updates (mirror of ozadp/qr.hpp; proj/src/qr.cpp).

    QrResult, geqrf_blocked, materialize_q, upper_r, QrAccuracy, qr_residual,
    histogram_csv

Same names, argument meaning and error behaviour (ValueError for the
reference's std::invalid_argument). Everything runs in libadpb200.so on the
device (adpb200_geqrf_blocked / _qr_materialize_q / _qr_residual): the panel
factorisation in the reference's operation order and the three trailing-update
products per panel through the ADP GEMM, so with the default AdpConfig the
factors, T blocks and traces are bitwise the reference's.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np
import torch

from . import _lib
from ._lib import check, lib
from .adp import AdpConfig, AdpTrace, Handle, _device, _ptr, _stream, _to_dev

__all__ = ["QrResult", "geqrf_blocked", "materialize_q", "upper_r", "QrAccuracy", "qr_residual", "histogram_csv"]


@dataclass
class QrResult:
    """qr.hpp:16-21: factors (R above the diagonal, reflector tails below),
    one T per panel, three traces per panel (call order), the panel width."""

    factors: torch.Tensor
    t_blocks: List[torch.Tensor] = field(default_factory=list)
    traces: List[AdpTrace] = field(default_factory=list)
    panel: int = 0
    _t_packed: Optional[torch.Tensor] = None

    def t_packed(self) -> torch.Tensor:
        return self._t_packed


def geqrf_blocked(a, panel: int, gemm_config: Optional[AdpConfig] = None, handle: Optional[Handle] = None) -> QrResult:
    """geqrf_blocked (qr.cpp:98-143). `a` is a row-major m x n matrix (numpy or
    CUDA float64 tensor, not modified); the factors come back as a CUDA tensor."""
    gemm_config = gemm_config or AdpConfig()
    dev = _device(a.device.index if isinstance(a, torch.Tensor) else None)
    handle = handle or Handle.default(dev.index)
    m, n = tuple(a.shape)
    f = _to_dev(a, dev).clone()
    ok = 1 <= panel <= 1024 and n >= 1   # otherwise the C ABI raises the reference's contract error
    panels = (n + panel - 1) // panel if ok else 0
    t = torch.zeros(max(1, panels * panel * panel), dtype=torch.float64, device=dev)
    tr = torch.zeros(max(1, 3 * panels) * _lib.TRACE_BYTES, dtype=torch.uint8, device=dev)
    o = gemm_config.to_c()
    check(lib().adpb200_geqrf_blocked(handle.h, m, n, panel, _ptr(f), _ptr(t), _ptr(tr), C.byref(o), _stream(dev)))
    raw = tr.cpu().numpy().tobytes()
    traces = [AdpTrace.from_c(_lib.Trace.from_buffer_copy(raw[i * _lib.TRACE_BYTES:(i + 1) * _lib.TRACE_BYTES]))
              for i in range(3 * panels)]
    blocks = []
    for p in range(panels):
        pw = min(panel, n - p * panel)
        blocks.append(t[p * panel * panel: p * panel * panel + pw * pw].view(pw, pw))
    return QrResult(f, blocks, traces, panel, t)


def materialize_q(qr: QrResult, handle: Optional[Handle] = None) -> torch.Tensor:
    """Thin Q (m x n), accumulated natively from the WY blocks (qr.cpp:145-173)."""
    f = qr.factors
    m, n = f.shape
    handle = handle or Handle.default(f.device.index)
    q = torch.empty((m, n), dtype=torch.float64, device=f.device)
    check(lib().adpb200_qr_materialize_q(handle.h, m, n, qr.panel, _ptr(f), _ptr(qr.t_packed()), _ptr(q),
                                         _stream(f.device)))
    return q


def upper_r(qr: QrResult) -> torch.Tensor:
    """The n x n upper triangle of the factors (qr.cpp:175-181)."""
    n = qr.factors.shape[1]
    return torch.triu(qr.factors[:n, :n])


@dataclass
class QrAccuracy:
    residual: float = 0.0
    orthogonality: float = 0.0


def qr_residual(a0, qr: QrResult, handle: Optional[Handle] = None) -> QrAccuracy:
    """|A0 - QR|_F / |A0|_F and |I - Q^T Q|_F via the native GEMM (qr.cpp:183-197)."""
    f = qr.factors
    m, n = f.shape
    if tuple(a0.shape) != (m, n):
        raise ValueError("qr_residual: shape mismatch")
    handle = handle or Handle.default(f.device.index)
    A0 = _to_dev(a0, f.device)
    out = torch.zeros(2, dtype=torch.float64, device=f.device)
    check(lib().adpb200_qr_residual(handle.h, m, n, qr.panel, _ptr(A0), _ptr(f), _ptr(qr.t_packed()), _ptr(out),
                                    _stream(f.device)))
    r, o = out.cpu().tolist()
    return QrAccuracy(r, o)


def histogram_csv(traces: List[AdpTrace]) -> str:
    """histogram_csv (qr.cpp:199-217)."""
    by = {}
    fallbacks = 0
    for t in traces:
        if t.path == "emulated":
            by[t.slices] = by.get(t.slices, 0) + 1
        else:
            fallbacks += 1
    out = "slices,count\n"
    for s in sorted(by):
        out += f"{s},{by[s]}\n"
    return out + f"native_fallback,{fallbacks}\n"
