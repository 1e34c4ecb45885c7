"""Host-side mirror of the reference's ADP GEMM interface over the adpb200 C ABI.

Names, argument meaning and error behaviour follow ozadp
(/root/reference/proj/include/ozadp/adp.hpp:16-87, igemm.hpp, slicing.hpp,
fpbits.hpp, esc.hpp, oracle.hpp):

    AdpConfig, AdpMode, AdpTrace, parse_mode, decide, adp_gemm,
    emulated_gemm, slice_pair_mm, decompose, block_exponent_stats,
    scan_matrix, esc_coarsened, native_gemm, required_slices

Matrices are row-major like ozadp::MatrixF64. Inputs may be numpy arrays
(copied to the GPU and the result copied back, like the reference's
value-returning API) or CUDA torch tensors (everything stays on the device).
std::invalid_argument maps to ValueError. PyTorch is used only for device
memory and streams; every byte of arithmetic runs in libadpb200.so.
"""
from __future__ import annotations

import ctypes as C
import enum
import json
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np
import torch

from . import _lib
from ._lib import PAIRS_FULL, PAIRS_TARGET, check, lib

__all__ = [
    "AdpMode", "AdpConfig", "AdpTrace", "Handle", "parse_mode", "decide", "adp_gemm", "dgemm", "dgemm_host",
    "emulated_gemm", "slice_pair_mm", "decompose", "block_exponent_stats", "scan_matrix", "esc_coarsened",
    "native_gemm", "required_slices", "PAIRS_FULL", "PAIRS_TARGET",
]


class AdpMode(enum.IntEnum):
    Auto = 0
    ForceEmulate = 1
    ForceNative = 2


ESC_METHODS = {"coarsened": 0, "certified": 1}
ROUNDING_MODES = {"auto": 0, "fused": 1, "deferred": 2}
FALLBACKS = {"reference": 0, "fast": 1}


@dataclass
class AdpConfig:
    """ozadp::AdpConfig (adp.hpp:18-33) + the B200 extensions."""

    target_bits: int = 53
    esc_block_len: int = 256
    max_slices: int = 18
    min_dim: int = 256
    mode: AdpMode = AdpMode.Auto
    forced_slices: int = 7
    cost_ratio: float = 512.0
    chunk_len: int = 65536
    pair_limit: int = PAIRS_FULL      # PAIRS_FULL (reference), PAIRS_TARGET (d_a+d_b <= s) or a limit
    guardrails_forced: bool = False   # ForceEmulate still runs scan + ESC + decide
    # "coarsened" (the reference's esc_coarsened) or "certified": the coarsened ESC
    # lowered to the s0 bound when an INT8 indicator GEMM certifies it (adpb200.h)
    esc_method: str = "coarsened"
    # where the NB = 64 GEMM rounds: "auto", "fused" (in its epilogue) or "deferred"
    # (a separate pass over parked folded words); bitwise the same C
    rounding: str = "auto"
    # native fallback flavour: "reference" (bitwise native_gemm) or "fast" (DMMA)
    fallback: str = "reference"

    def to_c(self) -> _lib.Options:
        o = _lib.default_options()
        o.target_bits = int(self.target_bits)
        o.esc_block_len = int(self.esc_block_len)
        o.max_slices = int(self.max_slices)
        o.min_dim = int(self.min_dim)
        o.mode = int(self.mode)
        o.forced_slices = int(self.forced_slices)
        o.cost_ratio = float(self.cost_ratio)
        o.chunk_len = int(self.chunk_len)
        o.pair_limit = int(self.pair_limit)
        o.guardrails_forced = 1 if self.guardrails_forced else 0
        o.esc_method = ESC_METHODS.get(self.esc_method, -1)
        o.rounding = ROUNDING_MODES.get(self.rounding, -1)
        o.fallback = FALLBACKS.get(self.fallback, -1)
        return o

    def validate(self) -> None:
        """AdpConfig::validate (adp.cpp:15-28): raises ValueError."""
        o = self.to_c()
        check(lib().adpb200_validate_options(C.byref(o)))


@dataclass
class AdpTrace:
    """ozadp::AdpTrace (adp.hpp:57-67) plus what the B200 pipeline did."""

    path: str = "native_fallback"
    reason: str = "ok"
    esc_bits: Optional[int] = None
    slices: Optional[int] = None
    m: int = 0
    n: int = 0
    k: int = 0
    scan_a: Tuple[int, int, int] = (0, 0, 0)  # nan, inf, -0
    scan_b: Tuple[int, int, int] = (0, 0, 0)
    modeled_cost_ratio: float = 0.0
    pair_limit: Optional[int] = None
    pairs: int = 0
    gemm_variant: int = 0
    k_chunks: int = 0
    rounding_deferred: bool = False

    @staticmethod
    def from_c(t: _lib.Trace) -> "AdpTrace":
        return AdpTrace(
            path=_lib.PATHS[t.path], reason=_lib.REASONS[t.reason],
            esc_bits=None if t.esc_bits < 0 else int(t.esc_bits),
            slices=None if t.slices < 0 else int(t.slices),
            m=int(t.m), n=int(t.n), k=int(t.k),
            scan_a=(int(t.nan_a), int(t.inf_a), int(t.negzero_a)),
            scan_b=(int(t.nan_b), int(t.inf_b), int(t.negzero_b)),
            modeled_cost_ratio=float(t.modeled_cost_ratio),
            pair_limit=None if t.pair_limit < 0 else int(t.pair_limit), pairs=int(t.pairs),
            gemm_variant=int(t.gemm_variant), k_chunks=int(t.k_chunks),
            rounding_deferred=bool(t.rounding_deferred),
        )

    @property
    def has_exceptional_a(self) -> bool:
        return self.scan_a[0] + self.scan_a[1] > 0

    @property
    def has_exceptional_b(self) -> bool:
        return self.scan_b[0] + self.scan_b[1] > 0

    def to_json(self) -> str:
        """Same stable keys as AdpTrace::to_json (adp.cpp:98-114)."""
        return json.dumps({"path": self.path, "reason": self.reason, "esc_bits": self.esc_bits,
                           "slices": self.slices if self.path == "emulated" else None,
                           "m": self.m, "n": self.n, "k": self.k}, separators=(",", ":"))


def parse_mode(text: str, config: AdpConfig) -> bool:
    """parse_mode (adp.cpp:116-137): 'auto' | 'native' | 'emulate:S'."""
    if text == "auto":
        config.mode = AdpMode.Auto
        return True
    if text == "native":
        config.mode = AdpMode.ForceNative
        return True
    prefix = "emulate:"
    if len(text) > len(prefix) and text.startswith(prefix):
        tail = text[len(prefix):]
        if not (tail.isascii() and tail.isdigit()):
            return False
        s = int(tail)
        if s < 1 or s > 32:
            return False
        config.mode = AdpMode.ForceEmulate
        config.forced_slices = s
        return True
    return False


def required_slices(target_bits: int, esc_bits: int) -> int:
    """esc.cpp:8-12."""
    if target_bits < 1:
        raise ValueError("required_slices: target_bits must be positive")
    if esc_bits < 0:
        raise ValueError("required_slices: esc_bits must be nonnegative")
    return (target_bits + esc_bits + 2 + 7) // 8


def decide(exc_a: bool, exc_b: bool, m: int, n: int, k: int, esc_bits: int, config: AdpConfig):
    """decide() (adp.cpp:46-96) run by the library's host copy of the device
    decision function. Returns (path, reason, slices, provider_called, esc_bits,
    modeled_cost_ratio)."""
    o = config.to_c()
    out = (C.c_int32 * 5)()
    cost = C.c_double(0.0)
    check(lib().adpb200_decide_host(int(exc_a), int(exc_b), m, n, k, esc_bits, C.byref(o), out, C.byref(cost)))
    return (_lib.PATHS[out[0]], _lib.REASONS[out[1]], int(out[2]), int(out[3]),
            None if out[4] < 0 else int(out[4]), cost.value)


class Handle:
    """Owns an adpb200 handle (device workspace) on one GPU."""

    _default = {}

    def __init__(self, device: int = 0):
        self.device = device
        h = C.c_void_p()
        check(lib().adpb200_create(C.byref(h), device))
        self.h = h

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().adpb200_destroy(self.h)
        except Exception:
            pass

    @classmethod
    def default(cls, device: int = 0) -> "Handle":
        if device not in cls._default:
            cls._default[device] = Handle(device)
        return cls._default[device]

    def launches(self) -> int:
        return int(lib().adpb200_launch_count(self.h))

    def workspace_bytes(self) -> int:
        return int(lib().adpb200_workspace_bytes(self.h))

    def profile_enable(self, max_calls: int) -> None:
        """Record CUDA events around each pipeline stage of the next calls."""
        check(lib().adpb200_profile_enable(self.h, int(max_calls)))

    def profile_read(self):
        """List (one dict per recorded call) of stage -> milliseconds."""
        cap = 4096
        buf = (C.c_float * (cap * len(_lib.PROFILE_STAGES)))()
        n = C.c_int(0)
        check(lib().adpb200_profile_read(self.h, buf, C.byref(n)))
        ns = len(_lib.PROFILE_STAGES)
        return [{s: float(buf[c * ns + i]) for i, s in enumerate(_lib.PROFILE_STAGES)} for c in range(n.value)]


# ---------------------------------------------------------------------------------
def _device(dev: Optional[int]) -> torch.device:
    return torch.device("cuda", torch.cuda.current_device() if dev is None else dev)


def _to_dev(x, device: torch.device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        if x.dtype != torch.float64:
            raise ValueError("expected float64 data")
        return x.to(device).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(device)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None or t.numel() == 0 else C.c_void_p(t.data_ptr())


def _stream(device) -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _shape2(x) -> Tuple[int, int]:
    s = tuple(x.shape)
    if len(s) != 2:
        raise ValueError("expected a 2-D matrix")
    return s


def adp_gemm(a, b, alpha: float = 1.0, beta: float = 0.0, c=None, config: Optional[AdpConfig] = None,
             handle: Optional[Handle] = None, out: Optional[torch.Tensor] = None):
    """ozadp::adp_gemm (adp.hpp:84-87): returns (alpha*a@b + beta*c, AdpTrace).

    numpy in -> numpy out (one synchronisation to copy the result back, like
    the reference's value return); CUDA tensors in -> CUDA tensor out, and the
    trace is read back only when the caller inspects it."""
    config = config or AdpConfig()
    host = not isinstance(a, torch.Tensor)
    (m, k), (k2, n) = _shape2(a), _shape2(b)
    if k != k2:
        raise ValueError("adp_gemm: inner dimensions differ")
    if beta != 0.0 and c is None:
        raise ValueError("adp_gemm: beta != 0 requires C")
    if c is not None and _shape2(c) != (m, n):
        raise ValueError("adp_gemm: C shape mismatch")
    dev = _device(a.device.index if isinstance(a, torch.Tensor) else None)
    handle = handle or Handle.default(dev.index)
    if host and out is None:
        # host in, host out: the library copies in, overlaps the copy-out with the GEMM
        A = np.ascontiguousarray(a, dtype=np.float64)
        B = np.ascontiguousarray(b, dtype=np.float64)
        Cin = np.ascontiguousarray(c, dtype=np.float64) if c is not None else None
        res = np.empty((m, n), dtype=np.float64)
        tr = _lib.Trace()
        o = config.to_c()
        p = lambda x: None if x is None or x.size == 0 else C.c_void_p(x.ctypes.data)  # noqa: E731
        check(lib().adpb200_adp_gemm_host(handle.h, m, n, k, float(alpha), p(A), p(B), float(beta), p(Cin), p(res),
                                          C.byref(o), C.byref(tr), _stream(dev)))
        return res, AdpTrace.from_c(tr)
    A, B = _to_dev(a, dev), _to_dev(b, dev)
    Cin = _to_dev(c, dev) if c is not None else None
    if out is None:
        out = torch.empty((m, n), dtype=torch.float64, device=dev)
    tr = torch.zeros(_lib.TRACE_BYTES, dtype=torch.uint8, device=dev)
    o = config.to_c()
    check(lib().adpb200_adp_gemm(handle.h, m, n, k, float(alpha), _ptr(A), _ptr(B), float(beta), _ptr(Cin),
                                 _ptr(out), C.byref(o), C.c_void_p(tr.data_ptr()), _stream(dev)))
    trace = _read_trace(tr)
    if host:
        return out.cpu().numpy(), trace
    return out, trace


def _read_trace(tr: torch.Tensor) -> AdpTrace:
    raw = tr.cpu().numpy().tobytes()
    return AdpTrace.from_c(_lib.Trace.from_buffer_copy(raw))


def dgemm(transa: str, transb: str, m: int, n: int, k: int, alpha: float, A: torch.Tensor, lda: int,
          B: torch.Tensor, ldb: int, beta: float, C_: torch.Tensor, ldc: int, config: Optional[AdpConfig] = None,
          handle: Optional[Handle] = None, trace: Optional[torch.Tensor] = None) -> None:
    """BLAS-style column-major DGEMM on CUDA float64 storage (the north-star
    entry point: trans, m/n/k, alpha, A/lda, B/ldb, beta, C/ldc + ADP options).
    Stream-ordered; never synchronises. `trace` (uint8 CUDA tensor of
    TRACE_BYTES) receives the device-side AdpTrace when given."""
    config = config or AdpConfig()
    dev = C_.device
    handle = handle or Handle.default(dev.index)
    o = config.to_c()
    check(lib().adpb200_dgemm(handle.h, transa.encode()[:1], transb.encode()[:1], m, n, k, float(alpha),
                              _ptr(A), lda, _ptr(B), ldb, float(beta), _ptr(C_), ldc, C.byref(o),
                              None if trace is None else C.c_void_p(trace.data_ptr()), _stream(dev)))


class GraphedDgemm:
    """One dgemm call captured in a CUDA graph: the pipeline is stream-ordered with
    no host synchronisation, so after a warm-up call (it sizes the handle's
    workspace and encodes the TMA descriptors) the whole call records into a graph.
    Each replay re-reads A, B (and C when beta != 0) from the captured buffers and
    re-takes the ADP decision on the device; it removes the per-kernel launch gaps
    that dominate small calls. Arguments as dgemm; the tensors must stay alive."""

    def __init__(self, transa: str, transb: str, m: int, n: int, k: int, alpha: float, A: torch.Tensor, lda: int,
                 B: torch.Tensor, ldb: int, beta: float, C_: torch.Tensor, ldc: int,
                 config: Optional[AdpConfig] = None, handle: Optional[Handle] = None):
        dev = C_.device
        self.handle = handle or Handle(dev.index)
        args = (transa, transb, m, n, k, alpha, A, lda, B, ldb, beta, C_, ldc, config, self.handle)
        self.stream = torch.cuda.Stream(dev)
        self.stream.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(self.stream):
            dgemm(*args)  # warm-up: workspace + descriptors, outside the capture
        self.stream.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            dgemm(*args)

    def __call__(self) -> None:
        """Replay on the current stream (stream-ordered, no synchronisation)."""
        self.graph.replay()


def dgemm_host(transa: str, transb: str, m: int, n: int, k: int, alpha: float, A: torch.Tensor, lda: int,
               B: torch.Tensor, ldb: int, beta: float, C_: torch.Tensor, ldc: int, config: Optional[AdpConfig] = None,
               handle: Optional[Handle] = None, device: int = 0) -> AdpTrace:
    """dgemm on HOST (CPU, ideally pinned) float64 storage: operands copied in,
    C copied out while the slice GEMM still runs; returns when C is on the host."""
    config = config or AdpConfig()
    handle = handle or Handle.default(device)
    o = config.to_c()
    tr = _lib.Trace()
    p = lambda x: C.c_void_p(x.data_ptr()) if x.numel() else None  # noqa: E731
    check(lib().adpb200_dgemm_host(handle.h, transa.encode()[:1], transb.encode()[:1], m, n, k, float(alpha), p(A),
                                   lda, p(B), ldb, float(beta), p(C_), ldc, C.byref(o), C.byref(tr),
                                   _stream(torch.device("cuda", device))))
    return AdpTrace.from_c(tr)


def emulated_gemm(a, b, slices: int = 7, alpha: float = 1.0, beta: float = 0.0, c=None,
                  pair_limit: int = PAIRS_FULL, handle: Optional[Handle] = None):
    """emulated_gemm (igemm.cpp:129-137): decompose -> tcgen05 slice products -> recompose."""
    host = not isinstance(a, torch.Tensor)
    (m, k), (_, n) = _shape2(a), _shape2(b)
    dev = _device(a.device.index if isinstance(a, torch.Tensor) else None)
    handle = handle or Handle.default(dev.index)
    A, B = _to_dev(a, dev), _to_dev(b, dev)
    Cin = _to_dev(c, dev) if c is not None else None
    out = torch.empty((m, n), dtype=torch.float64, device=dev)
    check(lib().adpb200_emulated_gemm(handle.h, _ptr(A), _ptr(B), m, n, k, float(alpha), float(beta), _ptr(Cin),
                                      _ptr(out), slices, pair_limit, _stream(dev)))
    return out.cpu().numpy() if host else out


def slice_pair_mm(a, b, slices: int, pair_limit: int = PAIRS_FULL, handle: Optional[Handle] = None):
    """slice_pair_mm (igemm.cpp:38-97) on the INT8 tensor cores: int64 [m][n][2s-1]."""
    host = not isinstance(a, torch.Tensor)
    (m, k), (_, n) = _shape2(a), _shape2(b)
    dev = _device(a.device.index if isinstance(a, torch.Tensor) else None)
    handle = handle or Handle.default(dev.index)
    A, B = _to_dev(a, dev), _to_dev(b, dev)
    acc = torch.zeros((m, n, 2 * slices - 1), dtype=torch.int64, device=dev)
    check(lib().adpb200_slice_pair_mm(handle.h, _ptr(A), _ptr(B), m, n, k, slices, pair_limit, _ptr(acc),
                                      _stream(dev)))
    return acc.cpu().numpy() if host else acc


def recompose(acc, row_scale, col_scale, alpha: float = 1.0, beta: float = 0.0, c=None,
              handle: Optional[Handle] = None):
    """recompose (igemm.cpp:99-127): FP64 [m][n] from int64 acc[m][n][2s-1] + the decompose scales."""
    host = not isinstance(acc, torch.Tensor)
    m, n, nd = acc.shape
    if nd % 2 == 0:
        raise ValueError("recompose: acc must hold 2s-1 diagonals")
    dev = _device(acc.device.index if isinstance(acc, torch.Tensor) else None)
    handle = handle or Handle.default(dev.index)
    A = torch.as_tensor(acc, dtype=torch.int64).to(dev).contiguous()
    rs = torch.as_tensor(row_scale, dtype=torch.int32).to(dev).contiguous()
    cs = torch.as_tensor(col_scale, dtype=torch.int32).to(dev).contiguous()
    Cin = _to_dev(c, dev) if c is not None else None
    out = torch.empty((m, n), dtype=torch.float64, device=dev)
    check(lib().adpb200_recompose(handle.h, _ptr(A), m, n, (nd + 1) // 2, _ptr(rs), _ptr(cs), float(alpha),
                                  float(beta), _ptr(Cin), _ptr(out), _stream(dev)))
    return out.cpu().numpy() if host else out


def decompose(a, orient: int, slices: int, handle: Optional[Handle] = None):
    """decompose (slicing.cpp:90-136): (digits[s][lines][len] int8, scale_exp[lines])."""
    host = not isinstance(a, torch.Tensor)
    rows, cols = _shape2(a)
    lines, length = (cols, rows) if orient else (rows, cols)
    dev = _device(a.device.index if isinstance(a, torch.Tensor) else None)
    handle = handle or Handle.default(dev.index)
    A = _to_dev(a, dev)
    dig = torch.zeros((slices, lines, length), dtype=torch.int8, device=dev)
    sc = torch.zeros(lines, dtype=torch.int32, device=dev)
    check(lib().adpb200_decompose(handle.h, _ptr(A), rows, cols, orient, slices, _ptr(dig), _ptr(sc), _stream(dev)))
    if host:
        return dig.cpu().numpy(), sc.cpu().numpy()
    return dig, sc


def block_exponent_stats(a, orient: int, block_len: int, handle: Optional[Handle] = None):
    """block_exponent_stats (fpbits.cpp:26-73): (max[lines][blocks], min, line_max, exceptional)."""
    host = not isinstance(a, torch.Tensor)
    rows, cols = _shape2(a)
    lines, length = (cols, rows) if orient else (rows, cols)
    blocks = 0 if length == 0 else (length + block_len - 1) // block_len
    dev = _device(a.device.index if isinstance(a, torch.Tensor) else None)
    handle = handle or Handle.default(dev.index)
    A = _to_dev(a, dev)
    mx = torch.empty((lines, blocks), dtype=torch.int32, device=dev)
    mn = torch.empty((lines, blocks), dtype=torch.int32, device=dev)
    lm = torch.empty(lines, dtype=torch.int32, device=dev)
    exc = torch.zeros(1, dtype=torch.int32, device=dev)
    check(lib().adpb200_block_stats(handle.h, _ptr(A), rows, cols, orient, block_len, _ptr(mx), _ptr(mn), _ptr(lm),
                                    _ptr(exc), _stream(dev)))
    if host:
        return mx.cpu().numpy(), mn.cpu().numpy(), lm.cpu().numpy(), bool(exc.item())
    return mx, mn, lm, exc


def scan_matrix(a, handle: Optional[Handle] = None):
    """scan_matrix (fpbits.cpp:5-24): ((nan, inf, -0), has_exceptional)."""
    dev = _device(a.device.index if isinstance(a, torch.Tensor) else None)
    handle = handle or Handle.default(dev.index)
    A = _to_dev(a, dev)
    cnt = torch.zeros(3, dtype=torch.int64, device=dev)
    check(lib().adpb200_scan(handle.h, _ptr(A), A.numel(), _ptr(cnt), _stream(dev)))
    c = tuple(int(x) for x in cnt.cpu().tolist())
    return c, c[0] + c[1] > 0


def esc_coarsened(a, b, block_len: int = 256, target_bits: int = 53, handle: Optional[Handle] = None):
    """esc_coarsened (esc.cpp:89-117) over device block stats: (esc_bits, window_bits, slices_required)."""
    dev = _device(a.device.index if isinstance(a, torch.Tensor) else None)
    handle = handle or Handle.default(dev.index)
    A, B = _to_dev(a, dev), _to_dev(b, dev)
    amx, amn, al, ea = block_exponent_stats(A, 0, block_len, handle)
    bmx, bmn, bl, eb = block_exponent_stats(B, 1, block_len, handle)
    if int(ea.item()) or int(eb.item()):
        raise ValueError("esc: Inf or NaN input")  # std::domain_error in the reference
    out = torch.zeros(3, dtype=torch.int32, device=dev)
    check(lib().adpb200_esc_coarsened(handle.h, _ptr(amx), _ptr(amn), _ptr(al), _ptr(bmx), _ptr(bmn), _ptr(bl),
                                      amx.shape[0], bmx.shape[0], amx.shape[1], target_bits, _ptr(out),
                                      _stream(dev)))
    return tuple(int(x) for x in out.cpu().tolist())


def esc_exact(a, b, target_bits: int = 53, handle: Optional[Handle] = None):
    """esc_exact (esc.cpp:61-87) on the GPU: (esc_bits, window_bits, slices_required);
    ValueError (the reference's std::domain_error) on Inf/NaN input."""
    (m, k), (k2, n) = _shape2(a), _shape2(b)
    if k != k2:
        raise ValueError("esc_exact: inner dimensions differ")
    dev = _device(a.device.index if isinstance(a, torch.Tensor) else None)
    handle = handle or Handle.default(dev.index)
    A, B = _to_dev(a, dev), _to_dev(b, dev)
    out = torch.zeros(3, dtype=torch.int32, device=dev)
    exc = torch.zeros(1, dtype=torch.int32, device=dev)
    check(lib().adpb200_esc_exact(handle.h, _ptr(A), _ptr(B), m, n, k, target_bits, _ptr(out), _ptr(exc),
                                  _stream(dev)))
    if int(exc.item()):
        raise ValueError("esc: Inf or NaN input")
    return tuple(int(x) for x in out.cpu().tolist())


def native_gemm(a, b, alpha: float = 1.0, beta: float = 0.0, c=None, handle: Optional[Handle] = None):
    """native_gemm (oracle.cpp:7-28) in the reference's summation order."""
    host = not isinstance(a, torch.Tensor)
    (m, k), (_, n) = _shape2(a), _shape2(b)
    if beta != 0.0 and c is None:
        raise ValueError("native_gemm: beta != 0 needs C")
    dev = _device(a.device.index if isinstance(a, torch.Tensor) else None)
    handle = handle or Handle.default(dev.index)
    A, B = _to_dev(a, dev), _to_dev(b, dev)
    Cin = _to_dev(c, dev) if c is not None else None
    out = torch.empty((m, n), dtype=torch.float64, device=dev)
    check(lib().adpb200_native_gemm(handle.h, _ptr(A), _ptr(B), m, n, k, float(alpha), float(beta), _ptr(Cin),
                                    _ptr(out), _stream(dev)))
    return out.cpu().numpy() if host else out
