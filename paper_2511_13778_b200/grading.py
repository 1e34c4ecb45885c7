"""Device grading harness: mirror of ozadp's grading API on the GPU.

Reference: /root/reference/proj/include/ozadp/grading.hpp and
proj/src/grading.cpp (gen_test2 :13-47, default_test2_b :49-54,
gen_uniform_rect :56-63, error_report :67-90, grade_uniform_point :92-134,
grade_a_check :158-181, csv_header/to_csv :183-222, run_test2_sweep :246-275,
run_uniform_grade :277-307).

Same names, argument meaning and error behaviour (ValueError for the
reference's std::invalid_argument). What changes: the inputs are generated on
the GPU (bitwise the reference's matrices), every GEMM runs through
libadpb200.so, and the reference's exact_gemm (a CPU superaccumulator) is
replaced by the device double-double oracle (adpb200_dd_gemm), which is
accurate to 2^-53 |AB| + gamma_2k^2 (|A||B|) -- far below every error this
harness measures. The Test-2 diagonal x^T x is computed exactly (integer
arithmetic) and rounded once, like exact_dot(...).rounded.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import adp as _adp
from ._lib import check, lib
from .adp import AdpConfig, AdpMode, Handle, _device, _ptr, _stream, parse_mode

__all__ = [
    "Test2Instance", "gen_test2", "default_test2_b", "gen_uniform_rect", "gen_uniform", "ErrorReport",
    "error_report", "dd_gemm", "exact_dot_x", "GradePoint", "grade_uniform_point", "GradeReport", "grade_a_check",
    "SweepRow", "csv_header", "to_csv", "run_test2_sweep", "UniformGradeResult", "run_uniform_grade",
    "Xoshiro256pp",
]


class Xoshiro256pp:
    """rng.hpp:11-54 (host side: seed derivation only; matrices are drawn on the GPU)."""

    M = (1 << 64) - 1

    def __init__(self, seed: int):
        x = seed & self.M
        self.s = []
        for _ in range(4):
            x = (x + 0x9E3779B97F4A7C15) & self.M
            z = x
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & self.M
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & self.M
            self.s.append(z ^ (z >> 31))

    @staticmethod
    def _rotl(v, k):
        return ((v << k) | (v >> (64 - k))) & Xoshiro256pp.M

    def __call__(self) -> int:
        s = self.s
        r = (self._rotl((s[0] + s[3]) & self.M, 23) + s[0]) & self.M
        t = (s[1] << 17) & self.M
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = self._rotl(s[3], 45)
        return r


def _handle(device: Optional[int]) -> Handle:
    return Handle.default(_device(device).index)


def gen_uniform_rect(rows: int, cols: int, seed: int, lo: float = 0.0, hi: float = 1.0,
                     device: Optional[int] = None) -> torch.Tensor:
    """gen_uniform_rect (grading.cpp:56-63), drawn on the GPU: row-major CUDA float64."""
    dev = _device(device)
    out = torch.empty((rows, cols), dtype=torch.float64, device=dev)
    check(lib().adpb200_gen_uniform_rect(_handle(dev.index).h, rows, cols, C.c_uint64(seed & ((1 << 64) - 1)),
                                         float(lo), float(hi), _ptr(out), _stream(dev)))
    return out


def gen_uniform(n: int, seed: int, lo: float = 0.0, hi: float = 1.0, device: Optional[int] = None) -> torch.Tensor:
    return gen_uniform_rect(n, n, seed, lo, hi, device)


@dataclass
class Test2Instance:
    """grading.hpp:17-27."""

    n: int
    b: int
    delta: float
    seed: int
    x: np.ndarray
    j: np.ndarray
    lhs: torch.Tensor
    rhs: torch.Tensor


def gen_test2(n: int, b: int, seed: int, device: Optional[int] = None) -> Test2Instance:
    """gen_test2 (grading.cpp:13-47): lhs(k, i) = x_s 2^j_s, rhs(i, k) = x_s 2^-j_s, s = (i-k) mod n."""
    if n < 2:
        raise ValueError("gen_test2: n must be at least 2")
    if b < 0:
        raise ValueError("gen_test2: b must be nonnegative")
    if b > 1022:
        raise ValueError("gen_test2: b too large, entries would leave the FP64 range")
    dev = _device(device)
    lhs = torch.empty((n, n), dtype=torch.float64, device=dev)
    rhs = torch.empty((n, n), dtype=torch.float64, device=dev)
    x = np.empty(n, dtype=np.float64)
    j = np.empty(n, dtype=np.int32)
    check(lib().adpb200_gen_test2(_handle(dev.index).h, n, int(b), C.c_uint64(seed & ((1 << 64) - 1)), _ptr(lhs),
                                  _ptr(rhs), C.c_void_p(x.ctypes.data), C.c_void_p(j.ctypes.data), _stream(dev)))
    return Test2Instance(n, b, (2.0 * b) / float(n - 1), seed, x, j, lhs, rhs)


def default_test2_b(n: int) -> int:
    """default_test2_b (grading.cpp:49-54)."""
    if n < 2:
        raise ValueError("default_test2_b: n must be at least 2")
    return 511 - (n - 1).bit_length() - 1


def exact_dot_x(x: np.ndarray) -> float:
    """exact_dot(x, x).rounded for x in [1, 2): each square is an exact 106-bit
    integer times 2^-104; the integer sum is exact and Python's int / int
    division rounds it once to nearest-even."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.size and not (np.all(x >= 1.0) and np.all(x < 2.0)):
        raise ValueError("exact_dot_x: entries must lie in [1, 2)")
    mant = (x * 2.0 ** 52).astype(np.int64)
    s = sum(int(v) * int(v) for v in mant)
    return s / (1 << 104)


@dataclass
class ErrorReport:
    """grading.hpp:53-58 (+ the grading ratio against (|A||B|)_ij)."""

    max_err: float = 0.0
    avg_err: float = 0.0
    counted: int = 0
    skipped: int = 0
    max_ratio: float = 0.0
    avg_ratio: float = 0.0


def error_report(c: torch.Tensor, c_ref: torch.Tensor, exact_diag: Optional[float] = None,
                 absab: Optional[torch.Tensor] = None) -> ErrorReport:
    """error_report (grading.cpp:67-90) on the GPU: componentwise relative
    errors against c_ref (the diagonal against exact_diag when given); with
    absab, also max/avg of |c - c_ref| / (2^-52 (|A||B|)_ij)."""
    if tuple(c.shape) != tuple(c_ref.shape):
        raise ValueError("error_report: shape mismatch")
    dev = c.device
    rows, cols = c.shape
    out = torch.zeros(7, dtype=torch.float64, device=dev)
    check(lib().adpb200_error_report(_handle(dev.index).h, rows, cols, _ptr(c.contiguous()), _ptr(c_ref.contiguous()),
                                     _ptr(absab), float(exact_diag) if exact_diag is not None else 0.0,
                                     1 if exact_diag is not None else 0, _ptr(out), _stream(dev)))
    v = out.cpu().tolist()
    return ErrorReport(v[0], v[1], int(v[2]), int(v[3]), v[4], v[5])


def dd_gemm(a: torch.Tensor, b: torch.Tensor, want_absab: bool = True):
    """Device double-double oracle: (RN(AB) to ~2^-106, (|A||B|) or None)."""
    (m, k), (k2, n) = a.shape, b.shape
    if k != k2:
        raise ValueError("dd_gemm: inner dimensions differ")
    dev = a.device
    ref = torch.empty((m, n), dtype=torch.float64, device=dev)
    ab = torch.empty((m, n), dtype=torch.float64, device=dev) if want_absab else None
    check(lib().adpb200_dd_gemm(_handle(dev.index).h, m, n, k, _ptr(a.contiguous()), _ptr(b.contiguous()), _ptr(ref),
                                _ptr(ab), _stream(dev)))
    return ref, ab


@dataclass
class GradePoint:
    """grading.hpp:64-74."""

    n: int = 0
    seed: int = 0
    emu_max_ratio: float = 0.0
    emu_avg_ratio: float = 0.0
    nat_max_ratio: float = 0.0
    nat_avg_ratio: float = 0.0
    esc_bits: int = -1
    slices: int = 0
    fallback: bool = False


def grade_uniform_point(n: int, seed: int, config: Optional[AdpConfig] = None,
                        device: Optional[int] = None) -> GradePoint:
    """grade_uniform_point (grading.cpp:92-134): uniform(0,1) operands from two
    seeds drawn off xoshiro(seed); ratios |C - AB| / (2^-52 AB) (entries are
    positive, so (|A||B|)_ij = (AB)_ij) of the dispatched and the native run."""
    if n < 1:
        raise ValueError("grade_uniform_point: n must be positive")
    config = config or AdpConfig()
    root = Xoshiro256pp(seed)
    seed_a, seed_b = root(), root()
    a = gen_uniform(n, seed_a, device=device)
    b = gen_uniform(n, seed_b, device=device)
    exact, _ = dd_gemm(a, b, want_absab=False)
    emu, trace = _adp.adp_gemm(a, b, 1.0, 0.0, None, config)
    nat = _adp.native_gemm(a, b)
    re = error_report(emu, exact, absab=exact)
    rn = error_report(nat, exact, absab=exact)
    p = GradePoint(n=n, seed=seed)
    p.fallback = trace.path == "native_fallback"
    p.slices = trace.slices if trace.path == "emulated" else 0
    p.esc_bits = trace.esc_bits if trace.esc_bits is not None else -1
    p.emu_max_ratio, p.emu_avg_ratio = re.max_ratio, re.avg_ratio
    p.nat_max_ratio, p.nat_avg_ratio = rn.max_ratio, rn.avg_ratio
    return p


@dataclass
class GradeReport:
    """grading.hpp:81-89."""

    c_calibrated: float = 0.0
    slope_max: float = 0.0
    slope_avg: float = 0.0
    native_slope_avg: float = 0.0
    eq1_pass: bool = False
    slope_pass: bool = False
    grade_a_pass: bool = False


def _loglog_slope(points: Sequence[GradePoint], attr: str) -> float:
    # grading.cpp:140-156: least squares of log2(max(y, 2^-20)) on log2(n)
    xs = [math.log2(float(p.n)) for p in points]
    ys = [math.log2(max(getattr(p, attr), 2.0 ** -20)) for p in points]
    mx, my = sum(xs) / len(xs), sum(ys) / len(ys)
    num = sum((x - mx) * (y - my) for x, y in zip(xs, ys))
    den = sum((x - mx) * (x - mx) for x in xs)
    if not den > 0:
        raise ValueError("grade_a_check: sizes must not all coincide")
    return num / den


def grade_a_check(points: Sequence[GradePoint]) -> GradeReport:
    """grade_a_check (grading.cpp:158-181)."""
    if len(points) < 4:
        raise ValueError("grade_a_check: need at least 4 sweep sizes")
    n_min = min(p.n for p in points)
    n_max = max(p.n for p in points)
    if n_max < 8 * n_min:
        raise ValueError("grade_a_check: sizes must span at least 8x")
    rep = GradeReport()
    rep.c_calibrated = max(p.nat_max_ratio / float(p.n) for p in points)
    rep.eq1_pass = all(not (p.emu_max_ratio > rep.c_calibrated * float(p.n)) for p in points)
    rep.slope_max = _loglog_slope(points, "emu_max_ratio")
    rep.slope_avg = _loglog_slope(points, "emu_avg_ratio")
    rep.native_slope_avg = _loglog_slope(points, "nat_avg_ratio")
    rep.slope_pass = rep.slope_max <= 1.15
    rep.grade_a_pass = rep.eq1_pass and rep.slope_pass
    return rep


@dataclass
class SweepRow:
    """grading.hpp:94-106."""

    test: str = ""
    n: int = 0
    b: Optional[int] = None
    mode: str = ""
    target_bits: int = 53
    esc_bits: Optional[int] = None
    slices: int = 0
    fallback: bool = False
    max_err: float = 0.0
    avg_err: float = 0.0
    seed: int = 0


def csv_header() -> str:
    return "test,n,b,mode,target_bits,esc_bits,slices,fallback,max_err,avg_err,seed"


def _num(v: float) -> str:
    """std::to_chars(double) (grading.cpp:186-191): shortest round-trip digits,
    fixed or scientific notation, whichever is shorter (fixed on a tie)."""
    v = float(v)
    if v != v:
        return "nan" if math.copysign(1.0, v) > 0 else "-nan"
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    sign = "-" if math.copysign(1.0, v) < 0 else ""
    v = abs(v)
    if v == 0.0:
        return sign + "0"
    r = repr(v)
    mant, _, exp = r.partition("e")
    e10 = int(exp) if exp else 0
    ip, _, fp = mant.partition(".")
    if fp == "0":
        fp = ""
    digits = (ip + fp).lstrip("0")
    # value = 0.digits... -> position of the decimal point relative to digits[0]
    point = len(ip) + e10 if ip != "0" else e10 - (len(fp) - len(fp.lstrip("0")))
    digits = digits.rstrip("0") or "0"
    sci_exp = point - 1
    sci = digits[0] + ("." + digits[1:] if len(digits) > 1 else "") + \
        "e" + ("-" if sci_exp < 0 else "+") + f"{abs(sci_exp):02d}"
    if point <= 0:
        fixed = "0." + "0" * (-point) + digits
    elif point >= len(digits):
        # an integer: the fixed form prints its exact digits (123456789012345683968,
        # not the shortest digits padded with zeros), like printf("%f")
        fixed = str(int(v))
    else:
        fixed = digits[:point] + "." + digits[point:]
    return sign + (fixed if len(fixed) <= len(sci) else sci)


def to_csv(row: SweepRow) -> str:
    """to_csv (grading.cpp:195-222)."""
    return ",".join([
        row.test, str(row.n), "" if row.b is None else str(row.b), row.mode, str(row.target_bits),
        "" if row.esc_bits is None else str(row.esc_bits), str(row.slices), "1" if row.fallback else "0",
        _num(row.max_err), _num(row.avg_err), str(row.seed),
    ])


def _mode_label(config: AdpConfig) -> str:
    if config.mode == AdpMode.ForceNative:
        return "native"
    if config.mode == AdpMode.ForceEmulate:
        return f"emulate:{config.forced_slices}"
    return "auto"


def _row_from_trace(trace, config: AdpConfig) -> SweepRow:
    row = SweepRow(mode=_mode_label(config), target_bits=config.target_bits)
    row.esc_bits = trace.esc_bits
    row.slices = trace.slices if trace.path == "emulated" else 0
    row.fallback = trace.path == "native_fallback"
    return row


def run_test2_sweep(n: int, b_list: Sequence[int], modes: Sequence[str], seed: int,
                    base: Optional[AdpConfig] = None, device: Optional[int] = None) -> List[SweepRow]:
    """run_test2_sweep (grading.cpp:246-275): per b one instance, the reference
    product = native_gemm (reference order), the diagonal against exact x^T x."""
    base = base or AdpConfig()
    base.validate()
    rows: List[SweepRow] = []
    for b in b_list:
        inst = gen_test2(n, b, seed, device)
        xtx = exact_dot_x(inst.x)
        ref = _adp.native_gemm(inst.lhs, inst.rhs)
        for mode in modes:
            cfg = AdpConfig(**{f: getattr(base, f) for f in base.__dataclass_fields__})
            if not parse_mode(mode, cfg):
                raise ValueError("run_test2_sweep: unknown mode: " + mode)
            c, trace = _adp.adp_gemm(inst.lhs, inst.rhs, 1.0, 0.0, None, cfg)
            rep = error_report(c, ref, xtx)
            row = _row_from_trace(trace, cfg)
            row.test, row.n, row.b = "test2", n, b
            row.max_err, row.avg_err, row.seed = rep.max_err, rep.avg_err, seed
            rows.append(row)
    return rows


@dataclass
class UniformGradeResult:
    points: List[GradePoint] = field(default_factory=list)
    rows: List[SweepRow] = field(default_factory=list)
    report: GradeReport = field(default_factory=GradeReport)


def run_uniform_grade(n_list: Sequence[int], seed: int, base: Optional[AdpConfig] = None,
                      device: Optional[int] = None) -> UniformGradeResult:
    """run_uniform_grade (grading.cpp:277-307)."""
    base = base or AdpConfig()
    base.validate()
    if not n_list:
        raise ValueError("run_uniform_grade: empty size list")
    res = UniformGradeResult()
    root = Xoshiro256pp(seed)
    for n in n_list:
        ps = root()
        p = grade_uniform_point(n, ps, base, device)
        emu = SweepRow(test="uniform", n=n, mode=_mode_label(base), target_bits=base.target_bits,
                       esc_bits=p.esc_bits if p.esc_bits >= 0 else None, slices=p.slices, fallback=p.fallback,
                       max_err=p.emu_max_ratio, avg_err=p.emu_avg_ratio, seed=ps)
        nat = SweepRow(test="uniform", n=n, mode="native", target_bits=base.target_bits, max_err=p.nat_max_ratio,
                       avg_err=p.nat_avg_ratio, seed=ps)
        res.rows += [emu, nat]
        res.points.append(p)
    res.report = grade_a_check(res.points)
    return res
