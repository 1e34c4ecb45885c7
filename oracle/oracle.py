"""TEST INFRASTRUCTURE ONLY — numpy front end for the CPU oracle.

Two back ends with the same API:
  * ``Oracle("port")``      -> oracle/liboracle.so, the plain-C restatement
                               (oracle/adp_oracle.c) — always available once
                               built, travels to the GPU box;
  * ``Oracle("reference")`` -> oracle/_ref/libozref*.so, the UNMODIFIED
                               reference sources (/root/reference/proj/src)
                               behind oracle/ref_shim.cpp.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs import this module, and only as the checker or the
timed CPU baseline. The product package never imports it.

Matrices are row-major numpy float64 arrays, like ozadp::MatrixF64
(proj/include/ozadp/matrix.hpp:12-43).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
NEG_SENTINEL = -1000000  # proj/include/ozadp/fpbits.hpp:22
REASONS = ["ok", "forced", "exceptional_values", "esc_too_large", "too_small", "cost_model"]


class OracleError(RuntimeError):
    pass


def _cpu_has_avx2() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            return " avx2 " in f.read()
    except OSError:
        return False


def build() -> None:
    """Build liboracle.so (+ _ref when /root/reference is present)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


def _load(kind: str) -> C.CDLL:
    if kind == "port":
        path = os.path.join(HERE, "liboracle.so")
    elif kind == "reference":
        v3 = os.path.join(HERE, "_ref", "libozref_v3.so")
        path = v3 if (_cpu_has_avx2() and os.path.exists(v3)) else os.path.join(HERE, "_ref", "libozref.so")
    else:
        raise ValueError(kind)
    if not os.path.exists(path):
        raise OracleError(f"oracle library missing: {path} (run `make -C oracle`)")
    return C.CDLL(path)


def available(kind: str) -> bool:
    try:
        _load(kind)
        return True
    except OracleError:
        return False


def _p(a: np.ndarray, ct=C.c_double):
    return a.ctypes.data_as(C.POINTER(ct))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class Config:
    """Mirror of ozadp::AdpConfig (proj/include/ozadp/adp.hpp:18-33)."""

    target_bits: int = 53
    esc_block_len: int = 256
    max_slices: int = 18
    min_dim: int = 256
    mode: int = 0  # 0 auto, 1 emulate, 2 native
    forced_slices: int = 7
    cost_ratio: float = 512.0
    chunk_len: int = 65536

    def ints(self):
        return (C.c_longlong * 7)(self.target_bits, self.esc_block_len, self.max_slices,
                                  self.min_dim, self.mode, self.forced_slices, self.chunk_len)


class _OzConfig(C.Structure):
    _fields_ = [("target_bits", C.c_int), ("esc_block_len", C.c_int64), ("max_slices", C.c_int),
                ("min_dim", C.c_int64), ("mode", C.c_int), ("forced_slices", C.c_int),
                ("cost_ratio", C.c_double), ("chunk_len", C.c_int64)]


class Oracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        self.lib = _load(kind)
        self.pre = "oz_" if kind == "port" else "ozref_"

    def _fn(self, name):
        return getattr(self.lib, self.pre + name)

    def _check(self, rc, what):
        if rc != 0:
            raise OracleError(f"{what} failed with code {rc}")

    # ---- inputs ------------------------------------------------------------
    def gen_uniform_rect(self, rows, cols, seed, lo=0.0, hi=1.0) -> np.ndarray:
        out = np.empty((rows, cols), np.float64)
        f = self._fn("gen_uniform_rect")
        if self.kind == "port":
            f(C.c_int64(rows), C.c_int64(cols), C.c_uint64(seed), C.c_double(lo), C.c_double(hi), _p(out))
        else:
            self._check(f(C.c_longlong(rows), C.c_longlong(cols), C.c_ulonglong(seed), C.c_double(lo),
                          C.c_double(hi), _p(out)), "gen_uniform_rect")
        return out

    def gen_test2(self, n, b, seed):
        lhs = np.empty((n, n), np.float64)
        rhs = np.empty((n, n), np.float64)
        f = self._fn("gen_test2")
        self._check(f(C.c_longlong(n), C.c_int(b), C.c_ulonglong(seed), _p(lhs), _p(rhs)), "gen_test2")
        return lhs, rhs

    # ---- guardrails ----------------------------------------------------------
    def scan(self, a):
        a = _f64(a)
        counts = (C.c_uint64 * 3)()
        exc = C.c_int(0)
        if self.kind == "port":
            self.lib.oz_scan(_p(a), C.c_int64(a.size), counts, C.byref(exc))
        else:
            r, c = a.shape
            self._check(self.lib.ozref_scan(_p(a), C.c_longlong(r), C.c_longlong(c), counts,
                                            C.byref(exc)), "scan")
        return tuple(int(x) for x in counts), bool(exc.value)

    def block_stats(self, a, orient, block_len):
        a = _f64(a)
        rows, cols = a.shape
        lines, length = (cols, rows) if orient else (rows, cols)
        blocks = 0 if length == 0 else (length + block_len - 1) // block_len
        mx = np.empty(max(lines * blocks, 1), np.int32)
        mn = np.empty(max(lines * blocks, 1), np.int32)
        lm = np.empty(max(lines, 1), np.int32)
        rc = self._fn("block_stats")(_p(a), C.c_int64(rows), C.c_int64(cols), C.c_int(orient),
                                     C.c_int64(block_len), _p(mx, C.c_int32), _p(mn, C.c_int32),
                                     _p(lm, C.c_int32))
        self._check(rc, "block_stats")
        return (mx[: lines * blocks].reshape(lines, blocks), mn[: lines * blocks].reshape(lines, blocks),
                lm[:lines])

    def esc_coarsened(self, a, b, block_len=256, target_bits=53):
        out = (C.c_int * 3)()
        if self.kind == "port":
            amx, amn, al = self.block_stats(a, 0, block_len)
            bmx, bmn, bl = self.block_stats(b, 1, block_len)
            m, n, t = amx.shape[0], bmx.shape[0], amx.shape[1]
            amx, amn, bmx, bmn = (np.ascontiguousarray(x) for x in (amx, amn, bmx, bmn))
            self.lib.oz_esc_coarsened(_p(amx, C.c_int32), _p(amn, C.c_int32), _p(al, C.c_int32),
                                      _p(bmx, C.c_int32), _p(bmn, C.c_int32), _p(bl, C.c_int32),
                                      C.c_int64(m), C.c_int64(n), C.c_int64(t), C.c_int(target_bits), out)
        else:
            a, b = _f64(a), _f64(b)
            self._check(self.lib.ozref_esc_coarsened(_p(a), _p(b), C.c_longlong(a.shape[0]),
                                                     C.c_longlong(b.shape[1]), C.c_longlong(a.shape[1]),
                                                     C.c_longlong(block_len), C.c_int(target_bits), out),
                        "esc_coarsened")
        return tuple(out)

    def esc_exact(self, a, b, target_bits=53):
        a, b = _f64(a), _f64(b)
        out = (C.c_int * 3)()
        f = self._fn("esc_exact")
        self._check(f(_p(a), _p(b), C.c_int64(a.shape[0]), C.c_int64(b.shape[1]), C.c_int64(a.shape[1]),
                      C.c_int(target_bits), out), "esc_exact")
        return tuple(out)

    def required_slices(self, target_bits, esc_bits):
        if self.kind == "port":
            return self.lib.oz_required_slices(C.c_int(target_bits), C.c_int(esc_bits))
        out = C.c_int(0)
        self._check(self.lib.ozref_required_slices(C.c_int(target_bits), C.c_int(esc_bits), C.byref(out)),
                    "required_slices")
        return out.value

    def decide(self, exc_a, exc_b, m, n, k, esc_in, cfg: Config):
        """Returns (path, reason, slices, provider_calls, esc_bits, cost_ratio)."""
        cost = C.c_double(0.0)
        if self.kind == "port":
            c = _OzConfig(cfg.target_bits, cfg.esc_block_len, cfg.max_slices, cfg.min_dim, cfg.mode,
                          cfg.forced_slices, cfg.cost_ratio, cfg.chunk_len)
            out = (C.c_int * 5)()
            self._check(self.lib.oz_decide(C.c_int(exc_a), C.c_int(exc_b), C.c_int64(m), C.c_int64(n),
                                           C.c_int64(k), C.c_int(esc_in), C.byref(c), out, C.byref(cost)),
                        "decide")
        else:
            out = (C.c_int * 5)()
            dd = (C.c_double * 1)(cfg.cost_ratio)
            self._check(self.lib.ozref_decide(C.c_int(exc_a), C.c_int(exc_b), C.c_longlong(m),
                                              C.c_longlong(n), C.c_longlong(k), C.c_int(esc_in), cfg.ints(),
                                              dd, out, C.byref(cost)), "decide")
        return out[0], out[1], out[2], out[3], out[4], cost.value

    # ---- emulation -----------------------------------------------------------
    def decompose(self, a, orient, slices):
        a = _f64(a)
        rows, cols = a.shape
        lines, length = (cols, rows) if orient else (rows, cols)
        dig = np.empty(max(slices * lines * length, 1), np.int8)
        sc = np.empty(max(lines, 1), np.int32)
        f = self._fn("decompose")
        self._check(f(_p(a), C.c_int64(rows), C.c_int64(cols), C.c_int(orient), C.c_int(slices),
                      _p(dig, C.c_int8), _p(sc, C.c_int32)), "decompose")
        return dig[: slices * lines * length].reshape(slices, lines, length), sc[:lines]

    def slice_pair_mm(self, a, b, slices, limit=-1, chunk=65536):
        a, b = _f64(a), _f64(b)
        m, k = a.shape
        n = b.shape[1]
        acc = np.empty(max(m * n * (2 * slices - 1), 1), np.int64)
        if self.kind == "port":
            sa, _ = self.decompose(a, 0, slices)
            sb, _ = self.decompose(b, 1, slices)
            sa, sb = np.ascontiguousarray(sa), np.ascontiguousarray(sb)
            self._check(self.lib.oz_slice_pair_mm(_p(sa, C.c_int8), _p(sb, C.c_int8), C.c_int64(m),
                                                  C.c_int64(n), C.c_int64(k), C.c_int(slices), C.c_int(limit),
                                                  _p(acc, C.c_int64)), "slice_pair_mm")
        else:
            self._check(self.lib.ozref_slice_pair_mm(_p(a), _p(b), C.c_longlong(m), C.c_longlong(n),
                                                     C.c_longlong(k), C.c_int(slices), C.c_longlong(chunk),
                                                     C.c_int(limit), _p(acc, C.c_longlong)), "slice_pair_mm")
        return acc[: m * n * (2 * slices - 1)].reshape(m, n, 2 * slices - 1)

    def emulated_gemm(self, a, b, slices, alpha=1.0, beta=0.0, c=None, limit=-1):
        a, b = _f64(a), _f64(b)
        m, k = a.shape
        n = b.shape[1]
        out = np.empty((m, n), np.float64)
        cp = _p(_f64(c)) if c is not None else None
        cc = _f64(c) if c is not None else None
        cp = _p(cc) if cc is not None else None
        if self.kind == "port":
            rc = self.lib.oz_emulated_gemm(_p(a), _p(b), C.c_int64(m), C.c_int64(n), C.c_int64(k),
                                           C.c_double(alpha), C.c_double(beta), cp, C.c_int(slices),
                                           C.c_int(limit), _p(out))
        else:
            rc = self.lib.ozref_emulated_gemm(_p(a), _p(b), C.c_longlong(m), C.c_longlong(n), C.c_longlong(k),
                                              C.c_double(alpha), C.c_double(beta), cp, C.c_int(slices),
                                              C.c_longlong(65536), C.c_int(limit), _p(out))
        self._check(rc, "emulated_gemm")
        return out

    def native_gemm(self, a, b, alpha=1.0, beta=0.0, c=None):
        a, b = _f64(a), _f64(b)
        m, k = a.shape
        n = b.shape[1]
        out = np.empty((m, n), np.float64)
        cc = _f64(c) if c is not None else None
        cp = _p(cc) if cc is not None else None
        f = self._fn("native_gemm")
        self._check(f(_p(a), _p(b), C.c_int64(m), C.c_int64(n), C.c_int64(k), C.c_double(alpha),
                      C.c_double(beta), cp, _p(out)), "native_gemm")
        return out

    def exact_gemm(self, a, b):
        a, b = _f64(a), _f64(b)
        m, k = a.shape
        n = b.shape[1]
        out = np.empty((m, n), np.float64)
        f = self._fn("exact_gemm")
        self._check(f(_p(a), _p(b), C.c_int64(m), C.c_int64(n), C.c_int64(k), _p(out)), "exact_gemm")
        return out

    def adp_gemm(self, a, b, alpha=1.0, beta=0.0, c=None, cfg: Config | None = None):
        """Returns (C, trace dict) like ozadp::adp_gemm (proj/src/adp.cpp:139-178)."""
        cfg = cfg or Config()
        a, b = _f64(a), _f64(b)
        m, k = a.shape
        n = b.shape[1]
        out = np.empty((m, n), np.float64)
        cc = _f64(c) if c is not None else None
        cp = _p(cc) if cc is not None else None
        cost = C.c_double(0.0)
        if self.kind == "port":
            oc = _OzConfig(cfg.target_bits, cfg.esc_block_len, cfg.max_slices, cfg.min_dim, cfg.mode,
                           cfg.forced_slices, cfg.cost_ratio, cfg.chunk_len)
            tr = (C.c_int64 * 10)()
            self._check(self.lib.oz_adp_gemm(_p(a), _p(b), C.c_int64(m), C.c_int64(n), C.c_int64(k),
                                             C.c_double(alpha), C.c_double(beta), cp, C.byref(oc), _p(out), tr,
                                             C.byref(cost)), "adp_gemm")
            t = dict(path=int(tr[0]), reason=int(tr[1]), esc_bits=int(tr[2]), slices=int(tr[3]),
                     scan_a=tuple(int(x) for x in tr[4:7]), scan_b=tuple(int(x) for x in tr[7:10]))
        else:
            ti = (C.c_longlong * 13)()
            td = (C.c_double * 1)()
            js = C.create_string_buffer(512)
            dd = (C.c_double * 1)(cfg.cost_ratio)
            self._check(self.lib.ozref_adp_gemm(_p(a), _p(b), C.c_longlong(m), C.c_longlong(n), C.c_longlong(k),
                                                C.c_double(alpha), C.c_double(beta), cp, cfg.ints(), dd, _p(out),
                                                ti, td, js, C.c_int(512)), "adp_gemm")
            t = dict(path=int(ti[0]), reason=int(ti[1]), esc_bits=int(ti[2]), slices=int(ti[3]),
                     scan_a=tuple(int(x) for x in ti[7:10]), scan_b=tuple(int(x) for x in ti[10:13]),
                     json=js.value.decode())
            cost = C.c_double(td[0])
        t["modeled_cost_ratio"] = cost.value
        t["m"], t["n"], t["k"] = m, n, k
        return out, t

    # ---- reference-only helpers ---------------------------------------------------
    def set_threads(self, n: int) -> None:
        if self.kind == "reference":
            self.lib.ozref_set_threads(C.c_int(n))

    def time_call(self, which: int, a, b, slices=7) -> float:
        """Reference arm timing (seconds) of one emulated(0)/adp(1)/native(2) call."""
        if self.kind != "reference":
            raise OracleError("time_call needs the reference build")
        a, b = _f64(a), _f64(b)
        self.lib.ozref_time_call.restype = C.c_double
        return float(self.lib.ozref_time_call(C.c_int(which), _p(a), _p(b), C.c_longlong(a.shape[0]),
                                              C.c_longlong(b.shape[1]), C.c_longlong(a.shape[1]),
                                              C.c_int(slices), None))

    # ---- grading (reference build only) ---------------------------------------
    def _need_ref(self, what):
        if self.kind != "reference":
            raise OracleError(f"{what} needs the reference build")

    def error_report(self, c, ref, exact_diag=None):
        """error_report (grading.cpp:67-90): (max_err, avg_err, counted, skipped)."""
        self._need_ref("error_report")
        c, ref = _f64(c), _f64(ref)
        out = (C.c_double * 4)()
        self._check(self.lib.ozref_error_report(_p(c), _p(ref), C.c_longlong(c.shape[0]), C.c_longlong(c.shape[1]),
                                                C.c_int(exact_diag is not None),
                                                C.c_double(exact_diag or 0.0), out), "error_report")
        return out[0], out[1], int(out[2]), int(out[3])

    def exact_dot(self, x, y) -> float:
        self._need_ref("exact_dot")
        x, y = _f64(x), _f64(y)
        out = C.c_double(0.0)
        self._check(self.lib.ozref_exact_dot(_p(x), _p(y), C.c_longlong(x.size), C.byref(out)), "exact_dot")
        return out.value

    def grade_uniform_point(self, n, seed):
        """grade_uniform_point (grading.cpp:92-134), default AdpConfig."""
        self._need_ref("grade_uniform_point")
        out = (C.c_double * 7)()
        self._check(self.lib.ozref_grade_uniform_point(C.c_longlong(n), C.c_ulonglong(seed), out),
                    "grade_uniform_point")
        return dict(emu_max_ratio=out[0], emu_avg_ratio=out[1], nat_max_ratio=out[2], nat_avg_ratio=out[3],
                    esc_bits=int(out[4]), slices=int(out[5]), fallback=bool(out[6]))

    def test2_row(self, n, b, mode, seed):
        """One row of run_test2_sweep (grading.cpp:246-275)."""
        self._need_ref("test2_row")
        out = (C.c_double * 5)()
        self._check(self.lib.ozref_test2_row(C.c_longlong(n), C.c_int(b), mode.encode(), C.c_ulonglong(seed), out),
                    "test2_row")
        return dict(max_err=out[0], avg_err=out[1], esc_bits=None if out[2] < 0 else int(out[2]),
                    slices=int(out[3]), fallback=bool(out[4]))

    def qr(self, a, panel, cfg: "Config | None" = None, want_q=True):
        """geqrf_blocked + materialize_q + qr_residual (qr.cpp) of the reference:
        (factors, t_packed, traces [3*panels x 7], q or None, (residual, orthogonality))."""
        self._need_ref("qr")
        cfg = cfg or Config()
        a = _f64(a)
        m, n = a.shape
        panels = (n + panel - 1) // panel
        fac = np.empty((m, n), np.float64)
        t = np.zeros(max(1, panels * panel * panel), np.float64)
        tr = np.zeros((max(1, 3 * panels), 7), np.int64)
        q = np.empty((m, n), np.float64) if want_q else None
        acc = (C.c_double * 2)()
        cd = (C.c_double * 1)(cfg.cost_ratio)
        self._check(self.lib.ozref_qr(_p(a), C.c_longlong(m), C.c_longlong(n), C.c_longlong(panel), cfg.ints(), cd,
                                      _p(fac), _p(t), _p(tr, C.c_longlong), None if q is None else _p(q), acc), "qr")
        return fac, t, tr[: 3 * panels], q, (acc[0], acc[1])

    def time_qr(self, a, panel, min_dim=256) -> float:
        self._need_ref("time_qr")
        a = _f64(a)
        self.lib.ozref_time_qr.restype = C.c_double
        return float(self.lib.ozref_time_qr(_p(a), C.c_longlong(a.shape[0]), C.c_longlong(a.shape[1]),
                                            C.c_longlong(panel), C.c_longlong(min_dim)))

    def write_matrix(self, path, a):
        self._need_ref("write_matrix")
        a = _f64(a)
        self._check(self.lib.ozref_write_matrix(path.encode(), _p(a), C.c_longlong(a.shape[0]),
                                                C.c_longlong(a.shape[1])), "write_matrix")

    def read_matrix(self, path):
        self._need_ref("read_matrix")
        dims = (C.c_longlong * 2)()
        self._check(self.lib.ozref_read_matrix(path.encode(), None, C.c_longlong(0), dims), "read_matrix")
        out = np.empty((dims[0], dims[1]), np.float64)
        self._check(self.lib.ozref_read_matrix(path.encode(), _p(out), C.c_longlong(out.size), dims), "read_matrix")
        return out


def exponent_field(a: np.ndarray) -> np.ndarray:
    """Effective exponents floor(log2|v|) with NEG_SENTINEL at zeros and non-finite
    values (esc.cpp:26-56 exponent_field; subnormals included via frexp)."""
    a = np.abs(_f64(a))
    _, e = np.frexp(a)
    ok = (a != 0) & np.isfinite(a)
    return np.where(ok, e.astype(np.int64) - 1, NEG_SENTINEL)


def certify_delta(target_bits: int, level: int = 0) -> int:
    """Indicator threshold of certificate level `level` (targets s0 + level slices,
    s0 = required_slices(target_bits, 0), esc.cpp:8-12): 2 delta + 1 is the largest
    ESC those slices tolerate; -1 when the level cannot help."""
    s = (target_bits + 2 + 7) // 8 + level
    e = 8 * s - target_bits - 2
    return (e - 1) // 2 if e >= 1 else -1


def esc_certified(a, b, coarse_esc: int, target_bits: int = 53, window: int = 512) -> int:
    """Numpy restatement of the certified ESC (adpb200_options.esc_method = 1,
    guard.cu certify_prep_kernel / certified_esc). Level l holds when every (i, j)
    has some position l among the first `window` with e(a_il) >= rowmax_i - delta_l
    and e(b_lj) >= colmax_j - delta_l (row / column maxima over whole lines): then
    the exact z_ij of esc_exact (esc.cpp:61-87) is >= rowmax_i + colmax_j - 2 delta_l
    and span_ij <= 2 delta_l + 1. A level is tested only when the coarsened ESC
    exceeds its bound; level 0 wins over level 1; otherwise coarse_esc stays."""
    d0, d1 = certify_delta(target_bits, 0), certify_delta(target_bits, 1)
    l0 = d0 >= 0 and coarse_esc > 2 * d0 + 1
    l1 = d1 >= 0 and coarse_esc > 2 * d1 + 1
    if not (l0 or l1):
        return coarse_esc
    ea, eb = exponent_field(a), exponent_field(b)
    rmax = ea.max(axis=1, initial=NEG_SENTINEL)
    cmax = eb.max(axis=0, initial=NEG_SENTINEL)
    ea, eb = ea[:, :window], eb[:window, :]

    def holds(delta):
        p = ((ea != NEG_SENTINEL) & (ea >= rmax[:, None] - delta)).astype(np.float64)
        q = ((eb != NEG_SENTINEL) & (eb >= cmax[None, :] - delta)).astype(np.float64)
        return bool(((p @ q) > 0).all())  # exact: 0/1 products, sums <= window < 2^53

    if l0 and holds(d0):
        return 2 * d0 + 1
    if l1 and holds(d1):
        return 2 * d1 + 1
    return coarse_esc


def fold_round(acc_row: np.ndarray, exp2: int) -> float:
    """Exact fold of one element's diagonal accumulators + RNE (port only)."""
    lib = _load("port")
    lib.oz_fold_round.restype = C.c_double
    a = np.ascontiguousarray(acc_row, dtype=np.int64)
    return float(lib.oz_fold_round(_p(a, C.c_int64), C.c_int(a.size), C.c_long(exp2)))
