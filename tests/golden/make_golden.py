"""Generate tests/golden/*.npz from the REFERENCE implementation.

Runs in the build container only (needs oracle/_ref, i.e. the reference's own
sources under /root/reference compiled by oracle/Makefile). The fixtures are
committed so the parity tests can pin the oracle and the GPU path to the
reference's outputs anywhere, including the GPU box where /root/reference does
not exist.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Config, Oracle  # noqa: E402


def wide(rows, cols, seed, span, subnormals=0.0):
    rng = np.random.default_rng(seed)
    m = rng.uniform(1.0, 2.0, (rows, cols)) * np.ldexp(1.0, rng.integers(-span, span + 1, (rows, cols)))
    m *= np.where(rng.random((rows, cols)) < 0.5, -1.0, 1.0)
    z = rng.random((rows, cols))
    m[z < 0.05] = 0.0
    m[(z >= 0.05) & (z < 0.075)] = -0.0
    if subnormals:
        s = rng.random((rows, cols)) < subnormals
        m[s] = np.ldexp(rng.uniform(1.0, 2.0, s.sum()), -1060)
    return m


def main():
    R = Oracle("reference")
    out = {}

    # case 1: xoshiro uniform operands (gen_uniform_rect, grading.cpp:56-63)
    m, n, k = 64, 48, 80
    a = R.gen_uniform_rect(m, k, 1, -1.0, 1.0)
    b = R.gen_uniform_rect(k, n, 2, -1.0, 1.0)
    c = R.gen_uniform_rect(m, n, 3, -1.0, 1.0)
    out["u_a"], out["u_b"], out["u_c"] = a, b, c
    for o, mat in ((0, a), (1, b)):
        mx, mn, lm = R.block_stats(mat, o, 16)
        out[f"u_stats{o}_max"], out[f"u_stats{o}_min"], out[f"u_stats{o}_line"] = mx, mn, lm
        for s in (4, 7, 9):
            d, sc = R.decompose(mat, o, s)
            out[f"u_dec{o}_s{s}"], out[f"u_dec{o}_s{s}_scale"] = d, sc
    out["u_esc_c16"] = np.array(R.esc_coarsened(a, b, 16))
    out["u_esc_c256"] = np.array(R.esc_coarsened(a, b, 256))
    out["u_esc_exact"] = np.array(R.esc_exact(a, b))
    out["u_acc_s7_full"] = R.slice_pair_mm(a, b, 7, -1)
    out["u_acc_s7_l7"] = R.slice_pair_mm(a, b, 7, 7)
    out["u_emu_s7"] = R.emulated_gemm(a, b, 7, -1.25, 0.5, c)
    out["u_emu_s9_l9"] = R.emulated_gemm(a, b, 9, 1.0, 0.0, None, 9)
    out["u_native"] = R.native_gemm(a, b, 2.5, -1.0, c)
    out["u_exact"] = R.exact_gemm(a, b)
    cfg = Config(min_dim=8)
    res, tr = R.adp_gemm(a, b, -1.25, 0.5, c, cfg)
    out["u_adp"] = res
    out["u_adp_trace"] = np.array([tr["path"], tr["reason"], tr["esc_bits"], tr["slices"]])

    # case 2: Test-2 exponent-span pair (grading.cpp:13-47), b = 8
    lhs, rhs = R.gen_test2(64, 8, 42)
    out["t2_lhs"], out["t2_rhs"] = lhs, rhs
    out["t2_esc"] = np.array(R.esc_coarsened(lhs, rhs, 16))
    res, tr = R.adp_gemm(lhs, rhs, 1.0, 0.0, None, Config(min_dim=8, esc_block_len=16))
    out["t2_adp"] = res
    out["t2_adp_trace"] = np.array([tr["path"], tr["reason"], tr["esc_bits"], tr["slices"]])

    # case 3: wide spans + subnormals
    wa = wide(40, 56, 7, 400, 0.03)
    wb = wide(56, 36, 8, 400, 0.03)
    out["w_a"], out["w_b"] = wa, wb
    for s in (7, 12):
        d, sc = R.decompose(wa, 0, s)
        out[f"w_dec0_s{s}"], out[f"w_dec0_s{s}_scale"] = d, sc
    out["w_emu_s9"] = R.emulated_gemm(wa, wb, 9)
    out["w_emu_s18_full"] = R.emulated_gemm(wa, wb, 18)

    # case 4: exceptional values route to native (adp.cpp:58-62)
    ea = a.copy()
    ea[3, 5] = np.nan
    eb = b.copy()
    eb[7, 2] = -np.inf
    res, tr = R.adp_gemm(ea, eb, 1.0, 0.0, None, Config(min_dim=8))
    out["x_a"], out["x_b"], out["x_adp"] = ea, eb, res
    out["x_adp_trace"] = np.array([tr["path"], tr["reason"], tr["esc_bits"], tr["slices"]])

    np.savez_compressed(os.path.join(HERE, "reference_vectors.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_vectors.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
