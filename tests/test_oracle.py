"""CPU: pin the oracle (oracle/adp_oracle.c, the C restatement) to the reference.

1. Against the committed golden vectors produced by the reference itself
   (tests/golden/reference_vectors.npz, generator committed beside it).
2. Against the reference's own known-answer tests, restated
   (proj/tests/test_slicing.cpp, test_fpbits.cpp, test_esc.cpp,
   test_igemm.cpp, test_adp.cpp).
3. Against the live reference build (oracle/_ref) on seeded random cases,
   when it is present (this container; skipped on the GPU box).
"""
import os

import numpy as np
import pytest

from conftest import assert_bitwise

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_vectors.npz")


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


# ---- 1. golden vectors ---------------------------------------------------------------------
def test_golden_inputs_regenerate(port, gold):
    # xoshiro256++ + splitmix64 streams are bit-identical (rng.hpp:11-54)
    assert np.array_equal(port.gen_uniform_rect(64, 80, 1, -1.0, 1.0), gold["u_a"])
    assert np.array_equal(port.gen_uniform_rect(80, 48, 2, -1.0, 1.0), gold["u_b"])
    lhs, rhs = port.gen_test2(64, 8, 42)
    assert np.array_equal(lhs, gold["t2_lhs"]) and np.array_equal(rhs, gold["t2_rhs"])


def test_golden_stats_esc(port, gold):
    a, b = gold["u_a"], gold["u_b"]
    for o, mat in ((0, a), (1, b)):
        mx, mn, lm = port.block_stats(mat, o, 16)
        assert np.array_equal(mx, gold[f"u_stats{o}_max"])
        assert np.array_equal(mn, gold[f"u_stats{o}_min"])
        assert np.array_equal(lm, gold[f"u_stats{o}_line"])
    assert list(port.esc_coarsened(a, b, 16)) == gold["u_esc_c16"].tolist()
    assert list(port.esc_coarsened(a, b, 256)) == gold["u_esc_c256"].tolist()
    assert list(port.esc_exact(a, b)) == gold["u_esc_exact"].tolist()
    assert list(port.esc_coarsened(gold["t2_lhs"], gold["t2_rhs"], 16)) == gold["t2_esc"].tolist()


def test_golden_slicing(port, gold):
    for o, mat in ((0, gold["u_a"]), (1, gold["u_b"])):
        for s in (4, 7, 9):
            d, sc = port.decompose(mat, o, s)
            assert np.array_equal(d, gold[f"u_dec{o}_s{s}"]) and np.array_equal(sc, gold[f"u_dec{o}_s{s}_scale"])
    for s in (7, 12):
        d, sc = port.decompose(gold["w_a"], 0, s)
        assert np.array_equal(d, gold[f"w_dec0_s{s}"]) and np.array_equal(sc, gold[f"w_dec0_s{s}_scale"])


def test_golden_products_and_gemm(port, gold):
    a, b, c = gold["u_a"], gold["u_b"], gold["u_c"]
    assert np.array_equal(port.slice_pair_mm(a, b, 7, -1), gold["u_acc_s7_full"])
    assert np.array_equal(port.slice_pair_mm(a, b, 7, 7), gold["u_acc_s7_l7"])
    assert_bitwise(port.emulated_gemm(a, b, 7, -1.25, 0.5, c), gold["u_emu_s7"], nan_equiv=False)
    assert_bitwise(port.emulated_gemm(a, b, 9, 1.0, 0.0, None, 9), gold["u_emu_s9_l9"], nan_equiv=False)
    assert_bitwise(port.native_gemm(a, b, 2.5, -1.0, c), gold["u_native"], nan_equiv=False)
    assert_bitwise(port.exact_gemm(a, b), gold["u_exact"], nan_equiv=False)
    assert_bitwise(port.emulated_gemm(gold["w_a"], gold["w_b"], 9), gold["w_emu_s9"], nan_equiv=False)
    assert_bitwise(port.emulated_gemm(gold["w_a"], gold["w_b"], 18), gold["w_emu_s18_full"], nan_equiv=False)


def test_golden_adp(port, gold):
    from oracle.oracle import Config

    res, tr = port.adp_gemm(gold["u_a"], gold["u_b"], -1.25, 0.5, gold["u_c"], Config(min_dim=8))
    assert_bitwise(res, gold["u_adp"], nan_equiv=False)
    assert [tr["path"], tr["reason"], tr["esc_bits"], tr["slices"]] == gold["u_adp_trace"].tolist()
    res, tr = port.adp_gemm(gold["t2_lhs"], gold["t2_rhs"], 1.0, 0.0, None, Config(min_dim=8, esc_block_len=16))
    assert_bitwise(res, gold["t2_adp"], nan_equiv=False)
    assert [tr["path"], tr["reason"], tr["esc_bits"], tr["slices"]] == gold["t2_adp_trace"].tolist()
    res, tr = port.adp_gemm(gold["x_a"], gold["x_b"], 1.0, 0.0, None, Config(min_dim=8))
    assert_bitwise(res, gold["x_adp"])
    assert [tr["path"], tr["reason"], tr["esc_bits"], tr["slices"]] == gold["x_adp_trace"].tolist()


# ---- 2. the reference's own known-answer tests ------------------------------------------
def test_kat_block_stats(port):
    # test_fpbits.cpp:120-139
    mx, mn, lm = port.block_stats(np.array([[1.0, 0.125, 0.0, 32.0]]), 0, 2)
    assert mx.tolist() == [[0, 5]] and mn.tolist() == [[-3, 5]] and lm.tolist() == [5]
    # all-zero block / line carry the sentinel (test_fpbits.cpp:141-155)
    mx, mn, lm = port.block_stats(np.zeros((1, 4)), 0, 2)
    assert (mx == -1000000).all() and (lm == -1000000).all()
    # ragged tail (test_fpbits.cpp:157-165)
    mx, _, _ = port.block_stats(np.array([[1.0, 2.0, 4.0, 8.0, 16.0]]), 0, 2)
    assert mx.tolist() == [[1, 3, 4]]
    # denormal exponents (test_fpbits.cpp:41-59)
    assert port.block_stats(np.array([[5e-324]]), 0, 1)[0].tolist() == [[-1074]]


def test_kat_required_slices(port):
    # test_esc.cpp:64-74
    assert port.required_slices(53, 1) == 7
    assert port.required_slices(53, 2) == 8
    assert port.required_slices(53, 17) == 9
    assert port.required_slices(24, 0) == 4


def test_kat_esc_two_term(port):
    # test_esc.cpp:76-89: exponents {100, 90} x {-100, -80} -> esc 11, window 64, 9 slices
    a = np.array([[2.0 ** 100, 2.0 ** 90]])
    b = np.array([[2.0 ** -100], [2.0 ** -80]])
    assert port.esc_exact(a, b) == (11, 64, 9)
    assert port.esc_coarsened(a, b, 1) == (11, 64, 9)  # b = 1 gives equality (test_esc.cpp:177-187)
    # aligned exponents give the minimal span (test_esc.cpp:91-96)
    assert port.esc_exact(np.ones((4, 4)), np.ones((4, 4)))[0] == 1
    # padding narrative p + 1 (test_esc.cpp:98-111)
    for p in (0, 3, 17, 60):
        a = np.array([[2.0 ** 100, 1.5 * 2.0 ** (100 - p)]])
        b = np.array([[0.0], [1.0]])
        assert port.esc_exact(a, b)[0] == p + 1
    # structurally zero dot products (test_esc.cpp:113-133)
    z, m = np.zeros((3, 3)), np.full((3, 3), 2.0)
    assert port.esc_exact(z, m)[0] == 0 and port.esc_coarsened(z, m, 2)[0] == 0


def test_kat_decompose(port):
    # test_slicing.cpp:192-231
    d, s = port.decompose(np.array([[1.0]]), 0, 4)
    assert s.tolist() == [2] and d[:, 0, 0].tolist() == [32, 0, 0, 0]
    d, s = port.decompose(np.array([[-1.0]]), 0, 4)
    assert d[:, 0, 0].tolist() == [-32, 0, 0, 0]
    d, s = port.decompose(np.array([[0.0, -0.0, 0.0]]), 0, 3)
    assert s.tolist() == [0] and not d.any()
    v = np.ldexp(2.0 - np.ldexp(1.0, -52), 10)
    d, s = port.decompose(np.array([[v]]), 0, 7)
    assert s.tolist() == [12] and d[:, 0, 0].tolist() == [64, 0, 0, 0, 0, 0, -2]


def test_kat_igemm(port):
    # test_igemm.cpp:62-75: 1x1 accumulator check; 32x32 U(1,2) s=7 bitwise = exact (:99-121)
    a = port.gen_uniform_rect(32, 32, 11, 1.0, 2.0)
    b = port.gen_uniform_rect(32, 32, 12, 1.0, 2.0)
    assert_bitwise(port.emulated_gemm(a, b, 7), port.exact_gemm(a, b), nan_equiv=False)
    # structurally zero dot -> +0.0 (test_igemm.cpp:224-236)
    z = port.emulated_gemm(np.array([[1.0, 0.0]]), np.array([[0.0], [5.0]]), 7)
    assert z.view(np.uint64)[0, 0] == 0
    # terminal overflow is +/-Inf and never a fallback (test_igemm.cpp:238-250)
    big = np.full((2, 2), 2.0 ** 1000)
    assert np.isinf(port.emulated_gemm(big, big, 7)).all()


def test_kat_decide_gate_order(port):
    # test_adp.cpp:82-151 with the fake ESC provider
    from oracle.oracle import Config

    cfg = Config()
    assert port.decide(0, 0, 1024, 1024, 1024, 1, cfg)[:4] == (0, 0, 7, 1)
    assert port.decide(1, 0, 1024, 1024, 1024, 1, cfg)[:4] == (1, 2, 0, 0)       # exceptional, no ESC
    assert port.decide(0, 0, 100, 1024, 1024, 1, cfg)[:4] == (1, 4, 0, 0)        # too small, no ESC
    assert port.decide(0, 0, 1024, 1024, 1024, 95, cfg)[:4] == (1, 3, 0, 1)      # 19 slices > 18
    assert port.decide(0, 0, 1024, 1024, 1024, 1, Config(mode=2))[:4] == (1, 1, 0, 0)
    assert port.decide(1, 0, 1024, 1024, 1024, 1, Config(mode=1, forced_slices=5))[:4] == (1, 2, 0, 0)
    assert port.decide(0, 0, 8, 8, 8, 1, Config(mode=1, forced_slices=5))[:4] == (0, 1, 5, 0)
    assert port.decide(0, 0, 1024, 1024, 1024, 1, Config(cost_ratio=16.0))[:4] == (1, 5, 0, 1)


# ---- 3. live reference -------------------------------------------------------------------------
@pytest.mark.reference
@pytest.mark.parametrize("shape", [(1, 1, 1), (5, 7, 300), (33, 17, 513)])
def test_port_matches_reference(port, ref, shape):
    from oracle.oracle import Config

    m, n, k = shape
    a = port.gen_uniform_rect(m, k, 1, -1.0, 1.0)
    b = port.gen_uniform_rect(k, n, 2, -1.0, 1.0)
    c = np.random.default_rng(0).standard_normal((m, n))
    for o, mat in ((0, a), (1, b)):
        for bl in (1, 3, 256):
            assert all(np.array_equal(x, y) for x, y in zip(port.block_stats(mat, o, bl), ref.block_stats(mat, o, bl)))
    assert port.esc_coarsened(a, b) == ref.esc_coarsened(a, b)
    assert port.esc_exact(a, b) == ref.esc_exact(a, b)
    for s in (1, 4, 7, 9, 17):
        for o, mat in ((0, a), (1, b)):
            x, y = port.decompose(mat, o, s), ref.decompose(mat, o, s)
            assert np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1])
        for lim in (-1, s, s - 1):
            assert np.array_equal(port.slice_pair_mm(a, b, s, lim), ref.slice_pair_mm(a, b, s, lim))
            assert_bitwise(port.emulated_gemm(a, b, s, -1.25, 0.5, c, lim),
                           ref.emulated_gemm(a, b, s, -1.25, 0.5, c, lim), nan_equiv=False)
    assert_bitwise(port.native_gemm(a, b, 2.5, -1, c), ref.native_gemm(a, b, 2.5, -1, c), nan_equiv=False)
    assert_bitwise(port.exact_gemm(a, b), ref.exact_gemm(a, b), nan_equiv=False)
    for mode in (0, 1, 2):
        cfg = Config(mode=mode, min_dim=1)
        x, tx = port.adp_gemm(a, b, 1.0, 0.0, None, cfg)
        y, ty = ref.adp_gemm(a, b, 1.0, 0.0, None, cfg)
        assert_bitwise(x, y, nan_equiv=False)
        for key in ("path", "reason", "esc_bits", "slices", "scan_a", "scan_b"):
            assert tx[key] == ty[key]


@pytest.mark.reference
def test_port_decide_matches_reference(port, ref):
    from oracle.oracle import Config

    rng = np.random.default_rng(5)
    for _ in range(300):
        cfg = Config(mode=int(rng.integers(0, 3)), min_dim=int(rng.integers(1, 600)),
                     cost_ratio=float(rng.choice([1.0, 16.0, 512.0, 3.7])), forced_slices=int(rng.integers(1, 33)),
                     max_slices=int(rng.integers(7, 33)))
        args = (int(rng.integers(0, 2)), int(rng.integers(0, 2)), int(rng.integers(0, 5000)),
                int(rng.integers(0, 5000)), int(rng.integers(0, 5000)), int(rng.integers(0, 200)))
        p, r = port.decide(*args, cfg), ref.decide(*args, cfg)
        assert p[:5] == r[:5]
        assert np.float64(p[5]).view(np.uint64) == np.float64(r[5]).view(np.uint64)
