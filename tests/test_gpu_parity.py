"""GPU parity: every stage of the B200 pipeline against the CPU oracle.

Bit-exact bar (integer / byte / index work and the exactly-rounded FP64
results): block stats, ESC, slice planes, int32->int64 slice products,
emulated C, native fallback C, the ADP decision. Inputs are seeded and
generated bit-identically to the reference (xoshiro256++ gen_uniform_rect).
"""
import numpy as np
import pytest

from conftest import assert_bitwise

pytestmark = pytest.mark.gpu


def wide_matrix(rows, cols, seed, span=40, zeros=0.05, subnormals=0.0):
    """Signed values with exponents spread over [-span, span], some zeros,
    -0.0 and optional subnormals — the ragged inputs the reference tests use."""
    rng = np.random.default_rng(seed)
    m = rng.uniform(1.0, 2.0, (rows, cols)) * np.ldexp(1.0, rng.integers(-span, span + 1, (rows, cols)))
    m *= np.where(rng.random((rows, cols)) < 0.5, -1.0, 1.0)
    z = rng.random((rows, cols))
    m[z < zeros] = 0.0
    m[(z >= zeros) & (z < zeros * 1.5)] = -0.0
    if subnormals:
        s = rng.random((rows, cols)) < subnormals
        m[s] = np.ldexp(rng.uniform(1.0, 2.0, s.sum()), -1060) * np.where(rng.random(s.sum()) < 0.5, -1, 1)
    return m


def _checker(port, request, work):
    """The single-threaded C restatement for small cases; above ~4e8 slice
    MACs the reference itself (oracle/_ref, OpenMP over every host core),
    which the restatement is pinned to (tests/test_oracle.py)."""
    if work <= 4e8:
        return port
    return request.getfixturevalue("ref")


# ---- K1: scan + block statistics ------------------------------------------------------
@pytest.mark.parametrize("shape", [(1, 1), (3, 1000), (257, 131), (64, 513), (1000, 7)])
@pytest.mark.parametrize("orient", [0, 1])
@pytest.mark.parametrize("block_len", [1, 3, 256])
def test_block_stats(gpu, port, shape, orient, block_len):
    a = wide_matrix(*shape, seed=sum(shape) + orient + block_len, span=300, subnormals=0.02)
    mx, mn, lm, exc = gpu.block_exponent_stats(a, orient, block_len)
    rmx, rmn, rlm = port.block_stats(a, orient, block_len)
    assert not exc
    assert np.array_equal(mx, rmx) and np.array_equal(mn, rmn) and np.array_equal(lm, rlm)


def test_block_stats_sentinel_and_hand_example(gpu):
    # test_fpbits.cpp:120-139: [1, 2^-3, 0, 2^5], b=2 -> (0,-3), (5,5)
    a = np.array([[1.0, 0.125, 0.0, 32.0]])
    mx, mn, lm, _ = gpu.block_exponent_stats(a, 0, 2)
    assert mx.tolist() == [[0, 5]] and mn.tolist() == [[-3, 5]] and lm.tolist() == [5]
    z = np.zeros((2, 5))
    mx, mn, lm, _ = gpu.block_exponent_stats(z, 0, 2)
    assert (mx == -1000000).all() and (mn == -1000000).all() and (lm == -1000000).all()


def test_scan_counts(gpu, port):
    a = wide_matrix(100, 77, seed=5)
    a[3, 4] = np.nan
    a[7, 7] = np.inf
    a[9, 1] = -np.inf
    a.view(np.uint64)[10, 10] = 0xFFF8DEADBEEFCAFE
    counts, exc = gpu.scan_matrix(a)
    rc, rexc = port.scan(a)
    assert counts == rc and exc == rexc and exc
    _, _, _, e = gpu.block_exponent_stats(a, 1, 16)
    assert e


# ---- K2: coarsened ESC -------------------------------------------------------------------
@pytest.mark.parametrize("m,n,k,lo,hi", [(1024, 1024, 1024, -1.0, 1.0), (300, 200, 700, 1.0, 2.0),
                                         (129, 513, 257, -1.0, 1.0)])
def test_esc_uniform(gpu, port, m, n, k, lo, hi):
    a = port.gen_uniform_rect(m, k, 1, lo, hi)
    b = port.gen_uniform_rect(k, n, 2, lo, hi)
    assert gpu.esc_coarsened(a, b) == port.esc_coarsened(a, b)


def test_esc_golden_uniform_1024(gpu, port):
    # SURVEY finding 6 / BASELINE.md: 1024^3 U[-1,1] seeds 1,2 -> esc 11, 9 slices
    a = port.gen_uniform_rect(1024, 1024, 1, -1.0, 1.0)
    b = port.gen_uniform_rect(1024, 1024, 2, -1.0, 1.0)
    assert gpu.esc_coarsened(a, b) == (11, 64, 9)


@pytest.mark.parametrize("b_span", [0, 1, 4, 16, 44, 48])
def test_esc_test2(gpu, port, b_span):
    lhs, rhs = port.gen_test2(512, b_span, 42)
    got = gpu.esc_coarsened(lhs, rhs)
    assert got == port.esc_coarsened(lhs, rhs)
    assert got[0] == 2 * b_span + 1  # esc = 2b+1 (SURVEY finding 6)


def test_esc_sparse_rows(gpu, port):
    a = wide_matrix(200, 600, seed=9, span=200, zeros=0.7)
    b = wide_matrix(600, 150, seed=10, span=200, zeros=0.7)
    a[5, :] = 0.0
    b[:, 7] = 0.0
    assert gpu.esc_coarsened(a, b, 64) == port.esc_coarsened(a, b, 64)


@pytest.mark.parametrize("where", ["first", "late", "none"])
@pytest.mark.parametrize("block_len", [256, 32])
def test_esc_tile_pruning_keeps_the_maximum(gpu, port, where, block_len):
    """The ESC kernel stops a tile once an upper bound of its spans (from the blocks
    seen so far) cannot exceed the maximum other tiles already published. Narrow
    exponents everywhere (U(1,2): every tile prunes after one block) with one
    (row, column) pair whose span is 40+1: a single large element in different
    blocks of an otherwise tiny row of A and column of B, in the first tile or in
    a late one, and with block_len 32 so that tile sees several staged rounds."""
    m, n, k = 1100, 1300, 2304
    a = port.gen_uniform_rect(m, k, 1, 1.0, 2.0)
    b = port.gen_uniform_rect(k, n, 2, 1.0, 2.0)
    if where != "none":
        i, j = (3, 5) if where == "first" else (m - 7, n - 11)
        a[i, :] *= 2.0 ** -40
        a[i, 5 * block_len + 3] = 1.5   # the row's only large element, in block 5
        b[:, j] *= 2.0 ** -40
        b[3 * block_len + 1, j] = 1.25  # the column's, in block 3
    got = gpu.esc_coarsened(a, b, block_len)
    assert got == port.esc_coarsened(a, b, block_len)
    assert got[0] == (41 if where != "none" else 1)


# ---- K3: slicing -----------------------------------------------------------------------------
@pytest.mark.parametrize("slices", [1, 2, 4, 7, 8, 9, 12, 16, 17, 18, 32])
@pytest.mark.parametrize("orient", [0, 1])
def test_decompose(gpu, port, slices, orient):
    a = wide_matrix(70, 133, seed=slices * 7 + orient, span=60, subnormals=0.01)
    dg, sg = gpu.decompose(a, orient, slices)
    dr, sr = port.decompose(a, orient, slices)
    assert np.array_equal(sg, sr)
    assert np.array_equal(dg, dr)


def test_decompose_golden(gpu):
    # test_slicing.cpp:192-231
    d, s = gpu.decompose(np.array([[1.0]]), 0, 4)
    assert s.tolist() == [2] and d[:, 0, 0].tolist() == [32, 0, 0, 0]
    d, s = gpu.decompose(np.array([[-1.0]]), 0, 4)
    assert s.tolist() == [2] and d[:, 0, 0].tolist() == [-32, 0, 0, 0]
    d, s = gpu.decompose(np.array([[0.0, -0.0, 0.0]]), 0, 3)
    assert s.tolist() == [0] and not d.any()
    v = np.ldexp(2.0 - np.ldexp(1.0, -52), 10)
    d, s = gpu.decompose(np.array([[v]]), 0, 7)
    assert s.tolist() == [12] and d[:, 0, 0].tolist() == [64, 0, 0, 0, 0, 0, -2]


def test_decompose_uniform_strided(gpu, port):
    a = port.gen_uniform_rect(384, 300, 3, -1.0, 1.0)
    for orient in (0, 1):
        for s in (7, 8):
            dg, sg = gpu.decompose(a, orient, s)
            dr, sr = port.decompose(a, orient, s)
            assert np.array_equal(dg, dr) and np.array_equal(sg, sr)


# ---- K4: int32 slice products on tcgen05 (per-diagonal int64) --------------------------------
@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (128, 64, 32), (130, 70, 100), (257, 129, 300), (64, 300, 1000)])
@pytest.mark.parametrize("slices,limit", [(1, -1), (2, -1), (3, -1), (4, -1), (5, -1), (6, -1), (7, 7), (7, -1), (8, 8),
                                          (9, 9), (12, 5), (8, -1), (17, 17)])
def test_slice_pair_mm(gpu, port, request, m, n, k, slices, limit):
    chk = _checker(port, request, m * n * k * slices * slices)
    a = wide_matrix(m, k, seed=m + k + slices, span=8)
    b = wide_matrix(k, n, seed=n + k + 2 * slices, span=8)
    got = gpu.slice_pair_mm(a, b, slices, limit)
    want = chk.slice_pair_mm(a, b, slices, limit)
    assert np.array_equal(got, want)


def test_slice_pair_mm_multichunk(gpu, port):
    # s=17 Full: max 17 products per diagonal -> int32 chunk of 7680 k; k=9000 needs 2 chunks
    a = wide_matrix(40, 9000, seed=1, span=3)
    b = wide_matrix(9000, 24, seed=2, span=3)
    assert np.array_equal(gpu.slice_pair_mm(a, b, 17, -1), port.slice_pair_mm(a, b, 17, -1))


# ---- K5: fused exact epilogue (emulated_gemm) -------------------------------------------------
@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (33, 17, 513), (128, 128, 128), (200, 150, 333)])
@pytest.mark.parametrize("slices,limit", [(7, -1), (7, 7), (8, 8), (9, -1), (4, 2), (16, 16), (18, 18), (9, 9), (5, -1), (6, 3)])
def test_emulated_gemm(gpu, port, request, m, n, k, slices, limit):
    chk = _checker(port, request, m * n * k * slices * slices)
    a = port.gen_uniform_rect(m, k, 1, -1.0, 1.0)
    b = port.gen_uniform_rect(k, n, 2, -1.0, 1.0)
    c = np.random.default_rng(3).standard_normal((m, n))
    for alpha, beta in ((1.0, 0.0), (-1.25, 0.5), (2.5, -1.0)):
        got = gpu.emulated_gemm(a, b, slices, alpha, beta, c if beta else None, limit)
        want = chk.emulated_gemm(a, b, slices, alpha, beta, c if beta else None, limit)
        assert_bitwise(got, want)


def test_emulated_gemm_wide_and_tiny(gpu, port):
    # wide exponent spans, subnormal results, cancellation, overflow to +/-Inf
    a = wide_matrix(96, 200, seed=11, span=500, subnormals=0.05)
    b = wide_matrix(200, 80, seed=12, span=500, subnormals=0.05)
    for s, lim in ((7, -1), (12, -1), (9, 9)):
        assert_bitwise(gpu.emulated_gemm(a, b, s, 1.0, 0.0, None, lim), port.emulated_gemm(a, b, s, 1.0, 0.0, None, lim))
    big = np.full((4, 4), 2.0 ** 1000)
    assert_bitwise(gpu.emulated_gemm(big, big, 7), port.emulated_gemm(big, big, 7))  # +Inf, no fallback
    tiny = np.full((3, 3), 2.0 ** -600)
    assert_bitwise(gpu.emulated_gemm(tiny, tiny, 7), port.emulated_gemm(tiny, tiny, 7))  # underflow to 0/subnormal
    x = np.array([[1.0, 1.0], [1.0, -1.0]])
    assert_bitwise(gpu.emulated_gemm(x, x, 7), port.emulated_gemm(x, x, 7))  # exact zeros -> +0.0


def test_emulated_gemm_multichunk(gpu, port):
    # s=7 Full: 7 products per diagonal -> int32 chunk 18720; k=20000 runs 2 chunks
    a = port.gen_uniform_rect(40, 20000, 5, -1.0, 1.0)
    b = port.gen_uniform_rect(20000, 36, 6, -1.0, 1.0)
    assert_bitwise(gpu.emulated_gemm(a, b, 7), port.emulated_gemm(a, b, 7))


def test_emulated_gemm_multichunk_16_column_variant(gpu, port):
    # s=9 Full: 17 diagonals -> the NB = 16 variant (5-limb fold parked in registers),
    # 9 products per diagonal -> int32 chunk 14563; k=16000 runs 2 chunks
    a = port.gen_uniform_rect(24, 16000, 7, -1.0, 1.0)
    b = port.gen_uniform_rect(16000, 20, 8, -1.0, 1.0)
    assert_bitwise(gpu.emulated_gemm(a, b, 9), port.emulated_gemm(a, b, 9))


# ---- K6: native fallback ------------------------------------------------------------------------
@pytest.mark.parametrize("m,n,k", [(1, 1, 0), (5, 7, 1), (65, 70, 131), (130, 64, 300)])
def test_native_gemm_bitwise(gpu, port, m, n, k):
    a = wide_matrix(m, k, seed=m + k, span=30)
    b = wide_matrix(k, n, seed=n + k, span=30)
    c = np.random.default_rng(1).standard_normal((m, n))
    for alpha, beta in ((1.0, 0.0), (2.5, -1.0)):
        assert_bitwise(gpu.native_gemm(a, b, alpha, beta, c if beta else None),
                       port.native_gemm(a, b, alpha, beta, c if beta else None))


# ---- end to end: adp_gemm ---------------------------------------------------------------------
def _cmp_trace(t, rt):
    assert t.path == ("emulated" if rt["path"] == 0 else "native_fallback")
    from oracle.oracle import REASONS

    assert t.reason == REASONS[rt["reason"]]
    assert (t.esc_bits if t.esc_bits is not None else -1) == rt["esc_bits"]
    assert (t.slices if t.slices is not None else -1) == rt["slices"]
    assert t.scan_a == rt["scan_a"] and t.scan_b == rt["scan_b"]


def test_adp_auto_uniform(gpu, port):
    from oracle.oracle import Config

    a = port.gen_uniform_rect(300, 260, 1, 1.0, 2.0)
    b = port.gen_uniform_rect(260, 280, 2, 1.0, 2.0)
    got, t = gpu.adp_gemm(a, b)
    want, rt = port.adp_gemm(a, b, cfg=Config())
    _cmp_trace(t, rt)
    assert t.path == "emulated"
    assert_bitwise(got, want)


@pytest.mark.parametrize("mode", ["auto", "native", "emulate:7", "emulate:11"])
def test_adp_modes_alpha_beta(gpu, port, mode):
    from oracle.oracle import Config

    a = port.gen_uniform_rect(270, 257, 1, -1.0, 1.0)
    b = port.gen_uniform_rect(257, 300, 2, -1.0, 1.0)
    c = port.gen_uniform_rect(270, 300, 3, -1.0, 1.0)
    cfg = gpu.AdpConfig()
    assert gpu.parse_mode(mode, cfg)
    rcfg = Config(mode=int(cfg.mode), forced_slices=cfg.forced_slices)
    got, t = gpu.adp_gemm(a, b, -1.25, 0.5, c, cfg)
    want, rt = port.adp_gemm(a, b, -1.25, 0.5, c, rcfg)
    _cmp_trace(t, rt)
    assert_bitwise(got, want)


def test_adp_exceptional_falls_back_bitwise(gpu, port):
    from oracle.oracle import Config

    rng = np.random.default_rng(0xE6)
    for case in range(6):
        a = port.gen_uniform_rect(260, 256, 10 + case, -1.0, 1.0)
        b = port.gen_uniform_rect(256, 270, 20 + case, -1.0, 1.0)
        tgt = a if case % 2 == 0 else b
        i, j = rng.integers(0, tgt.shape[0]), rng.integers(0, tgt.shape[1])
        tgt[i, j] = [np.nan, np.inf, -np.inf][case % 3]
        if case == 3:
            tgt.view(np.uint64)[i, j] = 0xFFF8DEADBEEFCAFE
        got, t = gpu.adp_gemm(a, b)
        want, rt = port.adp_gemm(a, b, cfg=Config())
        _cmp_trace(t, rt)
        assert t.reason == "exceptional_values"
        assert_bitwise(got, want)  # same bits, or both NaN


def test_adp_negzero_still_emulates(gpu, port):
    from oracle.oracle import Config

    a = port.gen_uniform_rect(256, 256, 1, 1.0, 2.0)
    b = port.gen_uniform_rect(256, 256, 2, 1.0, 2.0)
    a[0, 0] = -0.0
    got, t = gpu.adp_gemm(a, b)
    want, rt = port.adp_gemm(a, b, cfg=Config())
    _cmp_trace(t, rt)
    assert t.path == "emulated" and t.scan_a[2] == 1
    assert_bitwise(got, want)


@pytest.mark.parametrize("b_span,expect", [(4, "ok"), (48, "esc_too_large")])
def test_adp_test2_gates(gpu, port, b_span, expect):
    from oracle.oracle import Config

    lhs, rhs = port.gen_test2(256, b_span, 42)
    got, t = gpu.adp_gemm(lhs, rhs)
    want, rt = port.adp_gemm(lhs, rhs, cfg=Config())
    _cmp_trace(t, rt)
    assert t.reason == expect
    assert_bitwise(got, want)


def test_adp_too_small_and_cost_model(gpu, port):
    from oracle.oracle import Config

    a = port.gen_uniform_rect(100, 300, 1, -1.0, 1.0)
    b = port.gen_uniform_rect(300, 300, 2, -1.0, 1.0)
    got, t = gpu.adp_gemm(a, b)
    want, rt = port.adp_gemm(a, b, cfg=Config())
    _cmp_trace(t, rt)
    assert t.reason == "too_small"
    assert_bitwise(got, want)
    cfg = gpu.AdpConfig(min_dim=8, cost_ratio=16.0)
    got, t = gpu.adp_gemm(a, b, config=cfg)
    want, rt = port.adp_gemm(a, b, cfg=Config(min_dim=8, cost_ratio=16.0))
    _cmp_trace(t, rt)
    assert t.reason == "cost_model"
    assert_bitwise(got, want)


def test_adp_zero_dims(gpu, port):
    from oracle.oracle import Config

    for (m, n, k) in ((0, 5, 5), (5, 0, 5), (5, 5, 0)):
        a = np.ones((m, k))
        b = np.ones((k, n))
        for mode in (0, 1):
            cfg = gpu.AdpConfig(mode=gpu.AdpMode(mode))
            got, t = gpu.adp_gemm(a, b, config=cfg)
            want, rt = port.adp_gemm(a, b, cfg=Config(mode=mode))
            _cmp_trace(t, rt)
            assert got.shape == (m, n)
            assert_bitwise(got, want)


@pytest.mark.parametrize("ta,tb", [("N", "N"), ("T", "N"), ("N", "T"), ("T", "T")])
def test_dgemm_column_major(gpu, port, ta, tb):
    import torch

    m, n, k = 270, 300, 260
    a = port.gen_uniform_rect(m, k, 1, -1.0, 1.0)
    b = port.gen_uniform_rect(k, n, 2, -1.0, 1.0)
    c = port.gen_uniform_rect(m, n, 3, -1.0, 1.0)
    want, _ = port.adp_gemm(a, b, 0.75, -2.0, c)
    # column-major storage of op(A) / op(B): store X^T row-major for 'N'
    A_store = a.T.copy() if ta == "N" else a.copy()          # col-major m x k == row-major k x m
    B_store = b.T.copy() if tb == "N" else b.copy()
    lda = m if ta == "N" else k
    ldb = k if tb == "N" else n
    dev = torch.device("cuda", 0)
    A = torch.from_numpy(A_store).to(dev)
    B = torch.from_numpy(B_store).to(dev)
    Cm = torch.from_numpy(c.T.copy()).to(dev)  # column-major m x n
    gpu.dgemm(ta, tb, m, n, k, 0.75, A, lda, B, ldb, -2.0, Cm, m)
    got = Cm.cpu().numpy().T
    assert_bitwise(got, want)


def test_adp_target_pairs_close_to_full(gpu, port):
    """PAIRS_TARGET (d_a + d_b <= s) stays within a few FP64 ulps of the
    bitwise-reference Full result on uniform data (north-star bound)."""
    a = port.gen_uniform_rect(256, 512, 1, -1.0, 1.0)
    b = port.gen_uniform_rect(512, 256, 2, -1.0, 1.0)
    full, _ = port.adp_gemm(a, b)
    got, t = gpu.adp_gemm(a, b, config=gpu.AdpConfig(pair_limit=gpu.PAIRS_TARGET))
    assert t.path == "emulated" and t.pair_limit == t.slices
    ulp = np.spacing(np.abs(full))
    assert np.max(np.abs(got - full) / ulp) <= 2.0
