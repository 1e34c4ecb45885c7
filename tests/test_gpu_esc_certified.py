"""Certified ESC on the GPU (adpb200_options.esc_method = ADPB200_ESC_CERTIFIED):
the indicator planes + INT8 count GEMM must reproduce the numpy restatement
(oracle.esc_certified) exactly, the decision must follow the reference's
decide() on that ESC, and C must equal the reference-order emulated_gemm at
the decided s bitwise — on the device path, the streamed host path and at
4096^3, where U[-1,1] drops from the coarsened s = 8 to s = 7 with the
accuracy of a double-double oracle kept."""
import numpy as np
import pytest

from conftest import assert_bitwise
from oracle.oracle import Config, esc_certified

pytestmark = pytest.mark.gpu

PATHS = ("emulated", "native_fallback")


def _make(name, m, k, n, seed):
    rng = np.random.default_rng(seed)
    if name == "u12":
        return rng.uniform(1, 2, (m, k)), rng.uniform(1, 2, (k, n))
    a, b = rng.uniform(-1, 1, (m, k)), rng.uniform(-1, 1, (k, n))
    if name == "wide":
        a = a * np.exp2(rng.integers(-40, 40, (m, k)))
    elif name == "zero_col":
        b[:, 7] = 0.0
    elif name == "sparse":
        a = a * (rng.random((m, k)) < 0.05)
    elif name == "subnormal":
        a = a * 2.0 ** -1060
    elif name == "late_max":
        a[5, :600] *= 1e-3  # row 5's large entries all lie past the 512-position window
    return a, b


CASES = [("u11", 256, 300, 260, 53), ("u11", 300, 1000, 512, 53), ("u12", 512, 256, 300, 53),
         ("wide", 300, 400, 280, 53), ("zero_col", 256, 512, 256, 53), ("sparse", 260, 700, 300, 53),
         ("subnormal", 256, 260, 256, 53), ("u11", 256, 300, 260, 50), ("u11", 256, 300, 260, 54),
         ("u11", 1000, 640, 600, 53), ("late_max", 256, 1000, 300, 53), ("wide", 300, 400, 280, 54),
         ("wide", 300, 600, 280, 50)]


@pytest.mark.parametrize("name,m,k,n,tb", CASES)
def test_certified_decision_and_bits(gpu, port, name, m, k, n, tb):
    import torch

    a, b = _make(name, m, k, n, m + k + n)
    coarse = port.esc_coarsened(a, b, 256, tb)[0]
    want_esc = esc_certified(a, b, coarse, tb)
    if name == "late_max":
        assert want_esc == coarse and esc_certified(a, b, coarse, tb, window=k) == 1
    if name == "wide" and tb == 53:
        assert want_esc == 9 < coarse  # the second certificate level
    path, _, s, _, _, _ = port.decide(0, 0, m, n, k, want_esc, Config(target_bits=tb))
    cfg = gpu.AdpConfig(target_bits=tb, esc_method="certified")
    # device path (CUDA tensors) and the streamed host path (numpy)
    got_d, td = gpu.adp_gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), config=cfg)
    got_h, th = gpu.adp_gemm(a, b, config=cfg)
    for t in (td, th):
        assert t.esc_bits == want_esc, (t.esc_bits, want_esc, coarse)
        assert t.path == PATHS[path]
        if t.path == "emulated":
            assert t.slices == s
    want = port.emulated_gemm(a, b, s) if path == 0 else port.native_gemm(a, b)
    assert_bitwise(got_d.cpu().numpy(), want, nan_equiv=False)
    assert_bitwise(got_h, want, nan_equiv=False)
    # the default (coarsened) method is untouched
    _, tc_ = gpu.adp_gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), config=gpu.AdpConfig(target_bits=tb))
    assert tc_.esc_bits == coarse


def test_certified_4096_u11_accuracy_and_sampled_bits(gpu, port):
    import torch

    from paper_2511_13778_b200 import grading

    n = 4096
    A = grading.gen_uniform_rect(n, n, 1, -1.0, 1.0)
    B = grading.gen_uniform_rect(n, n, 2, -1.0, 1.0)
    Cc, tc_ = gpu.adp_gemm(A, B)
    Cx, tx = gpu.adp_gemm(A, B, config=gpu.AdpConfig(esc_method="certified"))
    assert tc_.slices == 8 and tc_.esc_bits > 1
    assert tx.path == "emulated" and tx.esc_bits == 1 and tx.slices == 7
    ref, absab = grading.dd_gemm(A, B)
    ec = grading.error_report(Cc, ref, absab=absab)
    ex = grading.error_report(Cx, ref, absab=absab)
    # both within a couple of units of 2^-52 |A||B| (componentwise bound of the method)
    assert ex.max_ratio < 4.0 and ec.max_ratio < 4.0, (ex, ec)
    rows = np.array([0, 1, 127, 128, 2047, 4095])
    cols = np.array([0, 5, 63, 64, 1000, 4095])
    want = port.emulated_gemm(A[rows].cpu().numpy(), B[:, cols].cpu().numpy(), 7)
    assert_bitwise(Cx[rows][:, cols].cpu().numpy(), want, nan_equiv=False)
    torch.cuda.synchronize()


@pytest.mark.parametrize("name,m,k,n", [("u11", 200, 300, 150), ("u12", 64, 700, 80), ("wide", 130, 257, 65),
                                        ("zero_col", 100, 100, 100), ("sparse", 150, 400, 120),
                                        ("subnormal", 70, 90, 50), ("u11", 1, 1, 1), ("u11", 33, 0, 17)])
def test_device_esc_exact_matches_reference(gpu, port, name, m, k, n):
    """esc_exact (esc.cpp:61-87) as a device stage (DPX max-plus): the same
    EscReport as the C restatement, and the certified ESC never below it."""
    a, b = _make(name, m, max(k, 1), n, 7 + m)
    a, b = a[:, :k], b[:k, :]
    for tb in (53, 50):
        assert gpu.esc_exact(a, b, tb) == tuple(port.esc_exact(a, b, tb))
    if k:
        coarse = port.esc_coarsened(a, b, 256, 53)[0]
        assert gpu.esc_exact(a, b)[0] <= esc_certified(a, b, coarse, 53) or name in ("zero_col", "sparse")
    bad = a.copy()
    if bad.size:
        bad.flat[0] = np.nan
        with pytest.raises(ValueError):
            gpu.esc_exact(bad, b)


def test_certified_bracket_at_2048(gpu):
    """esc_exact <= certified <= coarsened on the device at 2048^3 (U[-1,1], U(1,2), wide)."""
    import torch

    for name in ("u11", "u12", "wide"):
        a, b = _make(name, 2048, 2048, 2048, 11)
        A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        exact = gpu.esc_exact(A, B)[0]
        _, tc_ = gpu.adp_gemm(A, B, config=gpu.AdpConfig(mode=gpu.AdpMode.ForceEmulate, guardrails_forced=True))
        _, tx = gpu.adp_gemm(A, B, config=gpu.AdpConfig(mode=gpu.AdpMode.ForceEmulate, guardrails_forced=True,
                                                        esc_method="certified"))
        assert exact <= tx.esc_bits <= tc_.esc_bits, (name, exact, tx.esc_bits, tc_.esc_bits)


@pytest.mark.parametrize("ta,tb", [("N", "N"), ("T", "N"), ("N", "T")])
def test_certified_streamed_dgemm_host_matches_device(gpu, ta, tb):
    """adpb200_dgemm_host (B streamed in column chunks, speculated s) with the
    certified ESC: the same decision and bits as the device-resident dgemm, with
    alpha / beta, across the speculation hit / miss sequence of one handle."""
    import torch

    from paper_2511_13778_b200 import Handle

    h = Handle(0)
    m, n, k = 900, 1280, 700
    g = torch.Generator()
    g.manual_seed(5)
    cfg = gpu.AdpConfig(pair_limit=gpu.PAIRS_TARGET, esc_method="certified")
    for lo, hi, beta in ((-1.0, 1.0, 0.0), (-1.0, 1.0, 0.5), (1.0, 2.0, 0.0), (-1.0, 1.0, -2.0)):
        Ast = torch.rand((k, m) if ta == "N" else (m, k), generator=g, dtype=torch.float64) * (hi - lo) + lo
        Bst = torch.rand((n, k) if tb == "N" else (k, n), generator=g, dtype=torch.float64) * (hi - lo) + lo
        Ct = torch.rand((n, m), generator=g, dtype=torch.float64)
        lda = m if ta == "N" else k
        ldb = k if tb == "N" else n
        A_h, B_h, C_h = Ast.pin_memory(), Bst.pin_memory(), Ct.clone().pin_memory()
        tr = gpu.dgemm_host(ta, tb, m, n, k, -0.75, A_h, lda, B_h, ldb, beta, C_h, m, cfg, h)
        Cd = Ct.cuda()
        gpu.dgemm(ta, tb, m, n, k, -0.75, Ast.cuda(), lda, Bst.cuda(), ldb, beta, Cd, m, cfg, h)
        torch.cuda.synchronize()
        assert tr.path == "emulated" and tr.slices == 7  # U[-1,1] certified down to s0 = 7
        assert torch.equal(C_h.view(torch.int64), Cd.cpu().view(torch.int64))


@pytest.mark.parametrize("block_len", [16, 100, 1024])
def test_certified_with_other_esc_block_lengths(gpu, port, block_len):
    """The certificate composes with any esc_block_len: the device decision equals
    the restatement applied to the reference's coarsened ESC at that block length."""
    import torch

    for name in ("u11", "wide", "zero_col"):
        a, b = _make(name, 280, 900, 300, block_len)
        coarse = port.esc_coarsened(a, b, block_len, 53)[0]
        want = esc_certified(a, b, coarse, 53)
        cfg = gpu.AdpConfig(esc_method="certified", esc_block_len=block_len)
        got, t = gpu.adp_gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), config=cfg)
        assert t.esc_bits == want, (name, t.esc_bits, want, coarse)
        if t.path == "emulated":
            assert_bitwise(got.cpu().numpy(), port.emulated_gemm(a, b, t.slices), nan_equiv=False)
