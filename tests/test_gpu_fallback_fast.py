"""The opt-in fast native fallback (adpb200_options.fallback = ADPB200_FALLBACK_FAST):
FP64 tensor cores (DMMA) instead of the reference-order SIMT kernel.

It is not the reference's bits (fused multiply-adds, tiles), so it is checked
against the device double-double oracle with the componentwise bound of any
recursive FP64 dot product,
    |C - AB| <= gamma_k |A||B| + (alpha/beta roundings),  gamma_k = k u / (1 - k u),
on every element, over every transpose / layout the DMMA kernel specialises,
ragged tiles, alpha/beta, and the decision paths that reach the fallback
(ForceNative, a NaN in an operand, ESC too large). The default flavour stays
bitwise the reference (tests/test_gpu_parity.py, test_gpu_grading.py)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

U = 2.0 ** -53


def _bound_check(C, A, B, alpha, beta, C0, k):
    from paper_2511_13778_b200 import grading

    ref, absab = grading.dd_gemm(A, B)
    gamma = k * U / (1 - k * U)
    exact = alpha * ref + (beta * C0 if beta != 0.0 else 0.0)
    # error of sum (gamma_k |A||B|), then alpha (one rounding), beta*c and the add (two more)
    tol = abs(alpha) * gamma * absab + 3 * U * (abs(alpha) * absab + (abs(beta * C0) if beta != 0.0 else 0.0))
    tol = tol + 1e-300
    err = (C - exact).abs()
    worst = float((err / tol).max())
    assert worst <= 1.0, worst
    return worst


def _col_major(x):
    """A column-major copy: the returned tensor is the transpose's storage."""
    return x.t().contiguous()


@pytest.mark.parametrize("ta,tb", [("N", "N"), ("N", "T"), ("T", "N"), ("T", "T")])
@pytest.mark.parametrize("m,n,k", [(256, 256, 256), (300, 257, 129), (1000, 130, 517), (129, 1031, 64)])
def test_fast_fallback_bound_every_layout(gpu, ta, tb, m, n, k):
    g = torch.Generator(device="cuda").manual_seed(m * 7 + n * 3 + k)
    A = torch.rand((m, k), dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    B = torch.rand((k, n), dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    C0 = torch.rand((m, n), dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    alpha, beta = -1.25, 0.5
    # column-major storage of op(A), op(B) as the BLAS call sees them
    Ast = _col_major(A) if ta == "N" else A.contiguous()  # 'N': storage is A^T row-major = A col-major
    Bst = _col_major(B) if tb == "N" else B.contiguous()
    lda = m if ta == "N" else k
    ldb = k if tb == "N" else n
    Cst = _col_major(C0)  # C col-major, ldc = m
    cfg = gpu.AdpConfig(fallback="fast")
    assert gpu.parse_mode("native", cfg)
    gpu.dgemm(ta, tb, m, n, k, alpha, Ast, lda, Bst, ldb, beta, Cst, m, config=cfg)
    C = Cst.t()
    _bound_check(C, A, B, alpha, beta, C0, k)


def test_fast_fallback_after_nan_and_esc_too_large(gpu, grading):
    # a NaN in B: every element of the affected column is NaN, the rest within the bound
    n = 512
    A = grading.gen_uniform_rect(n, n, 1, -1.0, 1.0)
    B = grading.gen_uniform_rect(n, n, 2, -1.0, 1.0)
    B[7, 11] = float("nan")
    C, t = gpu.adp_gemm(A, B, config=gpu.AdpConfig(fallback="fast"))
    assert t.path == "native_fallback" and t.reason == "exceptional_values"
    assert bool(torch.isnan(C[:, 11]).all())
    assert not bool(torch.isnan(C[:, :11]).any()) and not bool(torch.isnan(C[:, 12:]).any())
    B[7, 11] = 0.0
    _bound_check(C[:, :11], A, B[:, :11], 1.0, 0.0, None, n)
    # Test-2 with a huge span: ESC too large -> fallback; the fast flavour stays within the bound
    inst = grading.gen_test2(512, 64, 42)
    C2, t2 = gpu.adp_gemm(inst.lhs, inst.rhs, config=gpu.AdpConfig(fallback="fast"))
    assert t2.path == "native_fallback" and t2.reason == "esc_too_large"
    _bound_check(C2, inst.lhs, inst.rhs, 1.0, 0.0, None, 512)


def test_fast_fallback_matches_reference_flavour_closely(gpu):
    """Both flavours of the same fallback call: the reference flavour is the
    reference's bits; the fast one differs by at most the two dot products'
    rounding bounds (checked elementwise)."""
    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.rand((640, 700), dtype=torch.float64, device="cuda", generator=g)
    B = torch.rand((700, 520), dtype=torch.float64, device="cuda", generator=g)
    slow, ts = gpu.adp_gemm(A, B, config=gpu.AdpConfig(mode=gpu.AdpMode.ForceNative))
    fast, tf = gpu.adp_gemm(A, B, config=gpu.AdpConfig(mode=gpu.AdpMode.ForceNative, fallback="fast"))
    assert ts.path == tf.path == "native_fallback"
    gamma = 700 * U / (1 - 700 * U)
    absab = A.abs() @ B.abs()
    assert bool(((slow - fast).abs() <= 2 * gamma * absab).all())
    assert not torch.equal(slow, fast)  # genuinely a different kernel


def test_fast_fallback_skipped_when_emulating(gpu, port):
    """With the fast flavour selected, an emulated call is unchanged (bitwise the
    reference) — the predicated fallback launch only reads the plan."""
    from oracle.oracle import Config

    a = port.gen_uniform_rect(320, 300, 1, -1.0, 1.0)
    b = port.gen_uniform_rect(300, 288, 2, -1.0, 1.0)
    got, t = gpu.adp_gemm(a, b, config=gpu.AdpConfig(fallback="fast"))
    want, rt = port.adp_gemm(a, b, 1.0, 0.0, None, Config())
    assert t.path == "emulated"
    assert np.array_equal(np.asarray(got).view(np.uint64), want.view(np.uint64))


def test_options_reject_unknown_fallback(gpu):
    with pytest.raises(ValueError):
        gpu.AdpConfig(fallback="bogus").validate()


@pytest.fixture(scope="module")
def grading(gpu):
    from paper_2511_13778_b200 import grading as g

    return g
