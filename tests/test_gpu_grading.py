"""GPU: the BLAS grading inputs (BASELINE config 3) — the reference's Test-2
exponent-span sweep (proj/src/grading.cpp:13-47, acceptance criterion 4,
proj/tests/acceptance/acceptance_main.cpp:224-247), NaN/Inf injection
(criterion 6, :269-334) and terminal overflow (test_igemm.cpp:238-250).

Every ADP decision (ESC bits, slice count, fallback reason) and every output
bit is checked against the oracle; the Test-2 diagonal, whose exact value is
x^T x, bounds the error like the reference's acceptance gate (<= 32 eps)."""
import numpy as np
import pytest

from conftest import assert_bitwise

pytestmark = pytest.mark.gpu

EPS = 2.0 ** -52
REASONS = ["ok", "forced", "exceptional_values", "esc_too_large", "too_small", "cost_model"]


@pytest.mark.parametrize("b_span", [0, 1, 2, 4, 8, 16, 32, 40, 44, 48, 64, 128, 500])
def test_test2_sweep(gpu, port, b_span):
    from oracle.oracle import Config

    n = 256
    lhs, rhs = port.gen_test2(n, b_span, 42)
    got, t = gpu.adp_gemm(lhs, rhs)
    want, rt = port.adp_gemm(lhs, rhs, cfg=Config())
    assert t.esc_bits == rt["esc_bits"] == 2 * b_span + 1     # esc = 2b + 1 (SURVEY finding 6)
    assert t.reason == REASONS[rt["reason"]]
    assert (t.slices or -1) == rt["slices"]
    expect_fallback = (53 + 2 * b_span + 1 + 2 + 7) // 8 > 18  # esc_too_large from b = 48
    assert (t.path == "native_fallback") == expect_fallback
    assert_bitwise(got, want, nan_equiv=False)
    # the diagonal is x^T x exactly (the two-sided scaling cancels): error bound of the acceptance gate
    exact_diag = port.exact_gemm(lhs[:1, :], rhs[:, :1])[0, 0]
    diag = np.diag(got)
    rel = np.max(np.abs(diag - exact_diag) / abs(exact_diag))
    assert rel <= 32 * EPS, rel


def test_forced_7_slices_degrade_like_the_reference(gpu, port):
    """Acceptance criterion 4's negative control: forced 7 slices on wide
    spans loses accuracy exactly as the reference does (bitwise equal)."""
    from oracle.oracle import Config

    lhs, rhs = port.gen_test2(256, 16, 42)
    cfg = gpu.AdpConfig()
    assert gpu.parse_mode("emulate:7", cfg)
    got, t = gpu.adp_gemm(lhs, rhs, config=cfg)
    want, _ = port.adp_gemm(lhs, rhs, cfg=Config(mode=1, forced_slices=7))
    assert t.path == "emulated" and t.slices == 7 and t.reason == "forced"
    assert_bitwise(got, want, nan_equiv=False)


def test_nan_inf_injection(gpu, port):
    """Criterion 6: NaN/Inf (incl. signalling-payload NaNs) anywhere -> native
    fallback, same bits or both NaN; -0.0 keeps emulating."""
    from oracle.oracle import Config

    rng = np.random.default_rng(0xE6)
    specials = [np.nan, np.inf, -np.inf, None]
    for case in range(12):
        a = port.gen_uniform_rect(256, 256, 100 + case, -1.0, 1.0)
        b = port.gen_uniform_rect(256, 260, 200 + case, -1.0, 1.0)
        tgt = a if case % 2 == 0 else b
        i, jj = rng.integers(0, tgt.shape[0]), rng.integers(0, tgt.shape[1])
        sp = specials[case % 4]
        if sp is None:
            tgt.view(np.uint64)[i, jj] = np.uint64(0x7FF8000000000000 | int(rng.integers(1, 1 << 50)))
        else:
            tgt[i, jj] = sp
        got, t = gpu.adp_gemm(a, b)
        want, rt = port.adp_gemm(a, b, cfg=Config())
        assert t.reason == "exceptional_values" and rt["reason"] == 2
        assert t.scan_a == rt["scan_a"] and t.scan_b == rt["scan_b"]
        assert_bitwise(got, want)


def test_terminal_overflow_is_not_a_fallback(gpu, port):
    a = np.full((256, 256), 2.0 ** 600)
    b = np.full((256, 256), 2.0 ** 600)
    a[0, :] = -(2.0 ** 600)
    got, t = gpu.adp_gemm(a, b)
    want, _ = port.adp_gemm(a, b)
    assert t.path == "emulated"
    assert np.isinf(got).all()
    assert_bitwise(got, want, nan_equiv=False)
