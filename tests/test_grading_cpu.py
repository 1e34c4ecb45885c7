"""CPU: host logic of the device grading harness (no GPU calls)."""
import math

import numpy as np
import pytest

from paper_2511_13778_b200 import grading


def test_xoshiro_matches_oracle_stream(port):
    for seed in (0, 1, 42, 0xE6, (1 << 64) - 1):
        r = grading.Xoshiro256pp(seed)
        draws = [r() for _ in range(16)]
        u = np.array([((d >> 11) + 0.5) * 2.0 ** -53 for d in draws])
        want = port.gen_uniform_rect(1, 16, seed, 0.0, 1.0)[0]
        assert np.array_equal(u, want)


def test_default_test2_b():
    # grading.cpp:49-54: 511 - ceil(log2 n) - 1
    assert grading.default_test2_b(2) == 509
    assert grading.default_test2_b(1024) == 500
    assert grading.default_test2_b(1025) == 499
    with pytest.raises(ValueError):
        grading.default_test2_b(1)


def test_exact_dot_x_is_exact():
    rng = np.random.default_rng(5)
    x = 1.0 + rng.random(777)
    from fractions import Fraction

    want = float(sum(Fraction(v) * Fraction(v) for v in x))
    assert grading.exact_dot_x(x) == want


def _pt(n, emu, nat, emu_avg=None, nat_avg=None):
    return grading.GradePoint(n=n, emu_max_ratio=emu, emu_avg_ratio=emu if emu_avg is None else emu_avg,
                              nat_max_ratio=nat, nat_avg_ratio=nat if nat_avg is None else nat_avg)


def test_grade_a_check_logic():
    pts = [_pt(n, 0.5, 0.01 * n) for n in (256, 512, 1024, 2048)]
    rep = grading.grade_a_check(pts)
    assert rep.c_calibrated == pytest.approx(0.01)
    assert rep.eq1_pass and rep.slope_pass and rep.grade_a_pass
    assert rep.slope_max == pytest.approx(0.0, abs=1e-12)
    assert rep.native_slope_avg == pytest.approx(1.0)
    # super-linear growth fails the slope gate
    bad = [_pt(n, 1e-6 * n * n, 0.01 * n * n) for n in (256, 512, 1024, 2048)]
    rep = grading.grade_a_check(bad)
    assert not rep.slope_pass and not rep.grade_a_pass
    # an emulated point above c*n fails eq. 1
    pts[2] = _pt(1024, 100.0, 0.01 * 1024)
    assert not grading.grade_a_check(pts).eq1_pass


def test_csv_format():
    row = grading.SweepRow(test="test2", n=256, b=4, mode="auto", esc_bits=9, slices=8, max_err=1e-16,
                           avg_err=0.0001, seed=42)
    assert grading.csv_header() == "test,n,b,mode,target_bits,esc_bits,slices,fallback,max_err,avg_err,seed"
    assert grading.to_csv(row) == "test2,256,4,auto,53,9,8,0,1e-16,1e-04,42"
    row2 = grading.SweepRow(test="uniform", n=512, mode="native", max_err=123.0, avg_err=1.5, seed=7)
    assert grading.to_csv(row2) == "uniform,512,,native,53,,0,0,123,1.5,7"
    assert grading._num(1.2345678901234568e20) == "123456789012345683968"
    assert grading._num(1e22) == "1e+22"
    assert grading._num(-0.0) == "-0"


def test_qr_histogram_csv():
    from paper_2511_13778_b200 import AdpTrace
    from paper_2511_13778_b200.qr import histogram_csv

    tr = [AdpTrace(path="emulated", slices=8), AdpTrace(path="emulated", slices=7),
          AdpTrace(path="emulated", slices=8), AdpTrace(path="native_fallback")]
    assert histogram_csv(tr) == "slices,count\n7,1\n8,2\nnative_fallback,1\n"
