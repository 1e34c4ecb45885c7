"""Certified ESC (adpb200_options.esc_method = 1), CPU side: the numpy
restatement in oracle/oracle.py is bracketed by the reference's own ESCs,
esc_exact <= certified <= esc_coarsened (esc.cpp:61-117), and the option
round-trips through the C ABI's validation."""
import numpy as np
import pytest

from oracle.oracle import certify_delta, esc_certified, exponent_field, NEG_SENTINEL


def _cases(port):
    rng = np.random.default_rng(5)
    out = []
    for m, k, n in ((40, 300, 33), (96, 700, 64), (17, 1029, 50)):
        out.append(("u11", rng.uniform(-1, 1, (m, k)), rng.uniform(-1, 1, (k, n))))
        out.append(("u12", rng.uniform(1, 2, (m, k)), rng.uniform(1, 2, (k, n))))
        wide = rng.uniform(-1, 1, (m, k)) * np.exp2(rng.integers(-40, 40, (m, k)))
        out.append(("wide", wide, rng.uniform(-1, 1, (k, n))))
        z = rng.uniform(-1, 1, (m, k))
        z[3] = 0.0  # an all-zero row: structurally zero dots, no certificate
        out.append(("zero_row", z, rng.uniform(-1, 1, (k, n))))
        sp = rng.uniform(-1, 1, (m, k)) * (rng.random((m, k)) < 0.02)
        out.append(("sparse", sp, rng.uniform(-1, 1, (k, n)) * (rng.random((k, n)) < 0.02)))
        sub = rng.uniform(-1, 1, (m, k)) * 2.0 ** -1060  # subnormals
        out.append(("subnormal", sub, rng.uniform(-1, 1, (k, n))))
    t = port.gen_test2(256, 4, 42)
    out.append(("test2", t[0], t[1]) if isinstance(t, tuple) else ("test2", t.lhs, t.rhs))
    return out


def test_exponent_field_matches_reference_definition():
    v = np.array([[1.0, 0.75, -2.0, 0.0, 2.0 ** -1074, 2.0 ** -1022, np.inf, np.nan, -0.0, 3.0]])
    e = exponent_field(v)[0]
    assert e.tolist() == [0, -1, 1, NEG_SENTINEL, -1074, -1022, NEG_SENTINEL, NEG_SENTINEL, NEG_SENTINEL, 1]


@pytest.mark.parametrize("tb", [53, 50, 45, 60])
def test_certified_bracketed_by_exact_and_coarsened(port, tb):
    for name, a, b in _cases(port):
        coarse = port.esc_coarsened(a, b, 256, tb)[0]
        exact = port.esc_exact(a, b, tb)[0]
        cert = esc_certified(a, b, coarse, tb)
        s0 = (tb + 2 + 7) // 8
        e0 = 8 * s0 - tb - 2
        levels = [2 * certify_delta(tb, lv) + 1 for lv in (0, 1) if certify_delta(tb, lv) >= 0]
        assert cert == coarse or cert in levels, name
        assert cert <= coarse, name
        if name not in ("zero_row", "sparse"):
            # (the reference's coarsened ESC itself can undercut esc_exact when zeros
            # line up; the certificate never applies there)
            assert exact <= cert, (name, exact, cert)
        if name in ("u11", "u12") and e0 >= 1:
            assert cert <= 2 * ((e0 - 1) // 2) + 1, (name, cert)  # U[-1,1] drops to s0
            assert port.required_slices(tb, cert) == s0
        if name in ("zero_row",):
            assert cert == coarse
        if name == "wide" and tb == 53:
            assert cert == 9 < coarse  # level 1: s0 + 1 = 8 slices where the coarsened ESC asks 9+


def test_certified_against_the_built_reference(ref):
    """Same bracket with esc_exact / esc_coarsened from the reference build."""
    rng = np.random.default_rng(9)
    for lo in (-1.0, 1.0):
        a = rng.uniform(lo, 2.0 if lo > 0 else 1.0, (64, 512))
        b = rng.uniform(lo, 2.0 if lo > 0 else 1.0, (512, 48))
        coarse = ref.esc_coarsened(a, b, 256, 53)[0]
        exact = ref.esc_exact(a, b, 53)[0]
        cert = esc_certified(a, b, coarse, 53)
        assert exact <= cert <= coarse and cert == 1


def test_esc_method_option_validation():
    pytest.importorskip("torch")
    import paper_2511_13778_b200 as adp

    adp.AdpConfig(esc_method="certified").validate()
    adp.AdpConfig().validate()
    with pytest.raises(ValueError):
        adp.AdpConfig(esc_method="exact").validate()
