"""GPU: the QR caller (proj/src/qr.cpp) — blocked Householder QR whose three
trailing-update products per panel run through the ADP GEMM — against the
reference built from its sources: factors, T blocks, every trace, thin Q and
the residual / orthogonality numbers must be BITWISE the reference's
(the panel work runs in the reference's operation order on the device)."""
import numpy as np
import pytest
import torch

from conftest import assert_bitwise

pytestmark = pytest.mark.gpu

REASONS = ["ok", "forced", "exceptional_values", "esc_too_large", "too_small", "cost_model"]


@pytest.fixture(scope="module")
def qrmod(gpu):
    from paper_2511_13778_b200 import qr

    return qr


def _check(gpu, qrmod, ref, a, panel, cfg_kwargs):
    from oracle.oracle import Config

    cfg = gpu.AdpConfig(**cfg_kwargs)
    res = qrmod.geqrf_blocked(a, panel, cfg)
    fac, t, tr, q, acc = ref.qr(a, panel, Config(**{k: int(v) for k, v in cfg_kwargs.items()}))
    assert_bitwise(res.factors.cpu().numpy(), fac, nan_equiv=False)
    m, n = a.shape
    assert len(res.t_blocks) == (n + panel - 1) // panel
    for p, tb in enumerate(res.t_blocks):
        pw = tb.shape[0]
        want = t[p * panel * panel: p * panel * panel + pw * pw].reshape(pw, pw)
        assert_bitwise(tb.cpu().numpy(), want, nan_equiv=False)
    assert len(res.traces) == 3 * len(res.t_blocks) == len(tr)
    for got, w in zip(res.traces, tr):
        assert (got.path == "emulated") == (w[0] == 0)
        assert got.reason == REASONS[w[1]]
        assert (got.esc_bits if got.esc_bits is not None else -1) == w[2]
        assert (got.slices if got.path == "emulated" else -1) == w[3]
        assert (got.m, got.n, got.k) == (w[4], w[5], w[6])
    qg = qrmod.materialize_q(res)
    assert_bitwise(qg.cpu().numpy(), q, nan_equiv=False)
    accg = qrmod.qr_residual(a, res)
    assert (accg.residual, accg.orthogonality) == acc
    return res, accg


def test_identity(gpu, qrmod, ref):
    eye = np.eye(32)
    res, acc = _check(gpu, qrmod, ref, eye, 8, {})
    assert np.array_equal(res.factors.cpu().numpy(), eye)
    assert acc.residual == 0.0 and acc.orthogonality == 0.0


def test_sign_reflector(gpu, qrmod, ref):
    res, acc = _check(gpu, qrmod, ref, np.array([[-3.0]]), 4, {})
    assert res.factors.item() == 3.0
    assert qrmod.materialize_q(res).item() == -1.0


def test_zero_column(gpu, qrmod, ref, port):
    a = port.gen_uniform_rect(8, 3, 5, -1.0, 1.0)
    a[:, 1] = 0.0
    res, _ = _check(gpu, qrmod, ref, a, 2, {})
    assert res.factors[1, 1].item() == 0.0


@pytest.mark.parametrize("cfg", [{"mode": 2}, {"min_dim": 8}, {}])
def test_square_64(gpu, qrmod, ref, port, cfg):
    a = port.gen_uniform_rect(64, 64, 99, -1.0, 1.0)
    res, acc = _check(gpu, qrmod, ref, a, 16, cfg)
    assert acc.residual <= 100.0 * 64 * 2.0 ** -52
    if cfg.get("min_dim") == 8:
        assert sum(t.path == "emulated" for t in res.traces) >= 6


def test_ragged_tail(gpu, qrmod, ref, port):
    a = port.gen_uniform_rect(100, 40, 17, 0.0, 1.0)
    res, _ = _check(gpu, qrmod, ref, a, 12, {"min_dim": 8})
    assert [tb.shape[0] for tb in res.t_blocks] == [12, 12, 12, 4]
    for t in res.traces[9:]:
        assert t.n == 0 and t.path == "native_fallback" and t.reason == "too_small"


@pytest.mark.parametrize("m,n,seed", [(256, 128, 0x9800), (512, 512, 0x9801)])
def test_acceptance_criterion_8(gpu, qrmod, ref, port, m, n, seed):
    """acceptance_main.cpp:378-420: panel 32, native vs emulating (min_dim 8)."""
    a = port.gen_uniform_rect(m, n, seed, 0.0, 1.0)
    _, acc_nat = _check(gpu, qrmod, ref, a, 32, {"mode": 2})
    res, acc_emu = _check(gpu, qrmod, ref, a, 32, {"min_dim": 8})
    bound = 100.0 * max(m, n) * 2.0 ** -52
    assert acc_emu.residual <= 10 * acc_nat.residual and acc_emu.residual <= bound and acc_nat.residual <= bound
    hist = {}
    for t in res.traces:
        if t.path == "emulated":
            hist[t.slices] = hist.get(t.slices, 0) + 1
    assert hist and hist[min(hist)] * 2 >= sum(hist.values())
    csv = qrmod.histogram_csv(res.traces)
    assert csv.startswith("slices,count\n") and csv.rstrip().split("\n")[-1].startswith("native_fallback,")


def test_contracts(gpu, qrmod):
    with pytest.raises(ValueError):
        qrmod.geqrf_blocked(np.zeros((3, 4)), 2)   # m < n
    with pytest.raises(ValueError):
        qrmod.geqrf_blocked(np.zeros((4, 4)), 0)   # panel 0
    with pytest.raises(ValueError):
        qrmod.geqrf_blocked(np.zeros((4, 4)), 2, gpu.AdpConfig(max_slices=3))
