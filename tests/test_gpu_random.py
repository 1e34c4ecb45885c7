"""GPU: randomized sweep of the drop-in against the CPU oracle (bitwise).

Random shapes (ragged vs the 128 x NB tiles and the 32-byte k-blocks), random
operand transposes, alpha/beta, and operand distributions that stress the
slicing and the exact epilogue: wide exponent spans, exact zeros and -0.0,
subnormals, values near the overflow threshold, whole zero rows/columns."""
import numpy as np
import pytest
import torch

from conftest import assert_bitwise

pytestmark = pytest.mark.gpu


def _operand(rng, rows, cols, kind):
    if kind == "uniform":
        x = rng.uniform(-1.0, 1.0, (rows, cols))
    elif kind == "span":
        x = rng.uniform(1.0, 2.0, (rows, cols)) * np.exp2(rng.integers(-40, 40, (rows, cols)))
        x *= rng.choice([-1.0, 1.0], (rows, cols))
    elif kind == "sparse":
        x = rng.uniform(-1.0, 1.0, (rows, cols)) * (rng.random((rows, cols)) < 0.1)
        x[rng.random((rows, cols)) < 0.05] = -0.0
        if rows > 2:
            x[1, :] = 0.0
    elif kind == "tiny":
        x = rng.uniform(-1.0, 1.0, (rows, cols)) * 2.0 ** -1040  # subnormal region
    else:  # "huge"
        x = rng.uniform(-1.0, 1.0, (rows, cols)) * 2.0 ** 500
    return np.ascontiguousarray(x)


@pytest.mark.parametrize("seed", range(12))
def test_random_adp_gemm_bitwise(gpu, port, seed):
    from oracle.oracle import Config

    rng = np.random.default_rng(1000 + seed)
    m, n, k = (int(v) for v in rng.integers(1, 700, 3))
    ka, kb = rng.choice(["uniform", "span", "sparse", "tiny", "huge"], 2)
    a = _operand(rng, m, k, ka)
    b = _operand(rng, k, n, kb)
    c = rng.uniform(-1.0, 1.0, (m, n))
    alpha = float(rng.choice([1.0, -1.0, 0.75, 3.0]))
    beta = float(rng.choice([0.0, 0.0, 1.0, -0.5]))
    min_dim = int(rng.choice([1, 8, 256]))
    got, t = gpu.adp_gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), alpha, beta,
                          torch.from_numpy(c).cuda() if beta else None, gpu.AdpConfig(min_dim=min_dim))
    want, rt = port.adp_gemm(a, b, alpha, beta, c if beta else None, Config(min_dim=min_dim))
    assert (t.path == "emulated") == (rt["path"] == 0)
    assert (t.slices or -1) == rt["slices"]
    assert_bitwise(got.cpu().numpy(), want)


@pytest.mark.parametrize("seed", range(6))
def test_random_dgemm_trans_bitwise(gpu, seed):
    """Column-major dgemm with every trans combination == the row-major facade on
    the materialised op(A), op(B) (both bitwise the reference)."""
    rng = np.random.default_rng(2000 + seed)
    m, n, k = (int(v) for v in rng.integers(1, 600, 3))
    ta, tb = rng.choice(["N", "T"], 2)
    A = rng.uniform(-1.0, 1.0, (m, k)) * np.exp2(rng.integers(-8, 8, (m, k)))
    B = rng.uniform(-1.0, 1.0, (k, n))
    C = rng.uniform(-1.0, 1.0, (m, n))
    alpha, beta = 1.5, float(rng.choice([0.0, 2.0]))
    cfg = gpu.AdpConfig(min_dim=8)
    want, _ = gpu.adp_gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), alpha, beta,
                           torch.from_numpy(C).cuda() if beta else None, cfg)
    # column-major storage: op(X) = X (N) stored as X^T row-major; op(X) = X^T (T) stored as X row-major
    As = torch.from_numpy(np.ascontiguousarray(A.T if ta == "N" else A)).cuda()
    Bs = torch.from_numpy(np.ascontiguousarray(B.T if tb == "N" else B)).cuda()
    lda = m if ta == "N" else k
    ldb = k if tb == "N" else n
    Cc = torch.from_numpy(np.ascontiguousarray(C.T)).cuda()
    gpu.dgemm(ta, tb, m, n, k, alpha, As, lda, Bs, ldb, beta, Cc, m, cfg)
    torch.cuda.synchronize()
    assert_bitwise(Cc.cpu().numpy().T, want.cpu().numpy())
