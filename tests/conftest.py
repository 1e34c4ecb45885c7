import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "reference: needs oracle/_ref (the reference built from its sources)")


def _ensure_oracle():
    lib = os.path.join(ROOT, "oracle", "liboracle.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True)


@pytest.fixture(scope="session")
def port():
    """The C restatement of the reference (test oracle)."""
    _ensure_oracle()
    from oracle.oracle import Oracle

    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    """The reference itself, built from /root/reference sources into oracle/_ref."""
    from oracle.oracle import Oracle, available

    if not available("reference"):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return Oracle("reference")


@pytest.fixture(scope="session")
def gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2511_13778_b200 as adp

    return adp


def bits(x):
    return np.ascontiguousarray(x, dtype=np.float64).view(np.uint64)


def assert_bitwise(got, want, nan_equiv=True):
    g, w = bits(got), bits(want)
    if nan_equiv:
        gn, wn = np.isnan(np.asarray(got)), np.isnan(np.asarray(want))
        assert np.array_equal(gn, wn), "NaN positions differ"
        mask = ~gn
        diff = np.nonzero(g[mask] != w[mask])[0]
    else:
        diff = np.nonzero(g.ravel() != w.ravel())[0]
    assert diff.size == 0, f"{diff.size} of {g.size} elements differ (first at flat index {diff[:5]})"
