"""The device path is stream-ordered with no host synchronisation, so once a
handle's workspace is sized (one warm-up call) adpb200_dgemm captures into a
CUDA graph as is: the replayed graph must reproduce the eager result bitwise,
including the ADP decision taken on the device, and follow new operand values
written into the captured buffers (decision re-taken at replay)."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,lo", [(512, 1.0), (1024, -1.0), (768, 1.0)])
def test_dgemm_graph_replay_bitwise(gpu, n, lo):
    from paper_2511_13778_b200 import grading

    A = grading.gen_uniform_rect(n, n, 1, lo, 2.0 if lo > 0 else 1.0)
    B = grading.gen_uniform_rect(n, n, 2, lo, 2.0 if lo > 0 else 1.0)
    C, Cg = (torch.empty((n, n), dtype=torch.float64, device="cuda") for _ in range(2))
    cfg = gpu.AdpConfig(pair_limit=gpu.PAIRS_TARGET)
    h = gpu.Handle(0)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        gpu.dgemm("N", "N", n, n, n, 1.0, A, n, B, n, 0.0, Cg, n, cfg, h)  # sizes the workspace
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        gpu.dgemm("N", "N", n, n, n, 1.0, A, n, B, n, 0.0, Cg, n, cfg, h)
    for trial in range(2):
        if trial:  # new data in the captured buffers: a different ESC / slice count at replay
            A.copy_(grading.gen_uniform_rect(n, n, 7, -1.0, 1.0) if lo > 0 else
                    grading.gen_uniform_rect(n, n, 7, 1.0, 2.0))
        gpu.dgemm("N", "N", n, n, n, 1.0, A, n, B, n, 0.0, C, n, cfg, h)
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(C.view(torch.int64), Cg.view(torch.int64))


def test_graphed_dgemm_helper(gpu):
    """adp.GraphedDgemm: capture once, replay; each replay follows the buffers' data."""
    import torch

    from paper_2511_13778_b200 import grading

    n = 640
    A = grading.gen_uniform_rect(n, n, 3, 1.0, 2.0)
    B = grading.gen_uniform_rect(n, n, 4, 1.0, 2.0)
    C, Cg = (torch.empty((n, n), dtype=torch.float64, device="cuda") for _ in range(2))
    cfg = gpu.AdpConfig()
    g = gpu.GraphedDgemm("N", "T", n, n, n, 0.5, A, n, B, n, 0.0, Cg, n, cfg)
    for seed in (5, 6):
        A.copy_(grading.gen_uniform_rect(n, n, seed, -1.0, 1.0))
        g()
        gpu.dgemm("N", "T", n, n, n, 0.5, A, n, B, n, 0.0, C, n, cfg)
        torch.cuda.synchronize()
        assert torch.equal(C.view(torch.int64), Cg.view(torch.int64))


_PDL_SCRIPT = r"""
import hashlib, sys, torch
sys.path.insert(0, sys.argv[1])
import paper_2511_13778_b200 as adp
from paper_2511_13778_b200 import grading
out = []
for (m, n, k, lo, ff) in ((384, 320, 1000, -1.0, None), (512, 512, 512, 1.0, None), (300, 200, 260, 1.0, "fast")):
    A = grading.gen_uniform_rect(k, m, 3, lo, 2.0 if lo > 0 else 1.0)
    B = grading.gen_uniform_rect(n, k, 4, lo, 2.0 if lo > 0 else 1.0)
    C = torch.empty((n, m), dtype=torch.float64, device="cuda")
    cfg = adp.AdpConfig(mode=adp.AdpMode.ForceNative, fallback=ff) if ff else adp.AdpConfig()
    h = adp.Handle(0)
    for _ in range(3):  # repeated calls: the chain of one call follows the previous call's kernels
        adp.dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m, cfg, h)
    torch.cuda.synchronize()
    out.append(hashlib.sha256(C.cpu().numpy().tobytes()).hexdigest())
print(" ".join(out))
"""


def test_programmatic_dependent_launch_bitwise():
    """The chain kernels launched with programmatic dependent launch (default for small
    calls) give the same bits as plain stream serialisation (ADPB200_PDL=0)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for pdl in ("1", "0"):
        env = dict(os.environ, ADPB200_PDL=pdl)
        res[pdl] = subprocess.run([sys.executable, "-c", _PDL_SCRIPT, root], env=env, capture_output=True,
                                  text=True, check=True, timeout=600).stdout.strip()
    assert res["1"] and res["1"] == res["0"]
