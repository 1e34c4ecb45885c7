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
