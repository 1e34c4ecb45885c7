"""adp.dgemm captured in a CUDA graph (the pipeline is stream-ordered with no host
synchronisation, so it captures as is once the handle's workspace is sized):
replay == eager bitwise, and the per-call time of graph replay vs eager launches.
Usage: python tools/graph_probe.py [n ...]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_13778_b200 as adp  # noqa: E402
from paper_2511_13778_b200 import grading  # noqa: E402

for n in [int(x) for x in sys.argv[1:]] or [512, 1024, 2048]:
    A = grading.gen_uniform_rect(n, n, 1, 1.0, 2.0)
    B = grading.gen_uniform_rect(n, n, 2, 1.0, 2.0)
    C = torch.empty((n, n), dtype=torch.float64, device="cuda")
    Cg = torch.empty_like(C)
    cfg = adp.AdpConfig(pair_limit=adp.PAIRS_TARGET)
    h = adp.Handle(0)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):  # sizes the workspace, encodes the TMA maps
            adp.dgemm("N", "N", n, n, n, 1.0, A, n, B, n, 0.0, Cg, n, cfg, h)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        adp.dgemm("N", "N", n, n, n, 1.0, A, n, B, n, 0.0, Cg, n, cfg, h)
    adp.dgemm("N", "N", n, n, n, 1.0, A, n, B, n, 0.0, C, n, cfg, h)
    g.replay()
    torch.cuda.synchronize()
    same = torch.equal(C.view(torch.int64), Cg.view(torch.int64))
    it = 200 if n <= 1024 else 50

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(it):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / it

    eager = timed(lambda: adp.dgemm("N", "N", n, n, n, 1.0, A, n, B, n, 0.0, C, n, cfg, h))
    graph = timed(g.replay)
    print(json.dumps({"n": n, "bitwise_equal": same, "eager_ms": eager, "graph_ms": graph,
                      "graph_tflops": 2.0 * n ** 3 / graph / 1e9}), flush=True)
