"""PCIe copy rates on the box (pinned host memory): H2D 1 GiB, D2H 0.5 GiB, and
both at once on two streams — the floor under the e2e number."""
import json

import torch

n = 8192
h_in = torch.empty((2 * n, n), dtype=torch.float64).pin_memory()
h_out = torch.empty((n, n), dtype=torch.float64).pin_memory()
d_in = torch.empty((2 * n, n), dtype=torch.float64, device="cuda")
d_out = torch.empty((n, n), dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, it=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it


def both():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


h2d = t(lambda: d_in.copy_(h_in, non_blocking=True))
d2h = t(lambda: h_out.copy_(d_out, non_blocking=True))
bo = t(both)
print(json.dumps({"h2d_1GiB_ms": h2d, "h2d_GBs": 2 * n * n * 8 / h2d / 1e6, "d2h_512MiB_ms": d2h,
                  "d2h_GBs": n * n * 8 / d2h / 1e6, "both_concurrent_ms": bo}))
