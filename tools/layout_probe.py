"""Timing probe: ADP DGEMM 8192^3 through the dgemm entry with NN (column-major
operands) vs TT (the reference's row-major matrices viewed column-major) vs the
row-major adp_gemm facade; same U(1,2) data. Prints one JSON line."""
import json
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2511_13778_b200 as adp  # noqa: E402
from paper_2511_13778_b200 import grading  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
A = grading.gen_uniform_rect(n, n, 1, 1.0, 2.0)
B = grading.gen_uniform_rect(n, n, 2, 1.0, 2.0)
C = torch.empty((n, n), dtype=torch.float64, device="cuda")
cfg = adp.AdpConfig(pair_limit=adp.PAIRS_TARGET)
h = adp.Handle.default(0)


def t(fn, it=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it


res = {}
res["NN"] = t(lambda: adp.dgemm("N", "N", n, n, n, 1.0, A, n, B, n, 0.0, C, n, cfg, h))
res["TT"] = t(lambda: adp.dgemm("T", "T", n, n, n, 1.0, A, n, B, n, 0.0, C, n, cfg, h))
res["facade"] = t(lambda: adp.adp_gemm(A, B, config=cfg, handle=h, out=C))
h.profile_enable(3)
for lay in ("N", "T"):
    adp.dgemm(lay, lay, n, n, n, 1.0, A, n, B, n, 0.0, C, n, cfg, h)
adp.adp_gemm(A, B, config=cfg, handle=h, out=C)
res["stages"] = h.profile_read()
print(json.dumps(res))
