"""Per-call time of the device-resident ADP DGEMM (8192^3, target pairs): U(1,2) and U[-1,1]."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_13778_b200 as adp  # noqa: E402
from paper_2511_13778_b200 import grading  # noqa: E402

n = 8192
h = adp.Handle.default(0)
C = torch.empty((n, n), dtype=torch.float64, device="cuda")
cfg = adp.AdpConfig(pair_limit=adp.PAIRS_TARGET)
out = {"speculation": os.environ.get("ADPB200_NO_SPECULATION") is None}
for lo in (1.0, -1.0):
    A = grading.gen_uniform_rect(n, n, 1, lo, 2.0 if lo > 0 else 1.0)
    B = grading.gen_uniform_rect(n, n, 2, lo, 2.0 if lo > 0 else 1.0)
    for _ in range(3):
        adp.dgemm("N", "N", n, n, n, 1.0, A, n, B, n, 0.0, C, n, cfg, h)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        adp.dgemm("N", "N", n, n, n, 1.0, A, n, B, n, 0.0, C, n, cfg, h)
    e1.record()
    torch.cuda.synchronize()
    out[f"lo={lo}"] = e0.elapsed_time(e1) / 20
print(json.dumps(out))
