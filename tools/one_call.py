"""One warm-up and one profiled ADP DGEMM call (8192^3 U(1,2), target pairs) for ncu captures:
    ncu --set full --launch-skip <per-call kernels> ... python tools/one_call.py [size]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_13778_b200 as adp  # noqa: E402
from paper_2511_13778_b200 import grading  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
A = grading.gen_uniform_rect(n, n, 1, 1.0, 2.0)
B = grading.gen_uniform_rect(n, n, 2, 1.0, 2.0)
C = torch.empty((n, n), dtype=torch.float64, device="cuda")
cfg = adp.AdpConfig(pair_limit=adp.PAIRS_TARGET)
h = adp.Handle.default(0)
for _ in range(2):
    adp.dgemm("N", "N", n, n, n, 1.0, A, n, B, n, 0.0, C, n, cfg, h)
torch.cuda.synchronize()
print("launches per call:", h.launches() // 2)
