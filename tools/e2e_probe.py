"""e2e timing of adpb200_dgemm_host (pinned host buffers, 8192^3 U(1,2), target pairs)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_13778_b200 as adp  # noqa: E402
from paper_2511_13778_b200 import grading  # noqa: E402

n = 8192
A = grading.gen_uniform_rect(n, n, 1, 1.0, 2.0).cpu().pin_memory()
B = grading.gen_uniform_rect(n, n, 2, 1.0, 2.0).cpu().pin_memory()
C = torch.empty((n, n), dtype=torch.float64).pin_memory()
cfg = adp.AdpConfig(pair_limit=adp.PAIRS_TARGET)
h = adp.Handle.default(0)
for _ in range(2):
    adp.dgemm_host("N", "N", n, n, n, 1.0, A, n, B, n, 0.0, C, n, cfg, h)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(8):
    adp.dgemm_host("N", "N", n, n, n, 1.0, A, n, B, n, 0.0, C, n, cfg, h)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 8
print(json.dumps({"e2e_ms": ms, "e2e_tflops": 2.0 * n ** 3 / ms / 1e9}))
