"""One geqrf_blocked call (after a warm-up) for ncu launch lists: python tools/qr_one.py m n panel"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_13778_b200 as adp  # noqa: E402
from paper_2511_13778_b200 import grading, qr  # noqa: E402

m, n, panel = (int(x) for x in sys.argv[1:4])
a = grading.gen_uniform_rect(m, n, 0x9802, 0.0, 1.0)
cfg = adp.AdpConfig(min_dim=8)
qr.geqrf_blocked(a, panel, cfg)
torch.cuda.synchronize()
