"""MMA-warp cycle accounting (ADPB200_DEBUG=4) of the slice GEMM on rectangular shapes:
how much of a tile's time the tensor pipe waits for the epilogue to drain TMEM.
Usage: ADPB200_DEBUG=4 python tools/tmem_wait_probe.py m n k [s]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_13778_b200 as adp  # noqa: E402
from paper_2511_13778_b200 import grading  # noqa: E402

m, n, k = (int(x) for x in sys.argv[1:4])
s = int(sys.argv[4]) if len(sys.argv) > 4 else 7
A = grading.gen_uniform_rect(m, k, 1, 1.0, 2.0)
B = grading.gen_uniform_rect(k, n, 2, 1.0, 2.0)
C = torch.empty((m, n), dtype=torch.float64, device="cuda")
cfg = adp.AdpConfig(mode=adp.AdpMode.ForceEmulate, forced_slices=s, pair_limit=adp.PAIRS_TARGET)
for _ in range(2):
    adp.adp_gemm(A, B, config=cfg, out=C)
torch.cuda.synchronize()
