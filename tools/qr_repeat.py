"""Repeated geqrf_blocked(4096 x 2048, panel 128) timings (warm-up and variance check)."""
import sys, time, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2511_13778_b200 as adp
from paper_2511_13778_b200 import grading, qr
a = grading.gen_uniform_rect(4096, 2048, 0x9802, 0.0, 1.0)
cfg = adp.AdpConfig(min_dim=8)
for i in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    res = qr.geqrf_blocked(a, 128, cfg)
    torch.cuda.synchronize(); print(i, round(time.perf_counter() - t0, 4), flush=True)
