"""Slice-GEMM stage timing at 8192^3 (U(1,2), s = 7, pairs d_a+d_b <= s) for
the ADPB200_DEBUG diagnostics (1: skip MMAs, 2: skip epilogue math, 4: cycle
counters). Usage: ADPB200_DEBUG=<mode> python tools/gemm_probe.py [size] [lo]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_13778_b200 as adp  # noqa: E402
from paper_2511_13778_b200 import grading  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
lo = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
A = grading.gen_uniform_rect(n, n, 1, lo, 2.0 if lo > 0 else 1.0)
B = grading.gen_uniform_rect(n, n, 2, lo, 2.0 if lo > 0 else 1.0)
C = torch.empty((n, n), dtype=torch.float64, device="cuda")
cfg = adp.AdpConfig(pair_limit=adp.PAIRS_TARGET)
h = adp.Handle.default(0)
for _ in range(3):
    adp.dgemm("N", "N", n, n, n, 1.0, A, n, B, n, 0.0, C, n, cfg, h)
torch.cuda.synchronize()
h.profile_enable(10)
for _ in range(10):
    adp.dgemm("N", "N", n, n, n, 1.0, A, n, B, n, 0.0, C, n, cfg, h)
st = h.profile_read()
print(json.dumps({"debug": os.environ.get("ADPB200_DEBUG", "0"), "n": n,
                  "gemm_ms": sorted(c["gemm"] for c in st)[len(st) // 2],
                  "slice_ms": sorted(c["slice"] for c in st)[len(st) // 2],
                  "esc_ms": sorted(c["esc"] for c in st)[len(st) // 2],
                  "stats_ms": sorted(c["stats"] for c in st)[len(st) // 2]}))
