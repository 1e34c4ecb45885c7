"""One warm-up and one profiled ADP DGEMM call for ncu captures (8192^3 U(1,2),
target pairs by default; --u11 for U[-1,1] operands, --certified for the
certified ESC option, --fast-fallback for the DMMA native fallback):
    ncu --set full --launch-skip <per-call kernels> ... python tools/one_call.py [size | m n k] [--u11] [--certified] [--full]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_13778_b200 as adp  # noqa: E402
from paper_2511_13778_b200 import grading  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
# [size] or [m n k]
m, n, k = (int(args[0]), int(args[1]), int(args[2])) if len(args) >= 3 else ((int(args[0]),) * 3 if args else (8192,) * 3)
lo = -1.0 if "--u11" in sys.argv else 1.0
A = grading.gen_uniform_rect(k, m, 1, lo, 2.0 if lo > 0 else 1.0)  # column-major m x k
B = grading.gen_uniform_rect(n, k, 2, lo, 2.0 if lo > 0 else 1.0)  # column-major k x n
C = torch.empty((n, m), dtype=torch.float64, device="cuda")
cfg = adp.AdpConfig(pair_limit=adp.PAIRS_TARGET, esc_method="certified" if "--certified" in sys.argv else "coarsened")
if "--full" in sys.argv:  # all s^2 slice pairs (the reference's adp_gemm policy)
    cfg = adp.AdpConfig(esc_method=cfg.esc_method)
if "--fast-fallback" in sys.argv:  # the native fallback's DMMA flavour (ForceNative)
    cfg = adp.AdpConfig(mode=adp.AdpMode.ForceNative, fallback="fast")
h = adp.Handle.default(0)
for _ in range(2):
    adp.dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, C, m, cfg, h)
torch.cuda.synchronize()
print("launches per call:", h.launches() // 2)
