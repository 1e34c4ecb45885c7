"""One warm-up and one profiled ADP DGEMM call for ncu captures (8192^3 U(1,2),
target pairs by default; --u11 for U[-1,1] operands, --certified for the
certified ESC option, --fast-fallback for the DMMA native fallback):
    ncu --set full --launch-skip <per-call kernels> ... python tools/one_call.py [size] [--u11] [--certified]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_13778_b200 as adp  # noqa: E402
from paper_2511_13778_b200 import grading  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
n = int(args[0]) if args else 8192
lo = -1.0 if "--u11" in sys.argv else 1.0
A = grading.gen_uniform_rect(n, n, 1, lo, 2.0 if lo > 0 else 1.0)
B = grading.gen_uniform_rect(n, n, 2, lo, 2.0 if lo > 0 else 1.0)
C = torch.empty((n, n), dtype=torch.float64, device="cuda")
cfg = adp.AdpConfig(pair_limit=adp.PAIRS_TARGET, esc_method="certified" if "--certified" in sys.argv else "coarsened")
if "--fast-fallback" in sys.argv:  # the native fallback's DMMA flavour (ForceNative)
    cfg = adp.AdpConfig(mode=adp.AdpMode.ForceNative, fallback="fast")
h = adp.Handle.default(0)
for _ in range(2):
    adp.dgemm("N", "N", n, n, n, 1.0, A, n, B, n, 0.0, C, n, cfg, h)
torch.cuda.synchronize()
print("launches per call:", h.launches() // 2)
