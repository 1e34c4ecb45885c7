"""ESC block length vs slice count and end-to-end time (the reference's own
AdpConfig.esc_block_len knob): 8192^3 U[-1,1] from the reference generator,
target pair policy. A finer block gives a tighter (still safe) coarsened ESC."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_13778_b200 as adp  # noqa: E402
from paper_2511_13778_b200 import grading  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
A = grading.gen_uniform_rect(n, n, 1, -1.0, 1.0)
B = grading.gen_uniform_rect(n, n, 2, -1.0, 1.0)
C = torch.empty((n, n), dtype=torch.float64, device="cuda")
h = adp.Handle.default(0)
ref, absab = grading.dd_gemm(A, B)
for bl in (256, 128, 64, 32, 16, 8):
    cfg = adp.AdpConfig(pair_limit=adp.PAIRS_TARGET, esc_block_len=bl)
    _, tr = adp.adp_gemm(A, B, config=cfg, handle=h, out=C)
    rep = grading.error_report(C, ref, absab=absab)
    for _ in range(2):
        adp.adp_gemm(A, B, config=cfg, handle=h, out=C)
    torch.cuda.synchronize()
    h.profile_enable(5)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        adp.adp_gemm(A, B, config=cfg, handle=h, out=C)
    e1.record()
    torch.cuda.synchronize()
    st = h.profile_read()
    ms = e0.elapsed_time(e1) / 5
    print(json.dumps({"esc_block_len": bl, "esc_bits": tr.esc_bits, "slices": tr.slices, "pairs": tr.pairs,
                      "ms": ms, "tflops": 2.0 * n ** 3 / ms / 1e9,
                      "esc_ms": sum(c["esc"] for c in st) / 5, "stats_ms": sum(c["stats"] for c in st) / 5,
                      "max_ratio_eps_absAB": rep.max_ratio, "max_rel_err": rep.max_err}), flush=True)
