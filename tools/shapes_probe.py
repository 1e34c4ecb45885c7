"""Probe of the BASELINE configs beyond the headline on one B200: C5a
(4096 x 4096 x 65536), C5b (65536 x 1024 x 1024) and C4 on one GPU
(32768^3), U[-1,1] operands from the reference generator (seeds 1, 2), ADP
auto with the target pair policy (coarsened and certified ESC), ADP with all pairs, forced 7 slices, and
cuBLAS DGEMM; accuracy against the device double-double oracle.
Usage: python tools/shapes_probe.py [c5a c5b c4 ...]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_13778_b200 as adp  # noqa: E402
from paper_2511_13778_b200 import grading  # noqa: E402

SHAPES = {"c5a": (4096, 4096, 65536), "c5b": (65536, 1024, 1024), "c4": (32768, 32768, 32768),
          "c2": (8192, 8192, 8192)}
h = adp.Handle.default(0)


def timed(fn, it):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it


for name in (sys.argv[1:] or ["c5a", "c5b"]):
    m, n, k = SHAPES[name]
    lo = -1.0
    A = grading.gen_uniform_rect(m, k, 1, lo, 1.0)
    B = grading.gen_uniform_rect(k, n, 2, lo, 1.0)
    C = torch.empty((m, n), dtype=torch.float64, device="cuda")
    flop = 2.0 * m * n * k
    it = max(2, min(20, int(2e13 / flop)))
    res = {"config": name, "m": m, "n": n, "k": k}
    for label, cfg in (("adp_target", adp.AdpConfig(pair_limit=adp.PAIRS_TARGET)),
                       ("adp_target_certified", adp.AdpConfig(pair_limit=adp.PAIRS_TARGET, esc_method="certified")),
                       ("adp_full", adp.AdpConfig()),
                       ("emulate7_target", adp.AdpConfig(mode=adp.AdpMode.ForceEmulate, forced_slices=7,
                                                          pair_limit=adp.PAIRS_TARGET))):
        _, tr = adp.adp_gemm(A, B, config=cfg, handle=h, out=C)
        ms = timed(lambda: adp.adp_gemm(A, B, config=cfg, handle=h, out=C), it)
        h.profile_enable(1)
        adp.adp_gemm(A, B, config=cfg, handle=h, out=C)
        st = h.profile_read()[0]
        h.profile_enable(0)
        d = {"ms": ms, "tflops": flop / ms / 1e9, "slices": tr.slices, "esc_bits": tr.esc_bits, "pairs": tr.pairs,
             "variant": tr.gemm_variant, "k_chunks": tr.k_chunks, "path": tr.path,
             "stages": {kk: round(v, 3) for kk, v in st.items()}}
        if label.startswith("adp_target") and name != "c4":
            ref, absab = grading.dd_gemm(A, B)
            rep = grading.error_report(C, ref, absab=absab)
            d["max_rel_err"], d["max_ratio"] = rep.max_err, rep.max_ratio
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            grading.dd_gemm(A, B)
            e1.record()
            torch.cuda.synchronize()
            d["dd_oracle_ms"] = e0.elapsed_time(e1)
            del ref, absab
        res[label] = d
    nat = timed(lambda: torch.mm(A, B, out=C), it)
    res["cublas_dgemm"] = {"ms": nat, "tflops": flop / nat / 1e9}
    print(json.dumps(res), flush=True)
    del A, B, C
    torch.cuda.empty_cache()
