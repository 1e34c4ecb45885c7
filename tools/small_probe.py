"""Small problems (BASELINE config 1: 1024^3 U[-1,1], fixed 7 slices = the 55-bit
window): per-call GPU time of the ADP pipeline (device buffers), cuBLAS DGEMM,
and the reference CPU emulated_gemm on the same inputs."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_13778_b200 as adp  # noqa: E402
from paper_2511_13778_b200 import grading  # noqa: E402
from oracle.oracle import Oracle, available  # noqa: E402

h = adp.Handle.default(0)
for n in (512, 1024, 2048, 4096):
    A = grading.gen_uniform_rect(n, n, 1, -1.0, 1.0)
    B = grading.gen_uniform_rect(n, n, 2, -1.0, 1.0)
    C = torch.empty((n, n), dtype=torch.float64, device="cuda")
    res = {"n": n}
    for label, cfg in (("emulate7_full", adp.AdpConfig(mode=adp.AdpMode.ForceEmulate, forced_slices=7)),
                       ("emulate7_target", adp.AdpConfig(mode=adp.AdpMode.ForceEmulate, forced_slices=7,
                                                         pair_limit=adp.PAIRS_TARGET)),
                       ("adp_auto_target", adp.AdpConfig(pair_limit=adp.PAIRS_TARGET))):
        for _ in range(3):
            adp.adp_gemm(A, B, config=cfg, handle=h, out=C)
        torch.cuda.synchronize()
        it = 20
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        for _ in range(it):
            adp.adp_gemm(A, B, config=cfg, handle=h, out=C)
        e1.record()
        torch.cuda.synchronize()
        host_us = (time.perf_counter() - t0) / it * 1e6
        ms = e0.elapsed_time(e1) / it
        res[label] = {"ms": ms, "tflops": 2.0 * n ** 3 / ms / 1e9, "host_us_per_call": host_us}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.mm(A, B, out=C)
    e0.record()
    for _ in range(20):
        torch.mm(A, B, out=C)
    e1.record()
    torch.cuda.synchronize()
    res["cublas_dgemm_tflops"] = 2.0 * n ** 3 / (e0.elapsed_time(e1) / 20) / 1e9
    if n == 1024 and available("reference"):
        ref = Oracle("reference")
        s = ref.time_call(0, A.cpu().numpy(), B.cpu().numpy(), 7)
        res["reference_cpu_emulated7_s"] = s
        res["reference_cpu_threads"] = os.cpu_count()
    print(json.dumps(res), flush=True)
