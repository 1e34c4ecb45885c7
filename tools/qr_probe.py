"""QR caller timing: geqrf_blocked on the GPU (panel kernel in reference order +
ADP trailing updates) vs the reference's CPU geqrf_blocked (oracle/_ref, all
host threads) and cusolverDnDgeqrf (torch.geqrf, cuSOLVER backend) on the same
GPU, acceptance-criterion-8 style inputs (uniform(0,1), panel 32,
min_dim 8 so the trailing products emulate). Prints one JSON line per size."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_13778_b200 as adp  # noqa: E402
from paper_2511_13778_b200 import grading, qr  # noqa: E402
from oracle.oracle import Oracle, available  # noqa: E402

ref = Oracle("reference") if available("reference") else None
# all GPU timings first: the reference's OpenMP threads keep spinning after a CPU run and
# would slow the host loop that issues the QR's ~2 launches per column
lines = []
for m, n, panel in ((1024, 512, 32), (2048, 1024, 64), (4096, 2048, 128), (8192, 4096, 128)):
    a = grading.gen_uniform_rect(m, n, 0x9802, 0.0, 1.0)
    cfg = adp.AdpConfig(min_dim=8)
    qr.geqrf_blocked(a, panel, cfg)
    torch.cuda.synchronize()
    times = []
    for _ in range(3):  # median of three timed calls
        t0 = time.perf_counter()
        res = qr.geqrf_blocked(a, panel, cfg)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    gpu_s = sorted(times)[1]
    acc = qr.qr_residual(a, res)
    emu = sum(t.path == "emulated" for t in res.traces)
    # cusolverDnDgeqrf (torch.geqrf with the cuSOLVER backend) on the same matrix, same device
    torch.backends.cuda.preferred_linalg_library("cusolver")
    torch.geqrf(a)
    torch.cuda.synchronize()
    ctimes = []
    for _ in range(5):
        t0 = time.perf_counter()
        torch.geqrf(a)
        torch.cuda.synchronize()
        ctimes.append(time.perf_counter() - t0)
    cus_s = sorted(ctimes)[2]
    line = {"m": m, "n": n, "panel": panel, "gpu_s": gpu_s, "residual": acc.residual,
            "orthogonality": acc.orthogonality, "emulated_gemms": emu, "gemms": len(res.traces),
            "cusolver_dgeqrf_s": cus_s, "gpu_vs_cusolver": cus_s / gpu_s}
    lines.append((line, a.cpu().numpy() if m <= 2048 else None))
for line, a_host in lines:
    if ref is not None and a_host is not None:
        line["ref_cpu_s"] = ref.time_qr(a_host, line["panel"], 8)
        line["ref_cpu_threads"] = os.cpu_count()
        line["speedup"] = line["ref_cpu_s"] / line["gpu_s"]
    print(json.dumps(line), flush=True)
