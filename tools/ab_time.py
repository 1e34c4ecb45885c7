"""Steady-state device time of one ADP call shape, for A/B comparisons of library
builds inside one gpurun session (ADPB200_LIB selects the .so):
    python tools/ab_time.py m n k [s|auto] [--seconds T] [--dist u12|u11] [--label X]
Warms up ~1 s (clock ramp, power cap), then times calls for T seconds with CUDA
events and prints one JSON line (ms per call, effective TFLOP/s, sampled SM clock)."""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_13778_b200 as adp  # noqa: E402
from paper_2511_13778_b200 import grading  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("m", type=int)
p.add_argument("n", type=int)
p.add_argument("k", type=int)
p.add_argument("s", nargs="?", default="7")
p.add_argument("--seconds", type=float, default=3.0)
p.add_argument("--dist", default="u12")
p.add_argument("--label", default=os.environ.get("ADPB200_LIB", "default"))
p.add_argument("--pairs", default="target")
p.add_argument("--fallback", default=None, help="time the native fallback flavour (mode native)")
a = p.parse_args()
lo, hi = (1.0, 2.0) if a.dist == "u12" else (-1.0, 1.0)
A = grading.gen_uniform_rect(a.m, a.k, 1, lo, hi)
B = grading.gen_uniform_rect(a.k, a.n, 2, lo, hi)
C = torch.empty((a.m, a.n), dtype=torch.float64, device="cuda")
pl = adp.PAIRS_TARGET if a.pairs == "target" else adp.PAIRS_FULL
if a.fallback:
    cfg = adp.AdpConfig(mode=adp.AdpMode.ForceNative, fallback=a.fallback)
elif a.s == "auto":
    cfg = adp.AdpConfig(pair_limit=pl)
else:
    cfg = adp.AdpConfig(mode=adp.AdpMode.ForceEmulate, forced_slices=int(a.s), pair_limit=pl)
h = adp.Handle.default(0)
flop = 2.0 * a.m * a.n * a.k


def run(n):
    for _ in range(n):
        adp.adp_gemm(A, B, config=cfg, out=C, handle=h)


run(2)
torch.cuda.synchronize()
t0 = time.time()
run(1)
torch.cuda.synchronize()
one = max(time.time() - t0, 1e-5)
t_end = time.time() + 1.0
while time.time() < t_end:
    run(max(1, int(0.2 / one)))
    torch.cuda.synchronize()
clocks = []
stop = False


def sample():
    while not stop:
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                           capture_output=True, text=True)
        try:
            c, pw = r.stdout.strip().split(",")
            clocks.append((float(c), float(pw)))
        except ValueError:
            pass
        time.sleep(0.1)


th = threading.Thread(target=sample)
th.start()
it = max(3, int(a.seconds / one))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
run(it)
e1.record()
torch.cuda.synchronize()
stop = True
th.join()
ms = e0.elapsed_time(e1) / it
cs = sorted(c for c, _ in clocks) or [0.0]
pw = sorted(p for _, p in clocks) or [0.0]
_, t = adp.adp_gemm(A, B, config=cfg, out=C, handle=h)
print(json.dumps({"label": os.path.basename(a.label), "m": a.m, "n": a.n, "k": a.k, "s": t.slices, "path": t.path,
                  "ms": round(ms, 4), "tflops": round(flop / ms / 1e9, 2), "iters": it,
                  "sm_mhz": cs[len(cs) // 2], "power_w": pw[len(pw) // 2]}), flush=True)
