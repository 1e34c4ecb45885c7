"""Per-call e2e times of 80 back-to-back dgemm_host calls (8192^3, pinned host buffers): warm-up and stability."""
import json, os, sys, time
import torch
sys.path.insert(0, "/root/repo") if os.path.exists("/root/repo") else None
sys.path.insert(0, os.getcwd())
import paper_2511_13778_b200 as adp
from paper_2511_13778_b200 import grading
n = 8192
A = grading.gen_uniform_rect(n, n, 1, 1.0, 2.0).cpu().pin_memory()
B = grading.gen_uniform_rect(n, n, 2, 1.0, 2.0).cpu().pin_memory()
C = torch.empty((n, n), dtype=torch.float64).pin_memory()
cfg = adp.AdpConfig(pair_limit=adp.PAIRS_TARGET)
h = adp.Handle.default(0)
ts = []
for i in range(80):
    t0 = time.perf_counter()
    adp.dgemm_host("N", "N", n, n, n, 1.0, A, n, B, n, 0.0, C, n, cfg, h)
    ts.append((time.perf_counter() - t0) * 1e3)
print(json.dumps({"first10": [round(x, 1) for x in ts[:10]], "last10": [round(x, 1) for x in ts[-10:]],
                  "median": sorted(ts)[40]}))
