"""Power / clock of the slice GEMM under ADPB200_DEBUG modes (0 normal, 1 data path
only: TMA + epilogue without MMAs, 2 no epilogue math), sampled by nvidia-smi
while the 8192^3 call loops for ~3 s."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_13778_b200 as adp  # noqa: E402
from paper_2511_13778_b200 import grading  # noqa: E402
from bench import ClockSampler  # noqa: E402

n = 8192
A = grading.gen_uniform_rect(n, n, 1, 1.0, 2.0)
B = grading.gen_uniform_rect(n, n, 2, 1.0, 2.0)
C = torch.empty((n, n), dtype=torch.float64, device="cuda")
cfg = adp.AdpConfig(pair_limit=adp.PAIRS_TARGET)
h = adp.Handle.default(0)
for _ in range(5):
    adp.dgemm("N", "N", n, n, n, 1.0, A, n, B, n, 0.0, C, n, cfg, h)
torch.cuda.synchronize()
s = ClockSampler(0)
s.start()
time.sleep(0.5)
t0 = time.time()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
it = 0
while time.time() - t0 < 3.0:
    for _ in range(10):
        adp.dgemm("N", "N", n, n, n, 1.0, A, n, B, n, 0.0, C, n, cfg, h)
    it += 10
    torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
t1 = time.time()
clk = s.stop(t0, t1)
print(json.dumps({"debug": os.environ.get("ADPB200_DEBUG", "0"), "ms_per_call": e0.elapsed_time(e1) / it,
                  "clocks": clk}))
