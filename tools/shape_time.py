"""Device time of one ADP call shape (forced s, target pairs): python tools/shape_time.py m n k [s]"""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_13778_b200 as adp  # noqa: E402
from paper_2511_13778_b200 import grading  # noqa: E402
m, n, k = (int(x) for x in sys.argv[1:4])
s = int(sys.argv[4]) if len(sys.argv) > 4 else 7
A = grading.gen_uniform_rect(m, k, 1, 1.0, 2.0)
B = grading.gen_uniform_rect(k, n, 2, 1.0, 2.0)
C = torch.empty((m, n), dtype=torch.float64, device="cuda")
cfg = adp.AdpConfig(mode=adp.AdpMode.ForceEmulate, forced_slices=s, pair_limit=adp.PAIRS_TARGET)
h = adp.Handle.default(0)
for _ in range(3):
    adp.adp_gemm(A, B, config=cfg, out=C, handle=h)
torch.cuda.synchronize()
it = max(3, int(5e12 / (2.0 * m * n * k)))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(it):
    adp.adp_gemm(A, B, config=cfg, out=C, handle=h)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / it
print(json.dumps({"m": m, "n": n, "k": k, "s": s, "ms": ms, "tflops": 2.0 * m * n * k / ms / 1e9}))
