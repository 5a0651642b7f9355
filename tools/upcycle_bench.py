"""K12 upcycle_copy throughput: one dense SwiGLU FFN (fp32 [H,F], [F,H], [H,F])
replicated into E bf16 experts in kernel layout; CUDA events, median of --reps.
Bytes: read 3*H*F*4, write E*3*H*F*2."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_09952_b200.upcycle import upcycle_experts  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--H", type=int, default=4096)
ap.add_argument("--F", type=int, default=14336)
ap.add_argument("--E", type=int, default=8)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
w1 = torch.randn(a.H, a.F, device="cuda")
w2 = torch.randn(a.F, a.H, device="cuda")
w3 = torch.randn(a.H, a.F, device="cuda")
ts = []
for i in range(a.reps + 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = upcycle_experts(w1, w2, w3, a.E)
    e1.record()
    e1.synchronize()
    if i:
        ts.append(e0.elapsed_time(e1))
    del out
ts.sort()
ms = ts[len(ts) // 2]
nbytes = 3 * a.H * a.F * 4 + a.E * 3 * a.H * a.F * 2
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
gbs = nbytes / (ms * 1e-3) / 1e9
print(json.dumps({"kernel": "upcycle_copy (K12)", "ms": round(ms, 3), "GBps": round(gbs, 1), "frac": round(gbs / peak, 3)}))
