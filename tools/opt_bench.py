"""Fused optimizer step throughput (model.cu optimizer_kernel): --gparams
billion fp32 master parameters with bf16 gradients and bf16 shadows (the
expert-weight case), CUDA events, median of --reps.  Bytes per parameter:
read p, m, v (12) + g (2), write p, m, v (12) + shadow (2) = 28."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_09952_b200.train import Optimizer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--gparams", type=float, default=1.0)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
n = int(a.gparams * 1e9) // 4096 * 4096
w = torch.randn(n, dtype=torch.bfloat16, device="cuda")
opt = Optimizer("adam", {"w": w})
w.grad = torch.randn(n, dtype=torch.bfloat16, device="cuda") * 1e-3
ts = []
for i in range(a.reps + 2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    opt.step(1e-4)
    e1.record()
    e1.synchronize()
    if i >= 2:
        ts.append(e0.elapsed_time(e1))
ts.sort()
ms = ts[len(ts) // 2]
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
gbs = 28 * n / (ms * 1e-3) / 1e9
print(json.dumps({"kernel": "optimizer_kernel (adam)", "params": n, "ms": round(ms, 3), "GBps": round(gbs, 1),
                  "frac": round(gbs / peak, 3)}))
