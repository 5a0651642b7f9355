"""Microbenchmark of b200moe_rmsnorm_bwd at the model shape (T=8192, H=4096,
residual gradient in, fp32 + bf16 dx out): median time over --reps launches
(CUDA events) and algorithmic HBM bytes / time."""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_09952_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--T", type=int, default=8192)
ap.add_argument("--H", type=int, default=4096)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
T, H = a.T, a.H
x = torch.randn(T, H, device="cuda")
gain = torch.ones(H, device="cuda")
dres = torch.randn(T, H, device="cuda")
dy = torch.randn(T, H, device="cuda").to(torch.bfloat16)
rstd = torch.rsqrt((x ** 2).mean(1) + 1e-5)
dx = torch.empty(T, H, device="cuda")
dxb = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)
dgain = torch.empty(H, device="cuda")
ws = torch.empty((T + 7) // 8 * H, device="cuda")
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")


def run():
    _lib.call("b200moe_rmsnorm_bwd", dy.data_ptr(), x.data_ptr(), rstd.data_ptr(), gain.data_ptr(), dres.data_ptr(),
              T, H, dx.data_ptr(), dxb.data_ptr(), dgain.data_ptr(), ws.data_ptr(), _lib.stream_ptr())


for _ in range(3):
    run()
ts = []
for _ in range(a.reps):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
ms = ts[len(ts) // 2]
alg = T * H * (2 + 4 + 4 + 4 + 2) + T * 4
print(json.dumps({"T": T, "H": H, "us": round(ms * 1e3, 1), "alg_bytes": alg, "GB_s": round(alg / ms / 1e6, 1)}))
