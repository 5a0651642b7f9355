"""Microbenchmark of the fused cross-entropy kernels at the lm-head shape
(T=8192 rows, V=128256 bf16 logits): median time (CUDA events) and HBM GB/s
of the forward (one read of the logits) and the backward (read + write)."""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_09952_b200 import _lib  # noqa: E402

T, V = int(os.environ.get("CE_T", 8192)), int(os.environ.get("CE_V", 128256))
reps = int(os.environ.get("CE_REPS", 10))
logits = (torch.randn(T, V, device="cuda") * 2).to(torch.bfloat16)
tg = torch.randint(0, V, (T,), device="cuda")
nll, lse, loss = torch.empty(T, device="cuda"), torch.empty(T, device="cuda"), torch.empty(1, device="cuda")
err = torch.zeros(1, dtype=torch.int32, device="cuda")
dl = torch.ones(1, device="cuda")
dlog = torch.empty_like(logits)
s = _lib.stream_ptr()
fns = {"fwd": lambda: _lib.call("b200moe_cross_entropy_fwd", logits.data_ptr(), tg.data_ptr(), T, V, nll.data_ptr(),
                                lse.data_ptr(), loss.data_ptr(), err.data_ptr(), s),
       "bwd": lambda: _lib.call("b200moe_cross_entropy_bwd", logits.data_ptr(), tg.data_ptr(), lse.data_ptr(),
                                dl.data_ptr(), T, V, dlog.data_ptr(), s)}
out = {}
for k, fn in fns.items():
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    nbytes = T * V * 2 * (1 if k == "fwd" else 2)
    out[k] = {"us": round(ms * 1e3, 1), "GB_s": round(nbytes / ms / 1e6, 1)}
print(json.dumps(out))
