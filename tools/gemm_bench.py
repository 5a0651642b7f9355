"""Microbenchmark of the five grouped-GEMM launches at the bench shape
(T=8192 tokens, CF=1 -> 8 experts x 1024 rows, H=4096, F=14336), each timed
with CUDA events (median of --reps), reported as TFLOP/s and fraction of the
measured bf16 peak.  `--only MODE` runs a single mode (for ncu -k)."""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_09952_b200 import _lib  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--H", type=int, default=4096)
p.add_argument("--F", type=int, default=14336)
p.add_argument("--E", type=int, default=8)
p.add_argument("--rows", type=int, default=1024, help="rows per expert")
p.add_argument("--reps", type=int, default=10)
p.add_argument("--cg", type=int, default=2)
p.add_argument("--only", default="")
p.add_argument("--max-ctas", type=int, default=148)
p.add_argument("--debug", type=int, default=0)
p.add_argument("--wgrad-acc", action="store_true", help="WGRAD adding into the existing gradients")
a = p.parse_args()
_lib.call("b200moe_gemm_set_debug", a.debug)

H, F, E, M = a.H, a.F, a.E, a.rows
dev = torch.device("cuda")
_lib.call("b200moe_gemm_set_cta_group", a.cg)
_lib.call("b200moe_gemm_set_max_ctas", a.max_ctas)
Mp = (M + 127) // 128 * 128
R = E * Mp + 256
base = torch.tensor([e * Mp for e in range(E)], dtype=torch.int32, device=dev)
cnt = torch.full((E,), M, dtype=torch.int32, device=dev)
sege = torch.arange(E, dtype=torch.int32, device=dev)
bf = dict(dtype=torch.bfloat16, device=dev)
g = torch.Generator(device=dev).manual_seed(0)
W1 = (torch.randn(E, F, H, generator=g, device=dev) * 0.02).to(torch.bfloat16)
W3 = (torch.randn(E, F, H, generator=g, device=dev) * 0.02).to(torch.bfloat16)
W2 = (torch.randn(E, H, F, generator=g, device=dev) * 0.02).to(torch.bfloat16)
xp = torch.randn(R, H, **bf)
dO = torch.randn(R, H, **bf)
A, B, Hh, dA, dB = (torch.randn(R, F, **bf) for _ in range(5))
O, dxp = torch.empty(R, H, **bf), torch.empty(R, H, **bf)
dW1, dW3, dW2 = torch.zeros_like(W1), torch.zeros_like(W3), torch.zeros_like(W2)
s = _lib.stream_ptr()
S = E * M
modes = {
    "fwd1": (2.0 * S * H * 2 * F, lambda: _lib.call("b200moe_expert_fwd1", xp.data_ptr(), W1.data_ptr(), W3.data_ptr(),
                                                      base.data_ptr(), cnt.data_ptr(), sege.data_ptr(), E, R, H, F, E,
                                                      A.data_ptr(), B.data_ptr(), Hh.data_ptr(), s)),
    "fwd2": (2.0 * S * F * H, lambda: _lib.call("b200moe_expert_fwd2", Hh.data_ptr(), W2.data_ptr(), base.data_ptr(),
                                                  cnt.data_ptr(), sege.data_ptr(), E, R, H, F, E, O.data_ptr(), s)),
    "bwd2": (2.0 * S * H * F, lambda: _lib.call("b200moe_expert_bwd2", dO.data_ptr(), W2.data_ptr(), A.data_ptr(),
                                                  B.data_ptr(), base.data_ptr(), cnt.data_ptr(), sege.data_ptr(), E, R,
                                                  H, F, E, dA.data_ptr(), dB.data_ptr(), s)),
    "wgrad": (2.0 * S * 3 * H * F, lambda: _lib.call("b200moe_expert_wgrad_acc", xp.data_ptr(), Hh.data_ptr(),
                                                       dO.data_ptr(), dA.data_ptr(), dB.data_ptr(), base.data_ptr(),
                                                       cnt.data_ptr(), sege.data_ptr(), E, R, H, F, E, dW1.data_ptr(),
                                                       dW2.data_ptr(), dW3.data_ptr(), int(a.wgrad_acc), s)),
    "bwd1": (2.0 * S * 2 * F * H, lambda: _lib.call("b200moe_expert_bwd1", dA.data_ptr(), dB.data_ptr(),
                                                      W1.data_ptr(), W3.data_ptr(), base.data_ptr(), cnt.data_ptr(),
                                                      sege.data_ptr(), E, R, H, F, E, dxp.data_ptr(), s)),
}
peak = 1692.0
res = {}
for name, (flops, fn) in modes.items():
    if a.only and name != a.only:
        continue
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    tf = flops / ms / 1e9
    res[name] = {"ms": round(ms, 4), "tflops": round(tf, 1), "frac": round(tf / peak, 3)}
tot_ms = sum(v["ms"] for v in res.values())
print(json.dumps({"cg": a.cg, "rows": M, "modes": res, "total_ms": round(tot_ms, 4)}))
