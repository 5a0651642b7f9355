"""Microbenchmark of the non-GEMM kernels at the bench shape (T=8192, H=4096,
E=8, k=2, CF=1): each C entry point timed alone with CUDA events (median of
--reps), with the HBM bytes it must move and the implied GB/s."""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_09952_b200 as P  # noqa: E402
from paper_2412_09952_b200 import _lib  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--T", type=int, default=8192)
p.add_argument("--H", type=int, default=4096)
p.add_argument("--reps", type=int, default=20)
a = p.parse_args()
T, H, E, k = a.T, a.H, 8, 2
dev = torch.device("cuda")
f32 = dict(dtype=torch.float32, device=dev)
bf = dict(dtype=torch.bfloat16, device=dev)
x = torch.randn(T, H, **bf)
wg = torch.randn(H, E, **f32) * 0.02
wn = torch.zeros(H, E, **f32)
logits, gates = torch.empty(T, E, **f32), torch.empty(T, E, **f32)
err = torch.zeros(1, dtype=torch.int32, device=dev)
ws = torch.empty(2 * H * 32 + T * 32, **f32)
s = _lib.stream_ptr()
_lib.call("b200moe_router_fwd", x.data_ptr(), wg.data_ptr(), wn.data_ptr(), None, T, H, E, k, 0, logits.data_ptr(),
          gates.data_ptr(), None, None, ws.data_ptr(), err.data_ptr(), s)
cap = P.expert_capacity(T, E, 1.0)
slot_rank, counts, seg_base, gate_mass, (imp, _), stats = P.moe._run_dispatch(gates, cap, "position")
torch.cuda.synchronize()
R = P.moe._rows_bound(T, E, k, cap)
xp = torch.zeros(R, H, **bf)
O = torch.randn(R, H, **bf)
y = torch.empty(T, H, **bf)
dy = torch.randn(T, H, **bf)
dO = torch.empty(R, H, **bf)
dg = torch.empty(T, E, **f32)
dxp = torch.randn(R, H, **bf)
dx = torch.empty(T, H, **bf)
dh = torch.empty(T, E, **f32)
wsw = torch.empty((T + 63) // 64 * H * E, **f32)
dwg = torch.empty(H, E, **f32)
MB = T * H * 2
S = int(counts.sum())
cases = {
    "router_fwd": (MB, lambda: _lib.call("b200moe_router_fwd", x.data_ptr(), wg.data_ptr(), wn.data_ptr(), None, T, H,
                                         E, k, 0, logits.data_ptr(), gates.data_ptr(), None, None, ws.data_ptr(),
                                         err.data_ptr(), s)),
    "dispatch": (T * E * 12, lambda: P.moe._run_dispatch(gates, cap, "position")),
    "permute": (MB + S * H * 2, lambda: _lib.call("b200moe_permute", x.data_ptr(), slot_rank.data_ptr(),
                                                   seg_base.data_ptr(), counts.data_ptr(), T, H, E, xp.data_ptr(), s)),
    "combine": (MB + S * H * 2, lambda: _lib.call("b200moe_combine", O.data_ptr(), gates.data_ptr(),
                                                   slot_rank.data_ptr(), seg_base.data_ptr(), T, H, E, y.data_ptr(),
                                                   s)),
    "combine_bwd": (MB + 2 * S * H * 2, lambda: _lib.call("b200moe_combine_bwd", dy.data_ptr(), O.data_ptr(),
                                                          gates.data_ptr(), slot_rank.data_ptr(), seg_base.data_ptr(),
                                                          counts.data_ptr(), T, H, E, dO.data_ptr(), dg.data_ptr(),
                                                          s)),
    "router_bwd": (MB + S * H * 2, lambda: _lib.call("b200moe_router_bwd", dxp.data_ptr(), slot_rank.data_ptr(),
                                                     seg_base.data_ptr(), dg.data_ptr(), None, 0, 0, gates.data_ptr(),
                                                     None, wg.data_ptr(), wn.data_ptr(), None, None, None, None, T, H,
                                                     E, k, 0,
                                                     dx.data_ptr(), dh.data_ptr(), None, ws.data_ptr(), s)),
    "router_wgrad": (MB, lambda: _lib.call("b200moe_router_wgrad", x.data_ptr(), dh.data_ptr(), None, T, H, E,
                                           dwg.data_ptr(), None, wsw.data_ptr(), None, s)),
}
res = {}
for name, (nbytes, fn) in cases.items():
    for _ in range(3):
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
    res[name] = {"us": round(ms * 1e3, 1), "GBps": round(nbytes / (ms * 1e-3) / 1e9, 0)}
print(json.dumps(res))
