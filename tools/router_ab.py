"""Router forward A/B at the bench shape (T=8192, H=4096, E=8): tensor-core K1
vs the CUDA-core K1 (b200moe_router_set_fma), CUDA events, best of 20."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_09952_b200 as B  # noqa: E402
from paper_2412_09952_b200 import _lib  # noqa: E402

T, H, E = 8192, 4096, 8
dev = torch.device("cuda")
x = torch.randn(T, H, device=dev).to(torch.bfloat16)
wg = torch.randn(H, E, device=dev) * 0.02
wn = torch.randn(H, E, device=dev) * 0.02
z = torch.randn(T, E, device=dev)
res = {}
for noise in (False, True):
    for fma in (0, 1, 0, 1):
        _lib.call("b200moe_router_set_fma", fma)
        logits, gates = torch.empty(T, E, device=dev), torch.empty(T, E, device=dev)
        na = torch.empty(T, E, device=dev)
        ws = B.moe._router_ws(H, E, dev)
        def run():
            _lib.call("b200moe_router_fwd", x.data_ptr(), wg.data_ptr(), wn.data_ptr(), z.data_ptr() if noise else None,
                      T, H, E, 2, 0, logits.data_ptr(), gates.data_ptr(), None, na.data_ptr() if noise else None,
                      ws.data_ptr(), None, _lib.stream_ptr())
        for _ in range(5):
            run()
        ts = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); run(); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        key = f"{'fma' if fma else 'tcgen05'}{'+noise' if noise else ''}"
        res[key] = min(res.get(key, 1e9), min(ts) * 1e3)
_lib.call("b200moe_router_set_fma", 0)
print(json.dumps({k: round(v, 2) for k, v in res.items()}), "us")
