"""Diagnostics for the gap between bench.py's device-resident `value` and its
`e2e` (host inputs): times the layer step (a) with inputs resident, (b) with
the e2e double-buffered H2D copies, (c) with (b) plus the per-step D2H read of
the aux loss, each over --steps steps with CUDA events."""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_09952_b200 as B  # noqa: E402
from paper_2412_09952_b200.upcycle import router_weights, upcycle_experts  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=30)
a = ap.parse_args()
H, F, E, T = 4096, 14336, 8, 8192
dev = torch.device("cuda")
torch.manual_seed(0)
w1, w2, w3 = ((torch.randn(*s, device=dev) * 0.02).to(torch.bfloat16) for s in ((H, F), (F, H), (H, F)))
W1, W2, W3 = (w.requires_grad_() for w in upcycle_experts(w1, w2, w3, E))
cfg_m = B.ModelConfig(vocab=32, hidden=H, layers=1, heads=32, kv_heads=8, ffn_hidden=F, seq_len=T)
wg, wn = router_weights(cfg_m, E, 0, 1, torch.float32, dev)
wg.requires_grad_()
layer = B.MoELayer.from_stacked(B.RouterParams(wg, wn), W1, W2, W3)
gate = B.GateConfig(n_experts=E, top_k=2, capacity_factor=1.0)
x = torch.randn(T, H, device=dev).to(torch.bfloat16)
dy = torch.randn(T, H, device=dev).to(torch.bfloat16)
lam = torch.tensor(0.01, device=dev)
params = [W1, W2, W3, wg]


def step(xin, dyin):
    for p in params:
        p.grad = None
    out = B.moe_forward(xin, layer, gate)
    aux = B.importance_penalty(out.gates)
    torch.autograd.backward([out.output, aux], [dyin, lam])
    return aux


xh, dyh = x.cpu().pin_memory(), dy.cpu().pin_memory()
res_h = torch.empty(a.steps + 4, dtype=torch.float32).pin_memory()
bufs = [(torch.empty_like(x), torch.empty_like(dy)) for _ in range(2)]
cs = torch.cuda.Stream()
main = torch.cuda.current_stream()


def run(mode, n):
    copied = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]
    for ev in consumed:
        ev.record(main)

    def prefetch(i):
        b = i % 2
        with torch.cuda.stream(cs):
            cs.wait_event(consumed[b])
            bufs[b][0].copy_(xh, non_blocking=True)
            bufs[b][1].copy_(dyh, non_blocking=True)
            copied[b].record(cs)

    if mode != "resident":
        prefetch(0)
    for i in range(n):
        b = i % 2
        if mode == "resident":
            aux = step(x.requires_grad_(), dy)
            continue
        if i + 1 < n:
            prefetch(i + 1)
        main.wait_event(copied[b])
        aux = step(bufs[b][0].detach().requires_grad_(), bufs[b][1])
        consumed[b].record(main)
        if mode == "h2d+d2h":
            res_h[i:i + 1].copy_(aux.detach().reshape(1), non_blocking=True)


out = {}
for rep in range(2):
    for mode in ("resident", "h2d", "h2d+d2h"):
        run(mode, 3)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run(mode, a.steps)
        e1.record()
        torch.cuda.synchronize()
        out.setdefault(mode, []).append(round(e0.elapsed_time(e1) / a.steps, 4))
print(json.dumps({"ms_per_step": out}))
