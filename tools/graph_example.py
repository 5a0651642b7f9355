"""The CUDA-graph launch example of INTEGRATION.md, runnable: a small E8T2
layer's training step captured once and replayed on new batches; each
replay's output and gradients are checked against the eager step on the same
batch (bit-identical)."""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_09952_b200 import GateConfig, MoELayer, RouterParams, importance_penalty, moe_forward  # noqa: E402
from paper_2412_09952_b200.graphs import capture  # noqa: E402


def main():
    T, H, F, E = 1024, 512, 1024, 8
    g = torch.Generator(device="cuda").manual_seed(0)
    W = [(torch.randn(s, generator=g, device="cuda") * 0.05).to(torch.bfloat16).requires_grad_()
         for s in ((E, F, H), (E, H, F), (E, F, H))]
    wg = (torch.randn(H, E, generator=g, device="cuda") * 0.1).requires_grad_()
    layer = MoELayer.from_stacked(RouterParams(wg, torch.zeros_like(wg)), *W)
    cfg = GateConfig(n_experts=E, top_k=2, capacity_factor=1.0)

    x = torch.empty(T, H, dtype=torch.bfloat16, device="cuda", requires_grad=True)   # captured inputs
    dy = torch.empty(T, H, dtype=torch.bfloat16, device="cuda")
    lam = torch.tensor(0.01, device="cuda")

    def step():
        for p in (x, *layer.stacked, layer.router.w_g):
            p.grad = None
        out = moe_forward(x, layer, cfg)
        torch.autograd.backward([out.output, importance_penalty(out.gates)], [dy, lam])
        return out

    with torch.no_grad():
        x.copy_(torch.randn(T, H, generator=g, device="cuda"))
        dy.copy_(torch.randn(T, H, generator=g, device="cuda"))
    graph = capture(step, warmup=2)
    # the tensors a replay writes its gradients into: .grad as the capture left it
    # (an eager step rebinds .grad to new tensors, so keep these references)
    params = [x, wg] + W
    grads = [p.grad for p in params]
    for i in range(3):
        xb = torch.randn(T, H, generator=g, device="cuda").to(torch.bfloat16)
        dyb = torch.randn(T, H, generator=g, device="cuda").to(torch.bfloat16)
        with torch.no_grad():
            x.copy_(xb)
            dy.copy_(dyb)
        graph.replay()
        torch.cuda.synchronize()
        got = [graph.outputs.output.clone()] + [t.clone() for t in grads]
        ref_out = step()                       # eager step on the same batch
        want = [ref_out.output] + [p.grad for p in params]
        same = all(torch.equal(a, b) for a, b in zip(got, want))
        print(f"batch {i}: graph replay == eager step: {same}")
        assert same


if __name__ == "__main__":
    main()
