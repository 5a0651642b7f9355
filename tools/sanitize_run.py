"""Small-shape driver for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel family of the layer at shapes that finish in seconds
under the tool, on one GPU:

  * the layer fwd+bwd (router K1, dispatch K1b, permute K2, grouped GEMMs
    FWD1/FWD2/BWD2/WGRAD/BWD1, combine K5/K6, router backward K10/K11,
    router wgrad, importance) for both routers / policies, capacity and
    dropless, noise on, with the CTA-pair AND the single-SM GEMM kernels;
  * WGRAD accumulate mode, the wide WGRAD tiles;
  * the standalone router_logits / gate backward;
  * upcycling copy (K12) and the checkpoint CRC32C kernel.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_09952_b200 as P  # noqa: E402
from paper_2412_09952_b200 import _lib  # noqa: E402
from paper_2412_09952_b200.upcycle import upcycle_experts  # noqa: E402


def layer_case(T, H, F, E, k, rt, pol, cf, noise, acc=False):
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(T + H + E)
    W1, W2, W3 = ((torch.randn(s, generator=g, device=dev) * 0.05).to(torch.bfloat16).requires_grad_()
                  for s in ((E, F, H), (E, H, F), (E, F, H)))
    wg = (torch.randn(H, E, generator=g, device=dev) * 0.1).requires_grad_()
    wn = (torch.randn(H, E, generator=g, device=dev) * 0.05).requires_grad_()
    x = torch.randn(T, H, generator=g, device=dev).to(torch.bfloat16).requires_grad_()
    z = torch.randn(T, E, generator=g, device=dev) if noise else None
    cfg = P.GateConfig(n_experts=E, top_k=k, router_type=rt, noise_enabled=noise, capacity_factor=cf,
                       drop_policy=pol)
    layer = P.MoELayer.from_stacked(P.RouterParams(wg, wn), W1, W2, W3)
    P.moe.set_expert_grad_accumulation_fusion(acc)
    try:
        for _ in range(2 if acc else 1):
            out = P.moe_forward(x, layer, cfg, training=True, noise=z)
            loss = (out.output.float() ** 2).sum() + 0.1 * P.importance_penalty(out.gates)
            loss.backward()
    finally:
        P.moe.set_expert_grad_accumulation_fusion(False)
    torch.cuda.synchronize()
    _ = out.stats.assigned


def main():
    dev = torch.device("cuda")
    for cg in (2, 1):
        _lib.call("b200moe_gemm_set_cta_group", cg)
        layer_case(300, 256, 512, 8, 2, "mixtral", "position", 1.0, True)
        layer_case(257, 512, 256, 8, 2, "st", "score", None, False)
        layer_case(200, 256, 256, 4, 2, "mixtral", "score", 0.5, True, acc=True)
        layer_case(96, 256, 512, 16, 4, "st", "position", 2.0, True)
    _lib.call("b200moe_gemm_set_cta_group", 2)
    _lib.call("b200moe_gemm_set_debug", 256)          # wide WGRAD tiles (opt-in variant)
    layer_case(300, 256, 512, 8, 2, "mixtral", "position", 1.0, False)
    _lib.call("b200moe_gemm_set_debug", 0)
    # standalone routing functions with their backward
    x = torch.randn(333, 256, device=dev).to(torch.bfloat16).requires_grad_()
    wg = (torch.randn(256, 8, device=dev) * 0.1).requires_grad_()
    wn = (torch.randn(256, 8, device=dev) * 0.1).requires_grad_()
    h = P.router_logits(x, P.RouterParams(wg, wn), True, noise=torch.randn(333, 8, device=dev))
    (P.gate_mixtral(h, 2).sum() + P.gate_st(h, 2).pow(2).sum()).backward()
    # upcycling copy and checkpoint CRC
    w = [torch.randn(s, device=dev) for s in ((256, 512), (512, 256), (256, 512))]
    upcycle_experts(*w, 4)
    from paper_2412_09952_b200.checkpoint import crc32c
    crc32c(torch.randn(1 << 16, device=dev))
    torch.cuda.synchronize()
    print("sanitize_run ok", flush=True)


if __name__ == "__main__":
    main()
