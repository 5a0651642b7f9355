"""Drop-in fidelity of the standalone routing functions and containers
(reference moe.py:72-186, tensor.py:192-227, 267-297, 503-521):

  * router_logits, gate_mixtral and gate_st are differentiable like the
    reference's tape Tensors: their gradients match the oracle's closed-form
    backward;
  * importance_penalty raises GateError at call time when the gate mass is 0;
  * a MoELayer built from a list of ExpertFFN (the reference caller's way,
    model.py:177-188) trains through the same kernels, re-stacks its experts
    only when they change, and hands every expert its own gradient.
"""

import numpy as np
import pytest
import torch

from oracle import moe_oracle as O

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2412_09952_b200 as B


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.mark.parametrize("noise", [False, True])
@pytest.mark.parametrize("T,H,E", [(300, 64, 8), (1000, 256, 4), (77, 512, 16)])
def test_router_logits_differentiable(noise, T, H, E):
    g = O.rng(3, E)
    x = torch.from_numpy(g.standard_normal((T, H)).astype(np.float32)).cuda().to(torch.bfloat16).requires_grad_()
    wg = torch.from_numpy((g.standard_normal((H, E)) * 0.1).astype(np.float32)).cuda().requires_grad_()
    wn = torch.from_numpy((g.standard_normal((H, E)) * 0.1).astype(np.float32)).cuda().requires_grad_()
    z = g.standard_normal((T, E)).astype(np.float32)
    R = g.standard_normal((T, E)).astype(np.float32)
    h = B.router_logits(x, B.RouterParams(wg, wn), noise_enabled=noise,
                        noise=torch.from_numpy(z).cuda() if noise else None)
    (h * torch.from_numpy(R).cuda()).sum().backward()
    xr = x.detach().float().cpu().numpy()
    wg_n, wn_n = wg.detach().cpu().numpy(), wn.detach().cpu().numpy()
    href, an = O.router_logits(xr, wg_n, wn_n, z if noise else None)
    assert rel(h.detach().cpu().numpy(), href) < 1e-5
    dx_ref = R @ wg_n.T
    if noise:
        dn = R * z * O.sigmoid(an)
        dx_ref = dx_ref + dn @ wn_n.T
        assert rel(wn.grad.cpu().numpy(), xr.T @ dn) < 1e-5
    else:
        assert wn.grad is None
    assert rel(wg.grad.cpu().numpy(), xr.T @ R) < 1e-5
    assert rel(x.grad.float().cpu().numpy(), dx_ref) < 1e-2    # dx is bf16 (x's dtype)


@pytest.mark.parametrize("rt", ["mixtral", "st"])
@pytest.mark.parametrize("k,E", [(1, 4), (2, 8), (3, 8), (2, 16), (8, 32)])
def test_gate_functions_differentiable(rt, k, E):
    g = O.rng(4, k * E)
    T = 513
    h = (g.standard_normal((T, E)) * 2).astype(np.float32)
    h[:7, 1] = h[:7, 0]                    # ties: lowest index wins
    R = g.standard_normal((T, E)).astype(np.float32)
    ht = torch.from_numpy(h).cuda().requires_grad_()
    fn = B.gate_mixtral if rt == "mixtral" else B.gate_st
    gates = fn(ht, k)
    (gates * torch.from_numpy(R).cuda()).sum().backward()
    gt = O.gate(h, k, rt)
    assert gates.detach().cpu().numpy().tobytes() == gt.gates.tobytes()
    dh_ref = O.gate_bwd(gt, R)
    assert rel(ht.grad.cpu().numpy(), dh_ref) < 1e-6


def test_gate_chain_router_to_loss_matches_oracle():
    """router_logits -> gate_mixtral -> importance_penalty, backpropagated, as a
    reference user would compose them (moe.py:136-173, tensor.py:503-521)."""
    T, H, E, k = 640, 128, 8, 2
    g = O.rng(5, 0)
    x = torch.from_numpy(g.standard_normal((T, H)).astype(np.float32)).cuda().to(torch.bfloat16)
    wg = torch.from_numpy((g.standard_normal((H, E)) * 0.2).astype(np.float32)).cuda().requires_grad_()
    h = B.router_logits(x, B.RouterParams(wg, torch.zeros_like(wg)), noise_enabled=False)
    gates = B.gate_mixtral(h, k)
    loss = B.importance_penalty(gates)
    loss.backward()
    xr = x.float().cpu().numpy()
    h_dev = h.detach().cpu().numpy()
    gt = O.gate(h_dev, k, "mixtral")
    lref, dimp = O.importance_penalty(gt.gates)
    assert abs(float(loss) - lref) <= 1e-5 * abs(lref)
    dh = O.gate_bwd(gt, np.broadcast_to(dimp, gt.gates.shape))
    assert rel(wg.grad.cpu().numpy(), xr.T @ dh) < 1e-4


def test_importance_penalty_zero_mass_raises_gate_error():
    with pytest.raises(B.GateError, match="positive total gate mass"):
        B.importance_penalty(torch.zeros(16, 8, device="cuda"))
    # gates from moe_forward never take the synchronous check path and stay valid
    assert float(B.importance_penalty(torch.full((16, 8), 0.125, device="cuda"))) == 0.0


def test_expert_list_layer_caches_stack_and_trains():
    T, H, F, E = 256, 256, 512, 4
    g = O.rng(9, 0)
    ws = [[torch.from_numpy((g.standard_normal(s) * 0.05).astype(np.float32)).cuda()
           for s in ((H, F), (F, H), (H, F))] for _ in range(E)]
    ws = [[w.to(torch.bfloat16).float().requires_grad_() for w in trio] for trio in ws]   # bf16-exact fp32
    wg = torch.from_numpy((g.standard_normal((H, E)) * 0.3).astype(np.float32)).cuda()
    router = B.RouterParams(wg, torch.zeros_like(wg))
    layer = B.MoELayer(router, [B.ExpertFFN(w1=a, w2=b, w3=c) for a, b, c in ws])
    cfg = B.GateConfig(n_experts=E, top_k=2, capacity_factor=2.0)
    x = torch.from_numpy(g.standard_normal((T, H)).astype(np.float32)).cuda()
    dy = torch.from_numpy(g.standard_normal((T, H)).astype(np.float32)).cuda()
    out = B.moe_forward(x, layer, cfg)
    stacks = layer._stack_cache[1]
    out2 = B.moe_forward(x, layer, cfg)
    assert layer._stack_cache[1] is stacks                        # no re-stack for unchanged weights
    assert torch.equal(out.output, out2.output)
    (out.output.float() * dy).sum().backward()
    # the same layer in the stacked layout: identical outputs and gradients
    W = [torch.stack([ws[e][j].detach().t() for e in range(E)]).to(torch.bfloat16).requires_grad_()
         for j in range(3)]
    ref = B.moe_forward(x, B.MoELayer.from_stacked(router, *W), cfg)
    (ref.output.float() * dy).sum().backward()
    assert torch.equal(out.output, ref.output)
    for e in range(E):
        for j in range(3):
            assert ws[e][j].grad is not None and ws[e][j].grad.dtype == torch.float32
            assert torch.equal(ws[e][j].grad, W[j].grad[e].t().float()), (e, j)
    with torch.no_grad():                                        # an optimizer step re-stacks
        ws[0][0].add_(0.01)
    B.moe_forward(x, layer, cfg)
    assert layer._stack_cache[1] is not stacks


def test_layer_gate_error_row_surfaces_through_routing_stats():
    """A token row with no finite logit (NaN input) makes the reference's
    softmax raise GateError (tensor.py:283-284).  The layer reports it through
    the dispatch statistics when they are read (no host sync in the forward),
    for the scan dispatch (position) and the per-expert select (score)."""
    T, H, F, E = 300, 256, 256, 8
    for pol in ("position", "score"):
        g = torch.Generator(device="cuda").manual_seed(1)
        W = [(torch.randn(s, generator=g, device="cuda") * 0.05).to(torch.bfloat16) for s in ((E, F, H), (E, H, F),
                                                                                            (E, F, H))]
        wg = torch.randn(H, E, generator=g, device="cuda") * 0.1
        layer = B.MoELayer.from_stacked(B.RouterParams(wg, torch.zeros_like(wg)), *W)
        cfg = B.GateConfig(n_experts=E, top_k=2, capacity_factor=1.0, drop_policy=pol)
        x = torch.randn(T, H, generator=g, device="cuda")
        ok = B.moe_forward(x, layer, cfg)
        assert ok.stats.assigned.sum() > 0                          # healthy batch: no error
        x[17] = float("nan")
        bad = B.moe_forward(x, layer, cfg)
        with pytest.raises(B.GateError):
            _ = bad.stats.assigned
