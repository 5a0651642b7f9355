"""Layer-level parity on a B200: moe_forward + backward (+ importance aux loss)
through the drop-in API against the CPU oracle run in float32 on the
bf16-rounded device inputs.

Parity rule: routing is compared bit-for-bit when the oracle is
fed the device's fp32 logits (gates, kept/dropped, slot order, counts);
values use the stated bf16 tolerances below (relative Frobenius error)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2412_09952_b200 as B
from oracle import moe_oracle as O

TOL_Y = 1.5e-2     # y, dx
TOL_W = 2e-2       # dW1, dW2, dW3, dW_g, dW_noise
CFS = (0.5, 1.0, 2.0, None)


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def bf16_round(a: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16).float().numpy()


def make_params(T, H, F, E, identical, seed=10, wscale=(0.5, 0.1, 0.3), skew=False):
    g = O.rng(seed, 0)
    wg = (g.standard_normal((H, E)) * wscale[0]).astype(np.float32)
    wn = (g.standard_normal((H, E)) * wscale[1]).astype(np.float32)
    n = 1 if identical else E
    w1 = [(g.standard_normal((H, F)) * wscale[2]).astype(np.float32) for _ in range(n)]
    w2 = [(g.standard_normal((F, H)) * wscale[2]).astype(np.float32) for _ in range(n)]
    w3 = [(g.standard_normal((H, F)) * wscale[2]).astype(np.float32) for _ in range(n)]
    if identical:
        w1, w2, w3 = w1 * E, w2 * E, w3 * E
    x = O.rng(seed + 1, 0).standard_normal((T, H)).astype(np.float32)
    dy = O.rng(seed + 2, 0).standard_normal((T, H)).astype(np.float32)
    z = O.rng(seed + 3, 0).standard_normal((T, E)).astype(np.float32)
    if skew:   # every token prefers experts 0 and 1: x has a positive mean, W_g favours those columns
        x += 1.0
        wg[:, 0] += 0.05
        wg[:, 1] += 0.04
    return wg, wn, w1, w2, w3, x, dy, z


def run_and_compare(T, H, F, E, rt, pol, cf, noise, identical=False, lam=0.37, seed=10, wscale=(0.5, 0.1, 0.3),
                    k=2, skew=False):
    wg, wn, w1, w2, w3, x, dy, z = make_params(T, H, F, E, identical, seed, wscale, skew)
    dev = torch.device("cuda")
    W1 = torch.stack([torch.from_numpy(w.T.copy()) for w in w1]).to(dev, torch.bfloat16).requires_grad_()
    W2 = torch.stack([torch.from_numpy(w.T.copy()) for w in w2]).to(dev, torch.bfloat16).requires_grad_()
    W3 = torch.stack([torch.from_numpy(w.T.copy()) for w in w3]).to(dev, torch.bfloat16).requires_grad_()
    wg_t = torch.from_numpy(wg).to(dev).requires_grad_()
    wn_t = torch.from_numpy(wn).to(dev).requires_grad_()
    layer = B.MoELayer.from_stacked(B.RouterParams(wg_t, wn_t), W1, W2, W3)
    x_t = torch.from_numpy(x).to(dev, torch.bfloat16).requires_grad_()
    dy_t = torch.from_numpy(dy).to(dev)
    cfg = B.GateConfig(n_experts=E, top_k=k, router_type=rt, noise_enabled=noise, capacity_factor=cf,
                       drop_policy=pol)
    out = B.moe_forward(x_t, layer, cfg, training=True, noise=torch.from_numpy(z).to(dev) if noise else None)
    loss = (out.output.float() * dy_t).sum() + lam * B.importance_penalty(out.gates)
    loss.backward()
    torch.cuda.synchronize()

    # ---- oracle on the same (bf16-rounded) inputs and the device logits
    logits = out.routing["logits"].cpu().numpy()
    xr = bf16_round(x)
    w1r = [bf16_round(w) for w in w1]
    w2r = [bf16_round(w) for w in w2]
    w3r = [bf16_round(w) for w in w3]
    ocfg = O.LayerCfg(n_experts=E, top_k=k, router_type=rt, noise=noise, capacity_factor=cf, drop_policy=pol)
    y_o, g_o, cache = O.moe_forward(xr, wg, wn, w1r, w2r, w3r, ocfg, z=z if noise else None, logits=logits)
    _, dimp = O.importance_penalty(g_o)
    gr = O.moe_backward(cache, bf16_round(dy), dgates=lam * dimp)

    # routing: bit-exact
    g_dev = out.gates.detach().cpu().numpy()
    assert g_dev.tobytes() == g_o.tobytes(), "gates differ"
    kept_dev = (out.routing["slot_rank"] >= 0).cpu().numpy()
    assert np.array_equal(kept_dev, cache.disp.kept)
    assert np.array_equal(out.routing["slot_rank"].cpu().numpy(), cache.disp.rows())
    assert np.array_equal(out.stats.assigned, cache.disp.assigned)
    assert out.stats.dropped == cache.disp.n_dropped and out.stats.total_slots == cache.disp.total_slots
    # values
    y_dev = out.output.detach().float().cpu().numpy()
    assert rel(y_dev, y_o) < TOL_Y, rel(y_dev, y_o)
    full_drop = ~cache.disp.kept.any(axis=1)
    assert np.all(y_dev[full_drop] == 0.0)
    assert rel(x_t.grad.float().cpu().numpy(), gr["dx"]) < TOL_Y, rel(x_t.grad.float().cpu().numpy(), gr["dx"])
    assert rel(wg_t.grad.cpu().numpy(), gr["dwg"]) < TOL_W, rel(wg_t.grad.cpu().numpy(), gr["dwg"])
    if noise:
        assert rel(wn_t.grad.cpu().numpy(), gr["dwn"]) < TOL_W
    else:
        assert wn_t.grad is None or float(wn_t.grad.abs().max()) == 0.0
    for name, W in (("dw1", W1), ("dw2", W2), ("dw3", W3)):
        dev_g = np.stack([W.grad[e].float().t().cpu().numpy() for e in range(E)])
        ref_g = np.stack(gr[name])
        assert rel(dev_g, ref_g) < TOL_W, (name, rel(dev_g, ref_g))
    return out


def _small_cases():
    return [(rt, pol, cf, noise) for rt in ("mixtral", "st") for pol in ("position", "score") for cf in CFS
            for noise in (False, True)]


@pytest.mark.parametrize("rt,pol,cf,noise", _small_cases())
def test_small_layer(rt, pol, cf, noise):
    """T=96, H=16, F=24 (padded to the GEMM tile internally), random experts."""
    run_and_compare(96, 16, 24, 8, rt, pol, cf, noise)


@pytest.mark.parametrize("rt", ["mixtral", "st"])
@pytest.mark.parametrize("cf", [1.0, 2.0, None])
def test_cfg1_upcycled_layer(rt, cf):
    """Config 1: T=2048, H=256, F=512, E8T2, identical (upcycled) experts."""
    # lam=1: with identical experts the expert-path router gradient cancels
    # exactly (sum of p*(dg - dg) = 0), so dW_g is carried by the aux term.
    run_and_compare(2048, 256, 512, 8, rt, "position", cf, False, identical=True, lam=1.0,
                    wscale=(0.02, 0.0, 0.02))


@pytest.mark.parametrize("E,k", [(2, 1), (4, 2), (4, 4), (6, 3), (16, 2), (16, 5), (32, 2), (32, 8)])
@pytest.mark.parametrize("rt,pol,cf", [("mixtral", "position", 1.0), ("st", "score", 2.0), ("mixtral", "score", None)])
def test_expert_count_and_fanout_sweep(E, k, rt, pol, cf):
    """Other E / top-k than E8T2 (every router / dispatch / backward template
    bucket: E in 4, 8, 16, 32 buckets, kept-per-token 1..8), with noise."""
    run_and_compare(160, 32, 48, E, rt, pol, cf, True, k=k, seed=30 + E + k)


@pytest.mark.parametrize("pol", ["position", "score"])
def test_random_experts_mid(pol):
    run_and_compare(1000, 512, 768, 8, "mixtral", pol, 1.0, True, seed=20, wscale=(0.05, 0.02, 0.05))


def test_identical_experts_mixtral_dropless_equals_dense_ffn():
    """Reference invariant test_moe.py:254-263 at bf16 tolerance."""
    T, H, F, E = 300, 256, 512, 4
    g = O.rng(6, 0)
    w1, w2, w3 = ((g.standard_normal(s) * 0.05).astype(np.float32) for s in ((H, F), (F, H), (H, F)))
    wg = (g.standard_normal((H, E)) * 0.5).astype(np.float32)
    x = g.standard_normal((T, H)).astype(np.float32)
    dev = torch.device("cuda")
    ckw = [torch.from_numpy(w).to(dev) for w in (w1, w2, w3)]
    from paper_2412_09952_b200.upcycle import upcycle_experts
    W1, W2, W3 = upcycle_experts(*ckw, E)
    layer = B.MoELayer.from_stacked(B.RouterParams(torch.from_numpy(wg).to(dev), torch.zeros(H, E, device=dev)),
                                    W1, W2, W3)
    out = B.moe_forward(torch.from_numpy(x).to(dev), layer, B.GateConfig(n_experts=E, top_k=2))
    dense = B.ffn_forward(torch.from_numpy(x).to(dev), *ckw)
    assert out.stats.dropped == 0
    assert rel(out.output.float().cpu().numpy(), dense.float().cpu().numpy()) < 1e-2


@pytest.mark.parametrize("cf,pol", [(None, "position"), (1.0, "position"), (1.0, "score"), (4.0, "position")])
def test_skewed_routing_hot_experts(cf, pol):
    """Load imbalance: nearly every token routes to experts 0 and 1, so two
    segments hold ~T rows each (dropless / CF 4) or overflow heavily (CF 1) and
    the other experts get few or no rows; routing bit-exact and values within
    tolerance as for uniform load."""
    out = run_and_compare(1536, 256, 512, 8, "mixtral", pol, cf, False, lam=0.01, skew=True,
                          wscale=(0.05, 0.0, 0.05))
    a = out.stats.assigned
    assert a[0] + a[1] >= 0.9 * min(a.sum(), 2 * 1536) if cf is None else a[0] > 0
    if cf == 1.0:
        assert out.stats.dropped > 1000


def test_capacity_drops_contribute_zero_and_determinism():
    wg, wn, w1, w2, w3, x, dy, z = make_params(512, 256, 256, 8, False, seed=30, wscale=(0.3, 0.0, 0.05))
    dev = torch.device("cuda")
    layer = B.MoELayer.from_stacked(
        B.RouterParams(torch.from_numpy(wg).to(dev), torch.from_numpy(wn).to(dev)),
        *(torch.stack([torch.from_numpy(w.T.copy()) for w in ws]).to(dev, torch.bfloat16) for ws in (w1, w2, w3)))
    cfg = B.GateConfig(n_experts=8, top_k=2, capacity_factor=0.5)
    xt = torch.from_numpy(x).to(dev, torch.bfloat16)
    a = B.moe_forward(xt, layer, cfg)
    b = B.moe_forward(xt, layer, cfg)
    assert torch.equal(a.output, b.output)   # run-to-run bitwise deterministic
    kept_any = (a.routing["slot_rank"] >= 0).any(dim=1)
    assert a.stats.dropped > 0
    assert bool((a.output[~kept_any] == 0).all())


def test_fused_expert_grad_accumulation_matches_autograd_adds():
    """set_expert_grad_accumulation_fusion: over three backward passes the
    expert gradients added inside WGRAD match autograd's accumulation (within
    bf16 rounding of the running sum), the first pass still hands a fresh
    gradient to autograd, other gradients are untouched, and the leaves'
    post-accumulate hooks fire on every pass."""
    wg, wn, w1, w2, w3, x, dy, z = make_params(512, 256, 512, 8, False, seed=40, wscale=(0.3, 0.0, 0.05))
    dev = torch.device("cuda")
    cfg = B.GateConfig(n_experts=8, top_k=2, capacity_factor=1.0)
    res = {}
    for fused in (False, True):
        Ws = [torch.stack([torch.from_numpy(w.T.copy()) for w in ws]).to(dev, torch.bfloat16).requires_grad_()
              for ws in (w1, w2, w3)]
        wg_t = torch.from_numpy(wg).to(dev).requires_grad_()
        layer = B.MoELayer.from_stacked(B.RouterParams(wg_t, torch.from_numpy(wn).to(dev)), *Ws)
        fired = []
        hooks = [W.register_post_accumulate_grad_hook(lambda t, i=i: fired.append(i)) for i, W in enumerate(Ws)]
        B.moe.set_expert_grad_accumulation_fusion(fused)
        try:
            for p in range(3):
                xt = (torch.from_numpy(x).to(dev) * (1 + 0.1 * p)).to(torch.bfloat16).requires_grad_()
                out = B.moe_forward(xt, layer, cfg)
                (out.output.float() * torch.from_numpy(dy).to(dev)).sum().backward()
        finally:
            B.moe.set_expert_grad_accumulation_fusion(False)
            for h in hooks:
                h.remove()
        torch.cuda.synchronize()
        assert sorted(fired) == [0, 0, 0, 1, 1, 1, 2, 2, 2]
        res[fused] = [W.grad.float() for W in Ws] + [wg_t.grad]
    for a, b in zip(res[False], res[True]):
        assert rel(b.cpu().numpy(), a.cpu().numpy()) < 5e-3
    assert torch.equal(res[False][3], res[True][3])   # router gradient path unchanged
