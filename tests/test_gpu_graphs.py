"""CUDA-graph launch path (paper_2412_09952_b200/graphs.py): a captured
layer training step -- moe_forward, importance_penalty, backward -- replays
to the same bits as the eager step, on the captured inputs and on new data
copied into them (the device-side dispatch epoch and wgrad tickets carry over
between replays), for the scan and the score dispatch, with noise given as a
device tensor, and for an expert-list layer whose weights change in place
between replays.  Bench's K-step graph (spans timed by event-record nodes)
is exercised by bench.py itself."""

import pytest
import torch

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2412_09952_b200 as B
    from paper_2412_09952_b200 import _lib
    from paper_2412_09952_b200.graphs import capture


def _layer(T, H, F, E, seed, list_layer=False):
    g = torch.Generator(device="cuda").manual_seed(seed)
    W = [(torch.randn(s, generator=g, device="cuda") * 0.05).to(torch.bfloat16) for s in ((E, F, H), (E, H, F),
                                                                                        (E, F, H))]
    wg = (torch.randn(H, E, generator=g, device="cuda") * 0.1).requires_grad_()
    wn = (torch.randn(H, E, generator=g, device="cuda") * 0.1).requires_grad_()
    router = B.RouterParams(wg, wn)
    if list_layer:
        experts = [B.ExpertFFN(w1=W[0][e].t().float().requires_grad_(), w2=W[1][e].t().float().requires_grad_(),
                               w3=W[2][e].t().float().requires_grad_()) for e in range(E)]
        layer = B.MoELayer(router, experts)
        params = [wg, wn] + [t for ex in experts for t in (ex.w1, ex.w2, ex.w3)]
    else:
        W = [w.requires_grad_() for w in W]
        layer = B.MoELayer.from_stacked(router, *W)
        params = [wg, wn] + W
    return layer, params


def _step_fn(layer, cfg, params, x, dy, noise=None):
    lam = torch.tensor(0.01, device="cuda")

    def step():
        for p in params + [x]:
            p.grad = None
        out = B.moe_forward(x, layer, cfg, training=noise is not None, noise=noise)
        aux = B.importance_penalty(out.gates)
        torch.autograd.backward([out.output, aux], [dy, lam])
        return out, aux
    return step


def _snap(out, aux, params, x):
    return [out.output.detach().clone(), aux.detach().clone(), x.grad.clone()] + [
        None if p.grad is None else p.grad.clone() for p in params]


def _same(a, b):
    assert len(a) == len(b)
    for i, (u, v) in enumerate(zip(a, b)):
        assert (u is None and v is None) or torch.equal(u, v), i


@pytest.mark.parametrize("policy,noise", [("position", False), ("score", False), ("position", True)])
def test_captured_step_replays_eager_bits(policy, noise):
    T, H, F, E = 1000, 256, 512, 8
    layer, params = _layer(T, H, F, E, 1)
    cfg = B.GateConfig(n_experts=E, top_k=2, capacity_factor=1.0, drop_policy=policy, noise_enabled=noise)
    x = torch.randn(T, H, device="cuda").to(torch.bfloat16).requires_grad_()
    dy = torch.randn(T, H, device="cuda").to(torch.bfloat16)
    z = torch.randn(T, E, device="cuda") if noise else None
    step = _step_fn(layer, cfg, params, x, dy, z)
    ref = _snap(*step(), params, x)
    ref_stats = step()[0].stats
    ref_assigned, ref_dropped = ref_stats.assigned.copy(), ref_stats.dropped

    cap = capture(step, warmup=1)
    for _ in range(3):                       # replays carry the device epoch / tickets forward
        cap.replay()
        torch.cuda.synchronize()
        out, aux = cap.outputs
        _same(_snap(out, aux, params, x), ref)
    st = out.stats
    assert (st.assigned == ref_assigned).all() and st.dropped == ref_dropped

    # new data through the captured inputs == eager on that data
    with torch.no_grad():
        x.copy_(torch.randn(T, H, device="cuda").to(torch.bfloat16))
        dy.copy_(torch.randn(T, H, device="cuda").to(torch.bfloat16))
        if z is not None:
            z.copy_(torch.randn(T, E, device="cuda"))
    cap.replay()
    torch.cuda.synchronize()
    got = _snap(*cap.outputs, params, x)
    _same(got, _snap(*step(), params, x))


def test_captured_list_layer_sees_in_place_updates():
    T, H, F, E = 512, 256, 256, 4
    layer, params = _layer(T, H, F, E, 2, list_layer=True)
    cfg = B.GateConfig(n_experts=E, top_k=2, capacity_factor=2.0)
    x = torch.randn(T, H, device="cuda").to(torch.bfloat16).requires_grad_()
    dy = torch.randn(T, H, device="cuda").to(torch.bfloat16)
    step = _step_fn(layer, cfg, params, x, dy)
    cap = capture(step, warmup=1)
    with torch.no_grad():                    # an optimizer-like in-place update between replays
        for p in params[2:]:
            p.mul_(1.5)
    cap.replay()
    torch.cuda.synchronize()
    got = _snap(*cap.outputs, params, x)
    _same(got, _snap(*step(), params, x))


def test_host_rng_noise_refuses_capture():
    T, H, F, E = 256, 256, 256, 4
    layer, params = _layer(T, H, F, E, 3)
    cfg = B.GateConfig(n_experts=E, top_k=2, capacity_factor=2.0, noise_enabled=True)
    x = torch.randn(T, H, device="cuda").to(torch.bfloat16)
    B.moe_forward(x, layer, cfg, rng=B.Rng(0), training=True)
    g = torch.cuda.CUDAGraph()
    with pytest.raises(B.ConfigError, match="CUDA graph"):
        with torch.cuda.graph(g):
            B.moe_forward(x, layer, cfg, rng=B.Rng(0), training=True)


def test_span_events_time_a_replayed_graph():
    """bench.py's in-step GEMM spans under capture: external event-record
    nodes, timed on every replay."""
    T, H, F, E = 2048, 512, 1024, 8
    layer, params = _layer(T, H, F, E, 4)
    cfg = B.GateConfig(n_experts=E, top_k=2, capacity_factor=1.0)
    x = torch.randn(T, H, device="cuda").to(torch.bfloat16).requires_grad_()
    dy = torch.randn(T, H, device="cuda").to(torch.bfloat16)
    step = _step_fn(layer, cfg, params, x, dy)
    step()
    prof = _lib.Profiler(spans=_lib.GEMM_SPANS)
    _lib.PROFILER = prof
    try:
        cap = capture(step, repeat=3, warmup=0)
    finally:
        _lib.PROFILER = None
    assert len(prof.span_pairs) == 6 and prof.launches > 0
    cap.replay()
    torch.cuda.synchronize()
    ms = prof.span_ms()
    assert 0.0 < ms < 1000.0
