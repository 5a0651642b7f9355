"""Large-batch parity (T = 65536 tokens): the full CPU oracle is too slow at
this size, so the checks are size-independent --
  * routing over ALL tokens bit-exact against the oracle fed the device's
    fp32 logits (gates, top-k, slot ranks, counts, drop statistics);
  * y and dx recomputed by the oracle for a random sample of tokens from the
    same routing, within the layer tolerances of tests/test_gpu_layer.py.
"""

import numpy as np
import pytest
import torch

from oracle import moe_oracle as O

pytestmark = pytest.mark.gpu

TOL = 1.5e-2


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16).float().numpy()


@pytest.mark.parametrize("rt,pol,cf", [("mixtral", "position", 1.0), ("st", "score", 1.0), ("mixtral", "score", None)])
def test_large_batch_routing_exact_and_sampled_values(rt, pol, cf):
    import paper_2412_09952_b200 as P
    T, H, F, E, k = 65536, 512, 1024, 8, 2
    g = O.rng(77, 0)
    wg = (g.standard_normal((H, E)) * 0.05).astype(np.float32)
    w1 = [bf16(g.standard_normal((H, F)) * 0.05) for _ in range(E)]
    w2 = [bf16(g.standard_normal((F, H)) * 0.05) for _ in range(E)]
    w3 = [bf16(g.standard_normal((H, F)) * 0.05) for _ in range(E)]
    x = bf16(O.rng(78, 0).standard_normal((T, H)))
    dy = bf16(O.rng(79, 0).standard_normal((T, H)))
    dev = torch.device("cuda")
    stack = lambda ws: torch.stack([torch.from_numpy(w.T.copy()) for w in ws]).to(dev, torch.bfloat16)  # noqa: E731
    W1, W2, W3 = (stack(w).requires_grad_() for w in (w1, w2, w3))
    wg_t = torch.from_numpy(wg).to(dev).requires_grad_()
    layer = P.MoELayer.from_stacked(P.RouterParams(wg_t, torch.zeros_like(wg_t)), W1, W2, W3)
    x_t = torch.from_numpy(x).to(dev, torch.bfloat16).requires_grad_()
    cfg = P.GateConfig(n_experts=E, top_k=k, router_type=rt, capacity_factor=cf, drop_policy=pol)
    out = P.moe_forward(x_t, layer, cfg, training=True)
    (out.output.float() * torch.from_numpy(dy).to(dev)).sum().backward()
    torch.cuda.synchronize()

    # ---- routing over every token, bit-exact
    logits = out.routing["logits"].cpu().numpy()
    gt = O.gate(logits, k, rt)
    assert out.gates.detach().cpu().numpy().tobytes() == gt.gates.tobytes()
    disp = O.dispatch(gt.gates, O.expert_capacity(T, E, cf), pol)
    assert np.array_equal(out.routing["slot_rank"].cpu().numpy(), disp.rows())
    assert np.array_equal(out.stats.assigned, disp.assigned)
    assert out.stats.dropped == disp.n_dropped and out.stats.total_slots == disp.total_slots

    # ---- values on a sample of tokens, from the same routing
    idx = np.sort(O.rng(80, 0).choice(T, 192, replace=False))
    xs, dys = x[idx], dy[idx]
    kept = disp.kept[idx]
    gates = gt.gates[idx]
    y_ref = np.zeros((idx.size, H), np.float64)
    dx_ref = np.zeros((idx.size, H), np.float64)
    dg = np.zeros((idx.size, E), np.float64)
    for e in range(E):
        rows = np.flatnonzero(kept[:, e])
        if rows.size == 0:
            continue
        xe = xs[rows].astype(np.float64)
        a, b = xe @ w1[e], xe @ w3[e]
        sg = 1.0 / (1.0 + np.exp(-a))
        h = a * sg * b
        o = h @ w2[e]
        ge = gates[rows, e][:, None]
        y_ref[rows] += ge * o
        dg[rows, e] = (dys[rows] * o).sum(axis=1)
        dm = (ge * dys[rows]) @ w2[e].T
        da = dm * b * sg * (1.0 + a * (1.0 - sg))
        db = dm * a * sg
        dx_ref[rows] += da @ w1[e].T + db @ w3[e].T
    sub = O.gate(logits[idx], k, rt)
    dh = O.gate_bwd(sub, dg)
    dx_ref += dh @ wg.T.astype(np.float64)
    y_dev = out.output.detach().float().cpu().numpy()[idx]
    dx_dev = x_t.grad.float().cpu().numpy()[idx]
    assert rel(y_dev, y_ref) < TOL, rel(y_dev, y_ref)
    assert rel(dx_dev, dx_ref) < TOL, rel(dx_dev, dx_ref)
    full_drop = ~disp.kept.any(axis=1)
    assert np.all(out.output.detach().float().cpu().numpy()[full_drop] == 0.0)
