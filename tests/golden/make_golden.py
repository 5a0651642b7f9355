"""Generate golden fixtures by running the REFERENCE (`moefold`) itself.

Run in the build container only (it needs /root/reference, which does not
exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Outputs (committed, small):
  routing_cfg1.npz   config-1 routing (T=2048,H=256,F=512,E=8,k=2) for both
                     routers x CF {0.5,1,2,None} x {position,score}
  routing_edge.npz   hand-made / extreme logit rows: ties, +-0, exp underflow,
                     non-finite entries, k=1..E
  layer_small.npz    full fwd+bwd (y, dx, dW_g, dW_noise, dW1..3) of small
                     random layers for every router/policy/CF/noise combo,
                     fp32 and fp64, loss = sum(y*dy) + lam*importance_penalty
  layer_cfg1.npz     config-1 fwd+bwd summaries (row norms, grad norms)
  upcycle.npz        sha256 digests of upcycle_full / upcycle_shard tensors
                     and the config-1 dense FFN / router bits
The numpy version and SIMD targets of the generating host are recorded in
each file (`meta`), since numpy's float32 exp is SIMD-path dependent.
"""

from __future__ import annotations

import hashlib
import io
import json
import os
import sys
from contextlib import redirect_stdout

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

from moefold.model import ModelConfig, init_dense  # noqa: E402
from moefold.moe import (ExpertFFN, GateConfig, MoELayer, RouterParams, dispatch,  # noqa: E402
                         expert_capacity, gate_mixtral, gate_st, moe_forward)
from moefold.rng import Rng  # noqa: E402
from moefold.tensor import Tensor, importance_penalty, mul, sum_all  # noqa: E402
from moefold.upcycle import router_weights, shard_dense, upcycle_full, upcycle_shard  # noqa: E402
from moefold.model import _moe_layer_view  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
CFS = (0.5, 1.0, 2.0, None)
POLICIES = ("position", "score")
ROUTERS = ("mixtral", "st")


def meta() -> str:
    buf = io.StringIO()
    with redirect_stdout(buf):
        np.show_runtime()
    return json.dumps({"numpy": np.__version__, "runtime": buf.getvalue()})


def cf_key(cf):
    return "none" if cf is None else str(cf).replace(".", "p")


def routing_cfg1():
    cfg = ModelConfig(vocab=32, hidden=256, layers=1, heads=4, kv_heads=2, ffn_hidden=512, seq_len=2048)
    dense = init_dense(cfg, seed=7, dtype=np.float32)
    moe = upcycle_full(dense, n_experts=8, top_k=2, router_seed=1, capacity_factor=1.0)
    layer = _moe_layer_view(moe.tensors, 0, 8)
    x = Tensor(Rng(123, 0).standard_normal((2048, 256)).astype(np.float32))
    h = (x.data @ layer.router.w_g.data)
    out = {"meta": meta(), "logits": h, "wg": layer.router.w_g.data}
    for rt in ROUTERS:
        g = (gate_mixtral if rt == "mixtral" else gate_st)(Tensor(h), 2).data
        assert g.dtype == np.float32
        out[f"{rt}_gates"] = g
        for cf in CFS:
            cap = expert_capacity(2048, 8, cf)
            for pol in POLICIES:
                d = dispatch(g, cap, pol)
                k = f"{rt}_{cf_key(cf)}_{pol}"
                out[k + "_kept"] = np.packbits(d.kept)
                out[k + "_dropped"] = np.packbits(d.dropped)
                out[k + "_assigned"] = d.stats.assigned
                out[k + "_gate_mass"] = d.stats.gate_mass
                out[k + "_stats"] = np.array([d.stats.dropped, d.stats.total_slots,
                                              -1 if cap is None else cap], dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, "routing_cfg1.npz"), **out)


def routing_edge():
    rows = []
    E = 8
    rows.append(np.zeros(E))                                   # all tied
    rows.append(np.array([-0.0, 0.0, 0.0, -1, -1, -1, -1, -1]))  # signed zero ties
    rows.append(np.array([0, 120, 0, 0, 0, 0, 0, 0]))           # f32 exp underflow: 1 slot
    rows.append(np.array([0, 103.9, 0, 0, 0, 0, 0, 0]))         # just above underflow
    rows.append(np.array([0, 103.98, 0, 0, 0, 0, 0, 0]))
    rows.append(np.array([5, 5, 5, 1, 5, 5, 5, 5]))
    rows.append(np.array([1, 3, 2, 0, -1, -2, -3, -4]))
    rows.append(np.array([-50, -60, -70, -80, -90, -100, -110, -120]))
    rows.append(np.array([1e-7, 2e-7, 1e-7, 0, 0, 0, 0, 0]))
    rows.append(np.array([3.4e38, -3.4e38, 3.0e38, 0, 0, 0, 0, 0]))
    rng = np.random.default_rng(20241213)
    finite = [np.stack(rows).astype(np.float32)]
    finite.append((rng.standard_normal((1500, E)) * 1.3).astype(np.float32))
    finite.append((rng.standard_normal((1000, E)) * 40.0).astype(np.float32))
    finite.append(np.round(rng.standard_normal((500, E)) * 2, 1).astype(np.float32))  # many ties
    h = np.concatenate(finite)
    out = {"meta": meta(), "logits": h}
    for rt in ROUTERS:
        for k in (1, 2, 3, 4, 8):
            g = (gate_mixtral if rt == "mixtral" else gate_st)(Tensor(h), k).data
            out[f"{rt}_k{k}_gates"] = g
    # non-finite rows (only reachable with non-finite activations)
    nf = np.array([[np.inf, 1, 2, 0, 0, 0, 0, 0],
                   [np.nan, 1, 2, 0, 0, 0, 0, 0],
                   [1, np.nan, 2, np.nan, 0, 0, 0, 0],
                   [-np.inf, 1, 2, 0, 0, 0, 0, 0],
                   [np.inf, np.inf, 2, 0, 0, 0, 0, 0]], dtype=np.float32)
    out["nonfinite_logits"] = nf
    for rt in ROUTERS:
        gs = []
        for r in nf:
            try:
                gs.append((gate_mixtral if rt == "mixtral" else gate_st)(Tensor(r[None, :]), 2).data[0])
            except Exception:  # GateError
                gs.append(np.full(E, -1.0, dtype=np.float32))
        out[f"nonfinite_{rt}_gates"] = np.stack(gs)
    # the token-prefix capacity example: token 0's 2nd choice evicts token 1's 1st
    ex = Tensor(np.array([[0, 2, 1], [0, 1, 2]], dtype=np.float32))
    g = gate_mixtral(ex, 2).data
    d = dispatch(g, 1, "position")
    out["prefix_example_gates"] = g
    out["prefix_example_kept"] = d.kept
    np.savez_compressed(os.path.join(OUT, "routing_edge.npz"), **out)


def small_layer(rng: Rng, hidden, ffn, n, dtype):
    router = RouterParams(w_g=Tensor(rng.normal((hidden, n), 0.5).astype(dtype), requires_grad=True),
                          w_noise=Tensor(rng.normal((hidden, n), 0.1).astype(dtype), requires_grad=True))
    experts = []
    for _ in range(n):
        experts.append(ExpertFFN(*(Tensor(rng.normal(s, 0.3).astype(dtype), requires_grad=True)
                                   for s in ((hidden, ffn), (ffn, hidden), (hidden, ffn)))))
    return MoELayer(router=router, experts=experts)


def layer_small():
    T, H, F, E = 96, 16, 24, 8
    lam = 0.37
    out = {"meta": meta(), "shape": np.array([T, H, F, E]), "lam": np.array(lam)}
    for dt_name, dt in (("f32", np.float32), ("f64", np.float64)):
        for rt in ROUTERS:
            for pol in POLICIES:
                for cf in CFS:
                    for noise in (False, True):
                        if dt_name == "f64" and (cf != 1.0 or pol != "position"):
                            continue
                        key = f"{dt_name}_{rt}_{pol}_{cf_key(cf)}_{'noise' if noise else 'clean'}"
                        layer = small_layer(Rng(10, 0), H, F, E, dt)
                        x = Tensor(Rng(11, 0).standard_normal((T, H)).astype(dt), requires_grad=True)
                        dy = Rng(12, 0).standard_normal((T, H)).astype(dt)
                        cfg = GateConfig(n_experts=E, top_k=2, router_type=rt, noise_enabled=noise,
                                         capacity_factor=cf, drop_policy=pol)
                        res = moe_forward(x, layer, cfg, rng=Rng(13, 0) if noise else None, training=noise)
                        loss = sum_all(mul(res.output, Tensor(dy))) + importance_penalty(res.gates) * lam
                        loss.backward()
                        out[key + "_y"] = res.output.data
                        out[key + "_gates"] = res.gates.data
                        z0 = lambda t: t.grad if t.grad is not None else np.zeros_like(t.data)  # noqa: E731
                        out[key + "_dx"] = z0(x)
                        out[key + "_dwg"] = z0(layer.router.w_g)
                        out[key + "_dwn"] = z0(layer.router.w_noise)
                        for w in ("w1", "w2", "w3"):
                            out[key + f"_d{w}"] = np.stack([
                                getattr(ex, w).grad if getattr(ex, w).grad is not None
                                else np.zeros_like(getattr(ex, w).data) for ex in layer.experts])
                        out[key + "_assigned"] = res.stats.assigned
                        out[key + "_dropped"] = np.array(res.stats.dropped)
    np.savez_compressed(os.path.join(OUT, "layer_small.npz"), **out)


def layer_cfg1():
    cfg = ModelConfig(vocab=32, hidden=256, layers=1, heads=4, kv_heads=2, ffn_hidden=512, seq_len=2048)
    dense = init_dense(cfg, seed=7, dtype=np.float32)
    out = {"meta": meta()}
    for rt in ROUTERS:
        moe = upcycle_full(dense, n_experts=8, top_k=2, router_seed=1, capacity_factor=1.0, router_type=rt)
        layer = _moe_layer_view(moe.tensors, 0, 8)
        x = Tensor(Rng(123, 0).standard_normal((2048, 256)).astype(np.float32), requires_grad=True)
        dy = Rng(124, 0).standard_normal((2048, 256)).astype(np.float32)
        res = moe_forward(x, layer, moe.gate)
        loss = sum_all(mul(res.output, Tensor(dy))) + importance_penalty(res.gates) * 0.01
        loss.backward()
        out[f"{rt}_y_rownorm"] = np.linalg.norm(res.output.data.astype(np.float64), axis=1)
        out[f"{rt}_dx_rownorm"] = np.linalg.norm(x.grad.astype(np.float64), axis=1)
        out[f"{rt}_dwg"] = layer.router.w_g.grad
        for w in ("w1", "w2", "w3"):
            out[f"{rt}_d{w}_norm"] = np.array([
                0.0 if getattr(ex, w).grad is None else np.linalg.norm(getattr(ex, w).grad.astype(np.float64))
                for ex in layer.experts])
        out[f"{rt}_assigned"] = res.stats.assigned
        out[f"{rt}_y_sum"] = np.array(res.output.data.astype(np.float64).sum())
    np.savez_compressed(os.path.join(OUT, "layer_cfg1.npz"), **out)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def upcycle_digests():
    tiny = ModelConfig(vocab=32, hidden=16, layers=2, heads=2, kv_heads=1, ffn_hidden=32, seq_len=16)
    d = {}
    for dt_name, dt in (("f32", np.float32), ("f64", np.float64)):
        dense = init_dense(tiny, seed=7, dtype=dt)
        full = upcycle_full(dense, n_experts=4, top_k=2, router_seed=5)
        d[f"tiny_{dt_name}_dense"] = {k: sha(v.data) for k, v in dense.tensors.items()}
        d[f"tiny_{dt_name}_full"] = {k: sha(v.data) for k, v in full.tensors.items()}
        for tp in (1, 2):
            for ep in (1, 2, 4):
                shards = [upcycle_shard(s, 4, 2, router_seed=5) for s in shard_dense(dense, tp, ep)]
                d[f"tiny_{dt_name}_shard_tp{tp}_ep{ep}"] = [
                    {"rank": s.rank, "tensors": {k: sha(v.data) for k, v in s.tensors.items()}} for s in shards]
    cfg1 = ModelConfig(vocab=32, hidden=256, layers=1, heads=4, kv_heads=2, ffn_hidden=512, seq_len=2048)
    dense = init_dense(cfg1, seed=7, dtype=np.float32)
    d["cfg1_f32_ffn"] = {w: sha(dense.tensors[f"layers.0.ffn.{w}"].data) for w in ("w1", "w2", "w3")}
    wg, wn = router_weights(cfg1, 8, 0, 1, np.float32)
    d["cfg1_f32_router_wg"] = sha(wg)
    d["cfg1_f32_router_wn"] = sha(wn)
    with open(os.path.join(OUT, "upcycle.json"), "w") as f:
        json.dump({"meta": json.loads(meta()), "digests": d}, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    routing_cfg1()
    routing_edge()
    layer_small()
    layer_cfg1()
    upcycle_digests()
    for n in sorted(os.listdir(OUT)):
        print(n, os.path.getsize(os.path.join(OUT, n)))
