"""EP parity on N GPUs (torchrun --nproc-per-node N tools/ep_check.py).

Every rank runs the expert-parallel layer (E/N experts, NCCL all-to-all) and
the single-GPU layer holding all experts on the same local batch, and checks:
routing bit-identical (gates, slot ranks), y and dx bit-identical (each row's
math is the same kernel on the same data), expert / router gradients equal to
the all-reduced single-GPU gradients within bf16 tolerance."""

import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_09952_b200 as P  # noqa: E402
from paper_2412_09952_b200.ep import ExpertParallelMoE  # noqa: E402


def rel(a, b):
    return float((a.double() - b.double()).norm() / b.double().norm().clamp_min(1e-30))


def case(rank, world, dev, T, H, F, router, policy, cf, noise, transport, E=8, k=2):
    El = E // world
    g = torch.Generator(device=dev).manual_seed(5)
    W1 = (torch.randn(E, F, H, generator=g, device=dev) * 0.05).to(torch.bfloat16)
    W2 = (torch.randn(E, H, F, generator=g, device=dev) * 0.05).to(torch.bfloat16)
    W3 = (torch.randn(E, F, H, generator=g, device=dev) * 0.05).to(torch.bfloat16)
    wg = torch.randn(H, E, generator=g, device=dev) * 0.05
    wn = torch.randn(H, E, generator=g, device=dev) * 0.02
    gx = torch.Generator(device=dev).manual_seed(100 + rank)
    x = torch.randn(T, H, generator=gx, device=dev).to(torch.bfloat16)
    dy = torch.randn(T, H, generator=gx, device=dev).to(torch.bfloat16)
    z = torch.randn(T, E, generator=gx, device=dev) if noise else None
    cfg = P.GateConfig(n_experts=E, top_k=k, router_type=router, noise_enabled=noise, capacity_factor=cf,
                       drop_policy=policy)
    own = slice(rank * El, (rank + 1) * El)

    # ---- expert parallel
    lw = [t.clone().requires_grad_() for t in (wg, wn, W1[own], W2[own], W3[own])]
    ep = ExpertParallelMoE(*lw, cfg, transport=transport)
    xe = x.clone().requires_grad_()
    oe = ep(xe, training=True, noise=z)
    loss = (oe.output.float() * dy.float()).sum() + 0.1 * P.importance_penalty(oe.gates)
    loss.backward()

    # ---- single GPU, all experts, same batch
    rw = [t.clone().requires_grad_() for t in (wg, wn, W1, W2, W3)]
    layer = P.MoELayer.from_stacked(P.RouterParams(rw[0], rw[1]), rw[2], rw[3], rw[4])
    xr = x.clone().requires_grad_()
    orf = P.moe_forward(xr, layer, cfg, training=True, noise=z)
    loss = (orf.output.float() * dy.float()).sum() + 0.1 * P.importance_penalty(orf.gates)
    loss.backward()
    torch.cuda.synchronize()

    ok = True
    msgs = []
    def check(name, cond):
        nonlocal ok
        if not cond:
            ok = False
            msgs.append(name)

    check("gates", torch.equal(oe.gates, orf.gates))
    check("slot_rank", torch.equal(oe.routing["slot_rank"], orf.routing["slot_rank"]))
    check("y", torch.equal(oe.output, orf.output))
    check("dx", rel(xe.grad, xr.grad) < 1e-2)
    for i, name in ((2, "dW1"), (3, "dW2"), (4, "dW3")):
        ref = rw[i].grad.float().clone()
        dist.all_reduce(ref)
        check(name, rel(lw[i].grad.float(), ref[own]) < 2e-2)
    refg = rw[0].grad.clone()
    dist.all_reduce(refg)
    check("dW_g", rel(lw[0].grad, refg) < 2e-2)
    if noise:
        refn = rw[1].grad.clone()
        dist.all_reduce(refn)
        check("dW_noise", rel(lw[1].grad, refn) < 2e-2)
    tag = f"[{transport}] T={T} H={H} F={F} E={E} k={k} {router} {policy} cf={cf} noise={noise}"
    print(f"rank {rank}: {'PASS' if ok else 'FAIL ' + ','.join(msgs)} {tag}", flush=True)
    return ok


def recompute_case(rank, world, dev, T=768, H=512, F=512, E=8, k=2):
    """p2p EP layer with selective recompute (a, b, h rebuilt by FWD1 in the
    backward) against the same layer keeping them: outputs and every gradient
    bit-identical (same kernels on the same inputs)."""
    El = E // world
    g = torch.Generator(device=dev).manual_seed(7)
    W = [(torch.randn(s_, generator=g, device=dev) * 0.05).to(torch.bfloat16) for s_ in ((El, F, H), (El, H, F),
                                                                                          (El, F, H))]
    wg = torch.randn(H, E, generator=g, device=dev) * 0.05
    gx = torch.Generator(device=dev).manual_seed(300 + rank)
    x = torch.randn(T, H, generator=gx, device=dev).to(torch.bfloat16)
    dy = torch.randn(T, H, generator=gx, device=dev).to(torch.bfloat16)
    cfg = P.GateConfig(n_experts=E, top_k=k, capacity_factor=2.0)
    res = []
    for rc in (False, True):
        lw = [t.clone().requires_grad_() for t in [wg, torch.zeros_like(wg)] + W]
        ep = ExpertParallelMoE(*lw, cfg, transport="p2p", buffer_slot=40 + int(rc), recompute=rc)
        xe = x.clone().requires_grad_()
        out = ep(xe)
        ((out.output.float() * dy.float()).sum() + 0.1 * P.importance_penalty(out.gates)).backward()
        torch.cuda.synchronize()
        res.append([out.output, xe.grad] + [t.grad for t in lw if t.grad is not None])
    # the pull variant of the return exchange (combine / router backward read the owners'
    # planes instead of rows FWD2 / BWD1 pushed): the same bits
    lw = [t.clone().requires_grad_() for t in [wg, torch.zeros_like(wg)] + W]
    ep = ExpertParallelMoE(*lw, cfg, transport="p2p", buffer_slot=44, gemm_push=False)
    xe = x.clone().requires_grad_()
    out = ep(xe)
    ((out.output.float() * dy.float()).sum() + 0.1 * P.importance_penalty(out.gates)).backward()
    torch.cuda.synchronize()
    res.append([out.output, xe.grad] + [t.grad for t in lw if t.grad is not None])
    ok = all(len(r) == len(res[0]) and all(torch.equal(a, b) for a, b in zip(res[0], r)) for r in res[1:])
    print(f"rank {rank}: {'PASS' if ok else 'FAIL'} [p2p recompute, pull exchange] bit-identical to keeping a, b, h "
          f"with the GEMM-pushed exchange", flush=True)
    return ok


def drop_h_case(rank, world, dev, T=768, H=512, F=512, E=8, k=2):
    """p2p EP layer that keeps a, b but not h (BWD2 rebuilds h for WGRAD)
    against the layer keeping h: y, dx, the router and dW1 / dW3 gradients
    bit-identical (the same kernels on the same a, b, da, db); dW2 = do^T h
    within bf16 rounding (the rebuilt h rounds silu(bf16 a) * bf16 b)."""
    El = E // world
    g = torch.Generator(device=dev).manual_seed(8)
    W = [(torch.randn(s_, generator=g, device=dev) * 0.05).to(torch.bfloat16) for s_ in ((El, F, H), (El, H, F),
                                                                                          (El, F, H))]
    wg = torch.randn(H, E, generator=g, device=dev) * 0.05
    gx = torch.Generator(device=dev).manual_seed(400 + rank)
    x = torch.randn(T, H, generator=gx, device=dev).to(torch.bfloat16)
    dy = torch.randn(T, H, generator=gx, device=dev).to(torch.bfloat16)
    cfg = P.GateConfig(n_experts=E, top_k=k, capacity_factor=2.0)
    res = []
    for dh in (False, True):
        lw = [t.clone().requires_grad_() for t in [wg, torch.zeros_like(wg)] + W]
        ep = ExpertParallelMoE(*lw, cfg, transport="p2p", buffer_slot=42 + int(dh), drop_h=dh)
        xe = x.clone().requires_grad_()
        out = ep(xe)
        ((out.output.float() * dy.float()).sum() + 0.1 * P.importance_penalty(out.gates)).backward()
        torch.cuda.synchronize()
        res.append(dict(y=out.output, dx=xe.grad, wg=lw[0].grad, w1=lw[2].grad, w3=lw[4].grad, w2=lw[3].grad))
    a, b = res
    exact = all(torch.equal(a[n], b[n]) for n in ("y", "dx", "wg", "w1", "w3"))
    r2 = rel(b["w2"], a["w2"])
    ok = exact and r2 < 1e-2
    print(f"rank {rank}: {'PASS' if ok else 'FAIL'} [p2p drop_h] y/dx/dW_g/dW1/dW3 bit-identical={exact}, "
          f"dW2 rel {r2:.2e}", flush=True)
    return ok


def graph_case(rank, world, dev, T=768, H=512, F=512, E=8, k=2):
    """The p2p EP layer step recorded into a CUDA graph (graphs.capture: device
    barriers, peer kernels, the GEMM-pushed exchange and the dW_g all_reduce
    are all stream work) replays the eager step's bits, also on new data
    copied into the captured inputs."""
    from paper_2412_09952_b200.graphs import capture
    El = E // world
    g = torch.Generator(device=dev).manual_seed(9)
    W = [(torch.randn(s_, generator=g, device=dev) * 0.05).to(torch.bfloat16).requires_grad_()
         for s_ in ((El, F, H), (El, H, F), (El, F, H))]
    wg = (torch.randn(H, E, generator=g, device=dev) * 0.05).requires_grad_()
    wn = torch.zeros(H, E, device=dev, requires_grad=True)
    gx = torch.Generator(device=dev).manual_seed(500 + rank)
    x = torch.randn(T, H, generator=gx, device=dev).to(torch.bfloat16).requires_grad_()
    dy = torch.randn(T, H, generator=gx, device=dev).to(torch.bfloat16)
    cfg = P.GateConfig(n_experts=E, top_k=k, capacity_factor=1.0)
    ep = ExpertParallelMoE(wg, wn, *W, cfg, transport="p2p", buffer_slot=46)
    params = [wg, wn, x] + W
    lam = torch.tensor(0.1, device=dev)

    def step():
        for p in params:
            p.grad = None
        out = ep(x)
        torch.autograd.backward([out.output, P.importance_penalty(out.gates)], [dy, lam])
        return out

    def snap(out):
        return [out.output.detach().clone()] + [p.grad.clone() for p in params if p.grad is not None]

    ref = snap(step())
    cap = capture(step, warmup=1)
    ok = True
    for _ in range(2):
        cap.replay()
        torch.cuda.synchronize()
        got = snap(cap.outputs)
        ok &= len(got) == len(ref) and all(torch.equal(a, b) for a, b in zip(got, ref))
    with torch.no_grad():
        x.copy_(torch.randn(T, H, generator=gx, device=dev).to(torch.bfloat16))
    cap.replay()
    torch.cuda.synchronize()
    got = snap(cap.outputs)
    want = snap(step())
    ok &= all(torch.equal(a, b) for a, b in zip(got, want))
    print(f"rank {rank}: {'PASS' if ok else 'FAIL'} [p2p graph] captured EP step replays the eager bits", flush=True)
    return ok


def oracle_case(rank, world, dev, T, H, F, router, policy, cf, noise, transport, E=8, k=2, lam=0.1):
    """EP layer against the CPU ORACLE (oracle/moe_oracle.py, the reference's
    closed form, moefold/moe.py:250-283) on each rank's own batch: routing
    bit-exact from the device logits, y / dx within the layer tolerances, and
    the owned experts' / router gradients against the oracle gradients summed
    over every rank's batch (rank-local capacity: SURVEY 8(e))."""
    import numpy as np
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import moe_oracle as O
    El = E // world
    g = O.rng(31, 0)
    bf = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).float().numpy()  # noqa
    w1 = [bf(g.standard_normal((H, F)) * 0.05) for _ in range(E)]
    w2 = [bf(g.standard_normal((F, H)) * 0.05) for _ in range(E)]
    w3 = [bf(g.standard_normal((H, F)) * 0.05) for _ in range(E)]
    wg = (g.standard_normal((H, E)) * 0.1).astype(np.float32)
    wn = (g.standard_normal((H, E)) * 0.05).astype(np.float32)
    x = bf(O.rng(123, rank).standard_normal((T, H)))
    dy = bf(O.rng(124, rank).standard_normal((T, H)))
    z = O.rng(5, rank).standard_normal((T, E)).astype(np.float32)
    cfg = P.GateConfig(n_experts=E, top_k=k, router_type=router, noise_enabled=noise, capacity_factor=cf,
                       drop_policy=policy)
    own = range(rank * El, (rank + 1) * El)
    stack = lambda ws: torch.stack([torch.from_numpy(ws[e].T.copy()) for e in own]).to(dev, torch.bfloat16)  # noqa
    lw = [torch.from_numpy(wg).to(dev).requires_grad_(), torch.from_numpy(wn).to(dev).requires_grad_()]
    lw += [stack(ws).requires_grad_() for ws in (w1, w2, w3)]
    ep = ExpertParallelMoE(*lw, cfg, transport=transport)
    xe = torch.from_numpy(x).to(dev, torch.bfloat16).requires_grad_()
    out = ep(xe, training=True, noise=torch.from_numpy(z).to(dev) if noise else None)
    aux = P.importance_penalty(out.gates)
    torch.autograd.backward([out.output, aux], [torch.from_numpy(dy).to(dev, torch.bfloat16),
                                                torch.tensor(lam, device=dev)])
    torch.cuda.synchronize()

    logits = out.routing["logits"].cpu().numpy()
    ocfg = O.LayerCfg(n_experts=E, top_k=k, router_type=router, noise=noise, capacity_factor=cf, drop_policy=policy)
    y_o, g_o, cache = O.moe_forward(x, wg, wn, w1, w2, w3, ocfg, z=z if noise else None, logits=logits)
    _, dimp = O.importance_penalty(g_o)
    gr = O.moe_backward(cache, dy, dgates=lam * dimp)
    relnp = lambda a, b: float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-30))  # noqa
    ok, msgs = True, []

    def check(name, cond):
        nonlocal ok
        if not cond:
            ok = False
            msgs.append(name)

    check("gates", out.gates.detach().cpu().numpy().tobytes() == g_o.tobytes())
    check("slot_rank", np.array_equal(out.routing["slot_rank"].cpu().numpy(), cache.disp.rows()))
    check("assigned", np.array_equal(out.stats.assigned, cache.disp.assigned))
    check("y", relnp(out.output.detach().float().cpu().numpy(), y_o) < 1.5e-2)
    check("dx", relnp(xe.grad.float().cpu().numpy(), gr["dx"]) < 1.5e-2)
    # weight gradients: oracle per rank, summed over ranks (the EP owner sums every source's rows)
    for i, name in ((2, "dw1"), (3, "dw2"), (4, "dw3")):
        ref = torch.from_numpy(np.ascontiguousarray(np.stack([gr[name][e].T for e in range(E)]), np.float32)).to(dev)
        dist.all_reduce(ref)
        check(name, relnp(lw[i].grad.float().cpu().numpy(), ref[rank * El:(rank + 1) * El].cpu().numpy()) < 2e-2)
    for i, name in ((0, "dwg"), (1, "dwn")):
        if name == "dwn" and not noise:
            continue
        ref = torch.from_numpy(np.ascontiguousarray(gr[name], np.float32)).to(dev)
        dist.all_reduce(ref)
        check(name, relnp(lw[i].grad.cpu().numpy(), ref.cpu().numpy()) < 2e-2)
    tag = f"[{transport} vs ORACLE] T={T} H={H} F={F} E={E} k={k} {router} {policy} cf={cf} noise={noise}"
    print(f"rank {rank}: {'PASS' if ok else 'FAIL ' + ','.join(msgs)} {tag}", flush=True)
    return ok


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    ok = True
    for transport in ("p2p", "nccl"):
        for args in [(1024, 512, 768, "mixtral", "position", 1.0, False),
                     (1000, 512, 512, "st", "score", 2.0, True),
                     (512, 256, 512, "mixtral", "position", None, False),
                     (2048, 1024, 1024, "mixtral", "position", 0.5, False)]:
            ok &= case(rank, world, dev, *args, transport)
        # more experts than E8T2 and a wider fan-out (E/N experts per rank, k=4)
        ok &= case(rank, world, dev, 768, 512, 512, "st", "score", None, True, transport, E=16, k=4)
        # one expert per rank, as EP8 runs E8T2 (E_local = 1: every segment of the local expert GEMMs
        # comes from a different source rank)
        ok &= case(rank, world, dev, 1024, 512, 512, "mixtral", "position", 1.0, False, transport, E=world, k=2)
        # against the CPU oracle directly (not the single-GPU CUDA layer)
        ok &= oracle_case(rank, world, dev, 512, 256, 512, "mixtral", "position", 1.0, True, transport)
        ok &= oracle_case(rank, world, dev, 384, 256, 256, "st", "score", None, False, transport)
    ok &= recompute_case(rank, world, dev)
    ok &= drop_h_case(rank, world, dev)
    ok &= graph_case(rank, world, dev)
    # canary bands around every symmetric receive plane (written by peers over NVLink) untouched
    from paper_2412_09952_b200.ep import _PeerBuffers
    torch.cuda.synchronize()
    dist.barrier()
    guards = all(pb.guards_intact() for pb in _PeerBuffers._cache.values())
    print(f"rank {rank}: {'PASS' if guards else 'FAIL'} symmetric-buffer guard bands "
          f"({len(_PeerBuffers._cache)} buffer sets)", flush=True)
    ok &= guards
    flag = torch.tensor([0 if ok else 1], device=dev)
    dist.all_reduce(flag)
    dist.destroy_process_group()
    sys.exit(int(flag.item() != 0))


if __name__ == "__main__":
    main()
