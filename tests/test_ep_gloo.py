"""Expert-parallel host logic on CPU with the gloo backend (world size 2 and 4).

The EP data movement of paper_2412_09952_b200.ep (EPPlan: fixed-capacity
segments, counts exchange, equal-split row all-to-all, segment tables of the
received rows) is driven end to end with the CPU oracle standing in for the
CUDA kernels, and each rank's output / gradients are compared with the oracle
run on that rank's batch alone (rank-local capacity makes them identical)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import moe_oracle as O


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ffn(x, w1, w2, w3):
    a = x @ w1
    b = x @ w3
    return ((a * O.sigmoid(a)) * b) @ w2


def _worker(rank, world, port, cf, policy, router, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2412_09952_b200.ep import EPPlan
        T, H, F, E = 64, 16, 24, 8
        g = O.rng(10, 0)
        wg = (g.standard_normal((H, E)) * 0.5).astype(np.float32)
        w1 = [(g.standard_normal((H, F)) * 0.3).astype(np.float32) for _ in range(E)]
        w2 = [(g.standard_normal((F, H)) * 0.3).astype(np.float32) for _ in range(E)]
        w3 = [(g.standard_normal((H, F)) * 0.3).astype(np.float32) for _ in range(E)]
        x = O.rng(123, rank).standard_normal((T, H)).astype(np.float32)
        cfg = O.LayerCfg(n_experts=E, top_k=2, router_type=router, capacity_factor=cf, drop_policy=policy)
        y_ref, gates, cache = O.moe_forward(x, wg, np.zeros_like(wg), w1, w2, w3, cfg)

        plan = EPPlan.make(world, rank, E, T, cf)
        assert plan.capacity == cache.disp.capacity
        rows = cache.disp.rows()
        send = torch.zeros(plan.send_rows, H)
        counts = torch.tensor(cache.disp.assigned, dtype=torch.int32)
        for t, e in zip(*np.nonzero(rows >= 0)):
            send[e * plan.cap_pad + rows[t, e]] = torch.from_numpy(x[t])
        rcounts = plan.exchange_counts(counts)
        allc = [torch.empty_like(counts) for _ in range(world)]
        dist.all_gather(allc, counts)
        expect = torch.stack([c[plan.owned.start:plan.owned.stop] for c in allc]).reshape(-1)
        assert torch.equal(rcounts, expect)
        recv = plan.exchange_rows(torch.empty_like(send), send)
        base, expert = plan.recv_segments("cpu")
        o_recv = torch.zeros_like(recv)
        for s in range(world * plan.e_local):
            b, c = int(base[s]), int(rcounts[s])
            e = plan.owned.start + int(expert[s])
            if c:
                o_recv[b:b + c] = torch.from_numpy(_ffn(recv[b:b + c].numpy(), w1[e], w2[e], w3[e]))
        o_send = plan.exchange_rows(torch.empty_like(o_recv), o_recv)
        y = np.zeros_like(x)
        for t in range(T):
            for e in range(E):
                if rows[t, e] >= 0:
                    y[t] += gates[t, e] * o_send[e * plan.cap_pad + rows[t, e]].numpy()
        err = float(np.abs(y - y_ref).max() / max(np.abs(y_ref).max(), 1e-30))
        out_q.put((rank, err, int(rcounts.sum())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cf,policy,router",
                         [(w, *c) for w in (2, 4) for c in ((1.0, "position", "mixtral"), (0.5, "score", "st"),
                                                           (None, "position", "mixtral"))]
                         + [(8, 1.0, "position", "mixtral")])   # one expert per rank, as on an 8-GPU box
def test_ep_plan_matches_rank_local_oracle(world, cf, policy, router):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cf, policy, router, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, _ in res:
        assert err < 1e-5, (rank, err)


def test_ep_plan_layout_rules():
    from paper_2412_09952_b200.ep import EPPlan
    from paper_2412_09952_b200.errors import ConfigError
    p = EPPlan.make(4, 1, 8, 8192, 1.0)
    assert (p.capacity, p.cap_pad, p.e_local, list(p.owned), p.send_rows) == (1024, 1024, 2, [2, 3], 8 * 1024)
    base, expert = p.recv_segments("cpu")
    assert base.tolist() == [i * 1024 for i in range(8)] and expert.tolist() == [0, 1] * 4
    assert EPPlan.make(2, 0, 8, 100, 1.0).cap_pad == 128          # ceil(100/8)=13 -> padded to 128
    assert EPPlan.make(2, 0, 8, 300, None).cap_pad == 384         # dropless: T rows per expert segment
    with pytest.raises(ConfigError):
        EPPlan.make(3, 0, 8, 64, 1.0)


def _tokens_worker(rank, world, port, same, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2412_09952_b200 import GateConfig
        from paper_2412_09952_b200.errors import ShapeError
        from paper_2412_09952_b200.ep import ExpertParallelMoE
        E, H, F = 4, 256, 256
        layer = ExpertParallelMoE(torch.zeros(H, E), torch.zeros(H, E), torch.zeros(E // world, F, H),
                                  torch.zeros(E // world, H, F), torch.zeros(E // world, F, H),
                                  GateConfig(n_experts=E, top_k=2, capacity_factor=1.0))
        T = 64 if same or rank == 0 else 32
        try:
            layer._check_tokens(T, torch.device("cpu"))
            out_q.put((rank, "ok"))
        except ShapeError as e:
            out_q.put((rank, "shape:" + str(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("same", [True, False])
def test_p2p_transport_rejects_unequal_tokens_per_rank(same):
    """the p2p receive segments are sized from T_local on every rank,
    so ranks with different T must raise ShapeError instead of writing past a
    smaller peer's buffer."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tokens_worker, args=(r, world, port, same, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    if same:
        assert res == {0: "ok", 1: "ok"}
    else:
        assert all(v.startswith("shape:") and "disagree on tokens" in v for v in res.values()), res
