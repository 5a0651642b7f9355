"""Data-parallel gradient reduction of the model step (train.DataParallelGrads)
on CPU with the gloo backend: replicated leaves are all-reduced as their
gradients appear during the backward, expert stacks and the self-reduced
embedding are left alone, and the result equals the gradient of the summed
per-rank losses."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2412_09952_b200.train import DataParallelGrads
        torch.manual_seed(0)                     # identical replicated weights on every rank
        leaves = {
            "lm_head": torch.randn(6, 5, requires_grad=True),
            "layers.0.attn_norm": torch.randn(6, requires_grad=True),
            "layers.0.moe.router.wnoise": torch.randn(6, 3, requires_grad=True),   # gets no gradient
            "layers.0.moe.experts.W1": torch.randn(2, 4, 6, requires_grad=True),  # EP-owned: not reduced
            "embedding": torch.randn(7, 6, requires_grad=True),                     # reduced inside its op
        }
        dp = DataParallelGrads(leaves)
        x = torch.full((3, 6), float(rank + 1))
        h = x * leaves["layers.0.attn_norm"]
        loss = (h @ leaves["lm_head"]).pow(2).sum() + (leaves["layers.0.moe.experts.W1"] * (rank + 1)).sum() \
            + (leaves["embedding"] * (rank + 1)).sum()
        loss.backward()
        dp.wait()
        dp.remove()
        # numpy, not tensors: a tensor is shared by fd and the sender may exit first
        q.put((rank, {k: (None if v.grad is None else v.grad.numpy().copy()) for k, v in leaves.items()}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_data_parallel_grads_sum_replicated_only(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # reference: each rank's gradient computed alone, summed for the replicated leaves
    torch.manual_seed(0)
    base = {"lm_head": torch.randn(6, 5), "layers.0.attn_norm": torch.randn(6)}
    want = {k: torch.zeros_like(v) for k, v in base.items()}
    for r in range(world):
        ls = {k: v.clone().requires_grad_(True) for k, v in base.items()}
        x = torch.full((3, 6), float(r + 1))
        ((x * ls["layers.0.attn_norm"]) @ ls["lm_head"]).pow(2).sum().backward()
        for k in want:
            want[k] += ls[k].grad
    for r in range(world):
        g = {k: (None if v is None else torch.from_numpy(v)) for k, v in res[r].items()}
        for k in want:
            torch.testing.assert_close(g[k], want[k], rtol=1e-5, atol=1e-5)
        assert g["layers.0.moe.router.wnoise"] is None
        torch.testing.assert_close(g["layers.0.moe.experts.W1"], torch.full((2, 4, 6), float(r + 1)))
        torch.testing.assert_close(g["embedding"], torch.full((7, 6), float(r + 1)))


def _worker_mb(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2412_09952_b200.train import DataParallelGrads
        torch.manual_seed(0)
        w = torch.randn(4, 3, requires_grad=True)
        dp = DataParallelGrads({"lm_head": w})
        for mb in range(3):                      # three micro-batches, reduction armed for the last only
            dp.enabled = mb == 2
            x = torch.full((2, 4), float(rank + 1 + 10 * mb))
            (x @ w).pow(2).sum().backward()
        dp.wait()
        dp.remove()
        q.put((rank, w.grad.numpy().copy()))
    finally:
        dist.destroy_process_group()


def test_data_parallel_grads_micro_batches_reduce_once():
    """Gradient accumulation (tools/model_bench.py --micro-batches): with the
    reduction disarmed for all but the last backward, each rank's summed
    micro-batch gradients are all-reduced exactly once."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_mb, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    torch.manual_seed(0)
    w0 = torch.randn(4, 3)
    want = torch.zeros(4, 3)
    for r in range(world):
        for mb in range(3):
            w = w0.clone().requires_grad_(True)
            (torch.full((2, 4), float(r + 1 + 10 * mb)) @ w).pow(2).sum().backward()
            want += w.grad
    for r in range(world):
        torch.testing.assert_close(torch.from_numpy(res[r]), want, rtol=1e-5, atol=1e-4)
