"""Kernel-time breakdown of one model training step (tools/model_bench.py's
step, single GPU) with torch.profiler (CUPTI kernel records): top kernels by
total device time, grouped into MoE (b200moe GEMMs / small kernels), library
GEMM/attention and elementwise.  Diagnostics only; bench numbers come from
model_bench.py."""

import argparse
import json
import os
import sys
from collections import defaultdict

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_09952_b200 as P  # noqa: E402
from paper_2412_09952_b200.train import OverlappedStep, TrainState  # noqa: E402
from tools.model_bench import random_dense  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=2)
ap.add_argument("--seq", type=int, default=8192)
ap.add_argument("--micro-batches", type=int, default=2)
ap.add_argument("--top", type=int, default=30)
a = ap.parse_args()
dev = torch.device("cuda")
cfg = P.ModelConfig(vocab=128256, hidden=4096, layers=a.layers, heads=32, kv_heads=8, ffn_hidden=14336, seq_len=a.seq)
moe = P.upcycle_full(random_dense(cfg, dev), 8, 2, router_seed=1, capacity_factor=1.0)
state = TrainState(moe)
opt = state.optimizer("adam")
ov = OverlappedStep(opt)
rng = np.random.default_rng(0)
M = a.micro_batches
batches = []
for _ in range(M):
    tok = rng.integers(0, cfg.vocab, (1, a.seq + 1))
    batches.append((tok[:, :-1], tok[:, 1:].reshape(-1)))


def step():
    for p in opt.params.values():
        p.grad = None
    for mb, (inp, tgt) in enumerate(batches):
        fwd = P.forward_with_stats(moe, inp, training=True, compute=state.compute)
        loss = P.cross_entropy(fwd.logits, tgt)
        for g in fwd.gates:
            loss = loss + (0.01 / len(fwd.gates)) * P.importance_penalty(g)
        loss = loss / M
        if mb == M - 1:
            ov.begin(1e-4)
        loss.backward()
        del fwd
    ov.finish()


for _ in range(3):
    step()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
agg, cnt = defaultdict(float), defaultdict(int)
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        agg[ev.name] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
        cnt[ev.name] += 1
tot = sum(agg.values())


def group(n):
    if "moe_gemm_kernel" in n:
        return "moe grouped GEMM"
    if "b200moe" in n:
        return "b200moe other"
    if "nvjet" in n or "gemm" in n.lower() or "cutlass" in n:
        return "library GEMM"
    if "sdpa" in n or "flash" in n or "fmha" in n:
        return "attention"
    return "torch elementwise/other"


groups = defaultdict(float)
for n, t in agg.items():
    groups[group(n)] += t
print(json.dumps({"layers": a.layers, "micro_batches": M, "device_ms_total": round(tot / 1e3, 3),
                  "groups_ms": {k: round(v / 1e3, 3) for k, v in sorted(groups.items(), key=lambda x: -x[1])}}))
for n, t in sorted(agg.items(), key=lambda x: -x[1])[:a.top]:
    print(f"{t / 1e3:9.3f} ms {100 * t / tot:5.1f}% {cnt[n]:5d}  {n[:110]}")
