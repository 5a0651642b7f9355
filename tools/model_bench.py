"""Model-level training-step benchmark:
a Llama-3-8B-shape E8T2 model with `--layers` transformer blocks (all MoE),
one full step = forward + cross-entropy + aux loss + backward + Adam over every
parameter, on one GPU.  Weights are random-init on the device (synthetic), the
batch is one sequence of `--seq` random token ids.  `--micro-batches M` runs M
forward+backward passes per optimizer step (gradient accumulation, as the
paper's global batch does over its micro-batches): gradients accumulate in the
leaves' dtype (expert weights inside the weight-gradient GEMM, fp32 add, unless
--no-fused-acc), the data-parallel reduction and the overlapped optimizer act in
the last backward only.

Prints one JSON line: tokens/s, ms/step, model MFU with the reference's
forward_flops(..., "6P") convention (plan.py:195-215) with the expert term
counted on kept slots, and a per-phase split measured with CUDA events.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_09952_b200 as P  # noqa: E402
from paper_2412_09952_b200.train import DataParallelGrads, OverlappedStep, TrainState  # noqa: E402


def model_flops(cfg, gate, tokens: int, kept_slots: int) -> float:
    """6 x matmul MACs of plan.py:forward_flops with S (kept slots) in place of
    tokens * top_k for the expert FFNs."""
    H, F, E = cfg.hidden, cfg.ffn_hidden, gate.n_experts
    attn = 2 * H * H + 2 * H * cfg.kv_width
    per_layer = tokens * (attn + H * E) + kept_slots * 3 * H * F
    macs = tokens * H * cfg.vocab + cfg.layers * per_layer
    macs += cfg.layers * 2 * tokens * min(tokens, cfg.seq_len) * H
    return 6.0 * macs


def random_dense(cfg, device):
    g = torch.Generator(device=device)
    g.manual_seed(0)
    tensors = {}
    for name, shape in sorted(P.dense_schema(cfg).items()):
        if name.endswith("norm"):
            tensors[name] = torch.ones(shape, dtype=torch.float32, device=device)
        else:
            tensors[name] = torch.randn(shape, generator=g, dtype=torch.float32, device=device) * 0.02
    return P.DenseCheckpoint(config=cfg, tensors=tensors)


def profile_step(step, rank, world):
    """One step under torch.profiler: device time per kernel name, the busy
    (union) time and the window, written to gpurun_out/model_prof_r<rank>.json."""
    from torch.profiler import ProfilerActivity, profile
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step()
        torch.cuda.synchronize()
    spans, per = [], {}
    for e in prof.events():
        if e.device_type != torch.autograd.DeviceType.CUDA:
            continue
        d = e.time_range.end - e.time_range.start
        k = per.setdefault(e.name[:120], [0.0, 0])
        k[0] += d
        k[1] += 1
        spans.append((e.time_range.start, e.time_range.end))
    spans.sort()
    busy, cs, ce = 0.0, None, None
    for s_, e_ in spans:
        if ce is None or s_ > ce:
            if ce is not None:
                busy += ce - cs
            cs, ce = s_, e_
        else:
            ce = max(ce, e_)
    if ce is not None:
        busy += ce - cs
    out = {"rank": rank, "window_us": (spans[-1][1] - spans[0][0]) if spans else 0, "busy_us": busy,
           "kernels": sorted(([n, round(t, 1), c] for n, (t, c) in per.items()), key=lambda r: -r[1])[:60]}
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/model_prof_r{rank}.json", "w") as f:
        json.dump(out, f, indent=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--seq", type=int, default=8192)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--cf", type=float, default=1.0)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--small", action="store_true", help="tiny shape for a smoke run")
    ap.add_argument("--no-shadows", action="store_true", help="cast fp32 GEMM weights per step instead")
    ap.add_argument("--transport", default="p2p", choices=("p2p", "nccl"))
    ap.add_argument("--micro-batches", type=int, default=1, help="forward+backward passes per optimizer step")
    ap.add_argument("--no-fused-acc", action="store_true",
                    help="accumulate expert gradients with autograd adds instead of inside the WGRAD GEMM")
    ap.add_argument("--serial-opt", action="store_true",
                    help="optimizer after the backward in one launch (default: overlapped with the backward)")
    ap.add_argument("--experts", type=int, default=8, help="experts per MoE layer (E8T2 = 8)")
    ap.add_argument("--recompute", type=int, default=0,
                    help="MoE layers (the first N, p2p EP) that rebuild a, b, h in the backward instead of keeping them")
    ap.add_argument("--cublas-proj", action="store_true",
                    help="A/B only: qkv / wo / lm-head through torch.matmul (cuBLAS) instead of the repo's tcgen05 GEMM")
    ap.add_argument("--dense-grid", type=int, default=0,
                    help="persistent-grid cap of the projection GEMMs (0 = all SMs; caps measured no faster)")
    ap.add_argument("--zero", action="store_true",
                    help="ZeRO-1: shard the replicated tensors' optimizer state over the ranks")
    ap.add_argument("--drop-h", action="store_true",
                    help="MoE layers outside the recompute set keep a, b but not h (BWD2 rebuilds it)")
    ap.add_argument("--profile", action="store_true",
                    help="after the timed steps, one more step under torch.profiler (CUPTI kernel records) on every "
                         "rank: kernel time by name -> gpurun_out/model_prof_r<rank>.json")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = 0
    group = None
    if world > 1:   # torchrun: EP over all ranks for the MoE layers, DP for the rest
        import torch.distributed as dist
        local = int(os.environ["LOCAL_RANK"])
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        rank, group = dist.get_rank(), dist.group.WORLD
    dev = torch.device("cuda", torch.cuda.current_device())
    import paper_2412_09952_b200.tensor as PT0
    PT0.set_dense_grid(a.dense_grid)
    if a.cublas_proj:
        import paper_2412_09952_b200.tensor as PT
        PT.linear = lambda x, w: x.to(torch.bfloat16) @ w.to(torch.bfloat16)   # noqa: E731
    if a.small:
        cfg = P.ModelConfig(vocab=1024, hidden=512, layers=a.layers, heads=8, kv_heads=2, ffn_hidden=1024,
                            seq_len=a.seq)
    else:
        cfg = P.ModelConfig(vocab=128256, hidden=4096, layers=a.layers, heads=32, kv_heads=8, ffn_hidden=14336,
                            seq_len=a.seq)
    dense = random_dense(cfg, dev)
    if world > 1:   # online upcycling of this rank's experts only (upcycle.py:187-227)
        moe = P.upcycle_shard(P.shard_dense(dense, 1, world)[rank], a.experts, 2, router_seed=1,
                              capacity_factor=a.cf)
    else:
        moe = P.upcycle_full(dense, a.experts, 2, router_seed=1, capacity_factor=a.cf)
    del dense
    torch.cuda.empty_cache()
    state = TrainState(moe, shadows=not a.no_shadows)
    if a.zero and (world == 1 or a.serial_opt):
        raise SystemExit("--zero needs N > 1 ranks and the overlapped optimizer")
    opt = state.optimizer("adam", zero_group=group if a.zero else None)
    ov = None if a.serial_opt else OverlappedStep(opt, group)
    dp = DataParallelGrads(state.leaves, group) if (world > 1 and ov is None) else None
    rng = np.random.default_rng(rank)
    M = a.micro_batches
    P.moe.set_expert_grad_accumulation_fusion(M > 1 and not a.no_fused_acc)
    batches = []
    for _ in range(M):
        tokens = rng.integers(0, cfg.vocab, (a.batch, a.seq + 1))
        batches.append((tokens[:, :-1], tokens[:, 1:].reshape(-1)))
    T = a.batch * a.seq * M   # tokens per optimizer step (this rank)
    aux = 0.01

    def step(ev=None):
        if ev is not None:
            ev[0].record()
        for p in opt.params.values():
            p.grad = None
        stats = []
        for mb, (inputs, targets) in enumerate(batches):
            last = mb == M - 1
            fwd = P.forward_with_stats(moe, inputs, training=True, compute=state.compute, ep_group=group,
                                       transport=a.transport, recompute_layers=range(a.recompute),
                                       drop_h_layers=range(cfg.layers) if a.drop_h else ())
            loss = P.cross_entropy(fwd.logits, targets)
            for g in fwd.gates:
                loss = loss + (aux / len(fwd.gates)) * P.importance_penalty(g)
            loss = loss / (world * M)
            if ev is not None and mb == 0:
                ev[1].record()
            if ov is not None and last:
                ov.begin(1e-4)
            if dp is not None:
                dp.enabled = last
            loss.backward()
            stats += fwd.stats
            del fwd
        if dp is not None:
            dp.wait()
        if ev is not None:
            ev[2].record()
        if ov is not None:
            ov.finish()          # updates ran on the side stream during the backward
        else:
            opt.step(1e-4)
        if ev is not None:
            ev[3].record()
        return loss, stats

    from bench import ClockSampler
    clk = ClockSampler(dev.index)   # started before the warm-up (see bench.run_single)
    for _ in range(a.warmup):
        loss, stats = step()
    torch.cuda.synchronize()
    kept = sum(int(s.assigned.sum()) for s in stats) // cfg.layers   # this rank's tokens' kept slots
    if world > 1:
        dist.barrier()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(a.steps)]
    with clk:
        t0 = time.perf_counter()
        for i in range(a.steps):
            loss, _ = step(evs[i])
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / a.steps
    clocks = clk.summary()
    if a.profile:
        profile_step(step, rank, world)
    ms = float(np.median([e[0].elapsed_time(e[3]) for e in evs]))
    if world > 1:   # the step takes as long as the slowest rank
        t = torch.tensor([ms, float(kept)], device=dev, dtype=torch.float64)
        dist.all_reduce(t[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:], op=dist.ReduceOp.SUM)
        ms, kept = float(t[0]), int(t[1]) // world
    split = {k: round(float(np.median([e[i].elapsed_time(e[i + 1]) for e in evs])), 3)
             for i, k in enumerate(("forward_mb0", "fwd_bwd_rest", "optimizer"))}
    flops = world * model_flops(cfg, moe.gate, T, kept)
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
    n_params = sum(t.numel() for t in opt.params.values())
    if rank != 0:
        dist.destroy_process_group()
        return
    out = {
        "metric": f"Llama-3-8B-shape E{a.experts}T2 {cfg.layers}-layer training step tokens/s",
        "value": round(world * T / (ms * 1e-3), 1), "unit": "tokens/s", "ms_per_step": round(ms, 3),
        "n_gpus": world, "parallelism": f"ep{world} (MoE) + dp{world} (rest)" if world > 1 else "single GPU",
        "wall_ms_per_step": round(wall * 1e3, 3), "phases_ms": split,
        "mfu": {"measured_peak": round(flops / (ms * 1e-3) / (world * peaks["bf16_tflops"] * 1e12), 4),
                "spec_2250": round(flops / (ms * 1e-3) / (world * 2250e12), 4), "flops_per_step": flops,
                "convention": "6P (plan.py:forward_flops) with kept slots for the expert FFNs"},
        "loss": float(loss.detach()) * world * M, "micro_batches": M,
        "expert_grad_accumulation": "fused into WGRAD" if (M > 1 and not a.no_fused_acc) else "autograd", "kept_slots_per_layer_per_rank": kept, "params_rank0": n_params,
        "max_mem_gb": round(torch.cuda.max_memory_allocated() / 2**30, 1),
        "optimizer_state_gb_rank0": round(opt.state_bytes() / 2**30, 2), "zero1": bool(a.zero),
        "recompute_moe_layers": a.recompute, "drop_h": bool(a.drop_h),
        "projections": "torch.matmul (cuBLAS), A/B run" if a.cublas_proj else
        f"tcgen05 dense GEMM (tensor.linear), grid cap {PT0._DENSE_GRID or 148}",
        "clocks": clocks,
        "config": {"vocab": cfg.vocab, "hidden": cfg.hidden, "layers": cfg.layers, "heads": cfg.heads,
                   "kv_heads": cfg.kv_heads, "ffn": cfg.ffn_hidden, "seq": a.seq, "batch": a.batch, "experts": a.experts,
                   "top_k": 2, "capacity_factor": a.cf,
                   "optimizer": "adam (fp32 masters), " + ("after the backward" if a.serial_opt else
                                                           "per tensor on a side stream during the backward")},
        "data": "synthetic (random token ids, random-init weights)",
    }
    print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
