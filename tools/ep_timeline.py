"""Kernel timeline of the expert-parallel layer step on every rank
(torchrun --nproc-per-node N tools/ep_timeline.py [--eager]): torch.profiler
(CUPTI activity) over 3 steps of the bench configuration (T=8192/rank,
H=4096, F=14336, E=8, k=2, CF 1, p2p transport), the step launched from a
CUDA graph like bench.py.  Writes gpurun_out/ep_timeline_r{rank}.json: per
kernel name total / count / mean, and the idle time between kernels on the
compute stream, so the non-GEMM share of an EP step can be attributed
(peer exchange, device barriers, all_reduce, gaps)."""

import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_09952_b200 as P  # noqa: E402
from paper_2412_09952_b200.ep import ExpertParallelMoE  # noqa: E402
from paper_2412_09952_b200.graphs import capture  # noqa: E402
from paper_2412_09952_b200.upcycle import router_weights, upcycle_experts  # noqa: E402


def main():
    eager = "--eager" in sys.argv
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    H, F, E, K, T = 4096, 14336, 8, 2, 8192
    torch.manual_seed(0)
    w1 = (torch.randn(H, F, device=dev) * 0.02).to(torch.bfloat16)
    w2 = (torch.randn(F, H, device=dev) * 0.02).to(torch.bfloat16)
    w3 = (torch.randn(H, F, device=dev) * 0.02).to(torch.bfloat16)
    W1, W2, W3 = (w.requires_grad_() for w in upcycle_experts(w1, w2, w3, E // world))
    cfg_m = P.ModelConfig(vocab=32, hidden=H, layers=1, heads=32, kv_heads=8, ffn_hidden=F, seq_len=T)
    wg, wn = router_weights(cfg_m, E, 0, 1, torch.float32, dev)
    wg.requires_grad_()
    wn.requires_grad_()
    gate = P.GateConfig(n_experts=E, top_k=K, capacity_factor=1.0)
    layer = ExpertParallelMoE(wg, wn, W1, W2, W3, gate, transport="p2p")
    g = torch.Generator(device=dev).manual_seed(1000 + rank)
    x = torch.randn(T, H, device=dev, generator=g).to(torch.bfloat16).requires_grad_()
    dy = torch.randn(T, H, device=dev, generator=g).to(torch.bfloat16)
    lam = torch.tensor(0.01, device=dev)
    params = [W1, W2, W3, wg, wn, x]

    def step():
        for p in params:
            p.grad = None
        out = layer(x)
        aux = P.importance_penalty(out.gates)
        torch.autograd.backward([out.output, aux], [dy, lam])

    for _ in range(20):
        step()
    torch.cuda.synchronize()
    cap = None if eager else capture(step, repeat=3, warmup=0)
    if cap is not None:
        cap.replay()
    torch.cuda.synchronize()
    dist.barrier()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        if cap is not None:
            cap.replay()
        else:
            for _ in range(3):
                step()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    kern = {}
    spans = []
    for e in evs:
        name = e.name
        d = e.time_range.end - e.time_range.start
        k = kern.setdefault(name, [0.0, 0])
        k[0] += d
        k[1] += 1
        spans.append((e.time_range.start, e.time_range.end, name))
    spans.sort()
    # union busy time and gaps (all streams together)
    busy, cur_s, cur_e = 0.0, None, None
    for s, e, _ in spans:
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                busy += cur_e - cur_s
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    if cur_e is not None:
        busy += cur_e - cur_s
    total = spans[-1][1] - spans[0][0] if spans else 0
    out = {"rank": rank, "world": world, "launch": "eager" if eager else "graph", "steps": 3,
           "window_us": total, "busy_us": busy, "idle_us": total - busy,
           "kernels": sorted(([n, round(t / 3, 1), c // 3, round(t / c, 1)] for n, (t, c) in kern.items()),
                             key=lambda r: -r[1]),
           "sequence_first_step": [(round(s - spans[0][0], 1), round(e - s, 1), n[:80]) for s, e, n in spans[:60]]}
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/ep_timeline_{'eager' if eager else 'graph'}_r{rank}.json", "w") as f:
        json.dump(out, f, indent=1)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
