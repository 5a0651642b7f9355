"""Kernel timeline of the N=1 layer step (bench configuration, CUDA-graph
launch like bench.py): torch.profiler (CUPTI) over 3 replayed steps; prints
every kernel of the middle step with its start offset, duration and the idle
gap before it, and the step's busy / idle totals -- where launch gaps and
kernel prologues cost time between the 13 launches.

    python tools/step_timeline.py > gpurun_out/step_timeline.json
"""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_09952_b200 as B  # noqa: E402
from paper_2412_09952_b200.graphs import capture  # noqa: E402
from paper_2412_09952_b200.upcycle import router_weights, upcycle_experts  # noqa: E402

H, F, E, K, T = 4096, 14336, 8, 2, 8192


def main():
    dev = torch.device("cuda")
    torch.manual_seed(0)
    w = [(torch.randn(s, device=dev) * 0.02).to(torch.bfloat16) for s in ((H, F), (F, H), (H, F))]
    W1, W2, W3 = (t.requires_grad_() for t in upcycle_experts(*w, E))
    cfg_m = B.ModelConfig(vocab=32, hidden=H, layers=1, heads=32, kv_heads=8, ffn_hidden=F, seq_len=T)
    wg, wn = router_weights(cfg_m, E, 0, 1, torch.float32, dev)
    wg.requires_grad_()
    wn.requires_grad_()
    layer = B.MoELayer.from_stacked(B.RouterParams(wg, wn), W1, W2, W3)
    gate = B.GateConfig(n_experts=E, top_k=K, capacity_factor=1.0)
    x = torch.randn(T, H, device=dev).to(torch.bfloat16).requires_grad_()
    dy = torch.randn(T, H, device=dev).to(torch.bfloat16)
    lam = torch.tensor(0.01, device=dev)
    params = [W1, W2, W3, wg, wn, x]

    def step():
        for p in params:
            p.grad = None
        out = B.moe_forward(x, layer, gate)
        aux = B.importance_penalty(out.gates)
        torch.autograd.backward([out.output, aux], [dy, lam])

    for _ in range(30):
        step()
    torch.cuda.synchronize()
    cap = capture(step, repeat=3, warmup=0)
    for _ in range(3):
        cap.replay()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        cap.replay()
        torch.cuda.synchronize()
    ks = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
                if e.device_type == torch.autograd.DeviceType.CUDA)
    n = len(ks) // 3
    mid = ks[n:2 * n]
    rows, prev_end, idle = [], None, 0.0
    for s, e, name in mid:
        gap = 0.0 if prev_end is None else max(0.0, s - prev_end)
        idle += gap
        rows.append({"kernel": name.split("(")[0][-60:], "start_us": round(s - mid[0][0], 1),
                     "dur_us": round(e - s, 1), "gap_before_us": round(gap, 2)})
        prev_end = e if prev_end is None else max(prev_end, e)
    out = {"kernels_per_step": n, "step_window_us": round(mid[-1][1] - mid[0][0], 1),
           "busy_us": round(sum(r["dur_us"] for r in rows), 1), "idle_gaps_us": round(idle, 1), "timeline": rows}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
