"""Benchmark: E8T2 MoE-layer fwd+bwd tokens/s and MFU on B200 (BASELINE.json).

Workload (BASELINE.json configs[1]): Llama-3-8B-shape E8T2 layer, hidden 4096,
ffn 14336, 8 experts top-2, mixtral router, capacity factor 1.0 (reference
formula ceil(T*CF/E)), position drop policy, 8192 tokens per GPU, bf16,
upcycled weights (random-init dense FFN copied into the experts), synthetic
inputs.  One step = moe_forward + importance aux loss + backward (all
gradients), i.e. what a training step does for this layer.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 is launched by torchrun: expert parallelism (E/N experts per rank, NCCL
all-to-all dispatch/combine), 8192 tokens per rank ("scaling": "weak").
--impl reference times the CPU reference path (the oracle port of moefold's
numpy implementation) on the host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

H, F, E, K_TOP = 4096, 14336, 8, 2
MEASURED = {"hbm_gbs": 6555.2, "bf16_tflops": 1692.0, "bf16_tflops_sustained": 1416.2}
try:
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as _f:
        MEASURED.update(json.load(_f))
except OSError:
    pass


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--tokens", type=int, default=8192)
    p.add_argument("--cf", type=lambda v: None if v.lower() in ("none", "dropless") else float(v), default=1.0,
                   help="capacity factor, or 'none' for dropless (moe.py:193-194)")
    p.add_argument("--router", default="mixtral")
    p.add_argument("--policy", default="position")
    p.add_argument("--cpu-tokens", type=int, default=512, help="bounded CPU sample (tokens per oracle step)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--eager", action="store_true",
                   help="launch every step from Python instead of replaying a captured CUDA graph")
    p.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                   help="EP exchange: fused NVLink peer-memory kernels (default) or NCCL all-to-all")
    p.add_argument("--gemm-debug", type=int, default=0, help=argparse.SUPPRESS)  # A/B experiment switches
    p.add_argument("--ep-pull", action="store_true", help=argparse.SUPPRESS)   # EP: peers pull expert rows (A/B)
    p.add_argument("--idle-before", type=float, default=0.0, help=argparse.SUPPRESS)  # A/B: idle seconds before timing
    return p.parse_args()


def cpu_sample(tokens: int, cf: float, router: str, policy: str, reps: int, threads: int | None = None):
    """Oracle (numpy port of moefold) fwd+bwd at the Llama shape on `tokens` tokens."""
    import numpy as np  # noqa: F401
    from threadpoolctl import threadpool_info, threadpool_limits
    from oracle import moe_oracle as O
    cores = threads or len(os.sched_getaffinity(0))
    # every host core, also under torchrun (which exports OMP_NUM_THREADS=1)
    with threadpool_limits(limits=cores, user_api="blas"):
        used = max([p["num_threads"] for p in threadpool_info() if p["user_api"] == "blas"] or [1])
        times = [O.time_fwd_bwd(tokens, H, F, E, K_TOP, cf, router, policy, reps=1) for _ in range(reps)]
    return times, used


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _smi_id(index: int) -> str:
    """nvidia-smi's id for torch device `index`: its UUID, so that the sampler
    reads the GPU the process runs on even when CUDA_VISIBLE_DEVICES remaps
    the ordinals (a box that hands out one GPU of eight)."""
    try:
        import torch
        u = str(torch.cuda.get_device_properties(index).uuid)
        return u if u.startswith("GPU-") else "GPU-" + u
    except Exception:
        return str(index)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 20 ms in the
    background; only samples whose timestamp falls inside the timed region
    (the `with` block) are summarised.  Started at construction -- before the
    warm-up, so that the GPU goes from the warm-up straight into the timed
    region -- with a reader thread draining the pipe (a long warm-up would
    otherwise fill it and stall the sampler)."""

    def __init__(self, index: int):
        import threading
        self.index = index
        self.smi_id = _smi_id(index)
        self.proc = None
        self.t0 = self.t1 = None
        self.lines = []
        self._reader = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.smi_id,
                 "--query-gpu=timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self._reader = threading.Thread(target=self._drain, daemon=True)
            self._reader.start()
            time.sleep(1.0)
        except OSError:
            self.proc = None

    def _drain(self):
        for ln in self.proc.stdout:
            if ln.strip():
                self.lines.append(ln)

    def __enter__(self):
        self.t0 = time.time()
        return self

    def __exit__(self, *a):
        self.t1 = time.time()
        time.sleep(0.1)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            if self._reader is not None:
                self._reader.join(timeout=5)

    def summary(self):
        import datetime
        sm, mx, reasons = [], 0, set()
        names = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
                 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
                 0x100: "display_clock_setting"}
        all_sm, idle = [], 0
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                s, m = float(parts[1]), float(parts[2])
                r = int(parts[3], 16)
            except (ValueError, IndexError):
                continue
            all_sm.append(s)
            if self.t0 is not None and not (self.t0 - 0.05 <= ts <= self.t1 + 0.05):
                continue
            sm.append(s)
            mx = max(mx, m)
            idle += bool(r & 0x1)
            for bit, nm in names.items():
                if r & bit and nm != "gpu_idle":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm), "idle_samples": idle, "gpu": self.smi_id}


def reference_arm(args, rank: int):
    if rank != 0:
        return
    reps = args.steps
    for _ in range(args.warmup):
        cpu_sample(args.cpu_tokens, args.cf, args.router, args.policy, 1)
    times, cores = cpu_sample(args.cpu_tokens, args.cf, args.router, args.policy, reps)
    tps = args.cpu_tokens * len(times) / sum(times)
    line = {
        "impl": "reference", "metric": "E8T2 MoE-layer fwd+bwd tokens/s", "value": round(tps, 3),
        "unit": "tokens/s", "n_gpus": args.gpus, "steps": len(times), "warmup": args.warmup,
        "ms_per_step": round(1e3 * sum(times) / len(times), 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"E8T2 layer fwd+bwd, H={H} F={F} E={E} k={K_TOP}, {args.router}, CF={args.cf}, "
                               f"{args.policy}; CPU sample of {args.cpu_tokens} tokens per step",
                   "tokens_per_step": args.cpu_tokens},
        "cpu_baseline": {"value": round(tps, 3), "unit": "tokens/s", "cores": cores, "kind": "port",
                         "sample": f"{args.cpu_tokens} tokens/step at Llama-3 shape, numpy/OpenBLAS fp32, "
                                   f"{cpu_model()}"},
        "e2e": {"value": round(tps, 3), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        reference_arm(args, rank)
        return
    import torch
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        from paper_2412_09952_b200.ep import run_ep_bench
        run_ep_bench(args, rank, world, dev, MEASURED)
        dist.destroy_process_group()
        return
    run_single(args, dev)


def gemm_traffic():
    """DRAM bytes (read + write) of one step's five grouped-GEMM launches from
    the committed ncu --set full capture (tools/ncu_traffic.py), or None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_gemm_traffic.json")))
    if not files:
        return None
    try:
        return json.load(open(files[-1]))["dram_bytes_per_step"]
    except (OSError, KeyError, ValueError):
        return None


def gemm_min_bytes(S: int) -> int:
    """Compulsory DRAM bytes of the five GEMM launches at S kept slots (bf16):
    every weight read twice (forward + dgrad) and its gradient written once;
    [S, F] activations: a, b (write + read), h, da, db (write + 2 reads) = 13
    transfers; [S, H]: xp (2 reads), o (write), do (2 reads), dxp (write) = 6."""
    w = 3 * E * H * F * 2                 # W1, W3, W2 (all experts)
    act_h = S * H * 2
    act_f = S * F * 2
    return int(3 * w + 13 * act_f + 6 * act_h)


WARMUP_SECONDS = 0.5


def warmup(args, fn, agree=None) -> int:
    """max(W, 3) untimed steps, then more until the warm-up has run for about
    WARMUP_SECONDS (at most 200 steps), so the timed steps start from a settled
    GPU (clock and power state) rather than from the first milliseconds of
    load: measured 6.80 vs 6.59-6.67 ms/step with W=5 vs W=100 on one box.
    The step count is decided from the first steps' time, so that all ranks of
    a multi-GPU run can agree on it (`agree`: e.g. an all_reduce MAX).
    Returns the number of warm-up steps run (reported as "warmup")."""
    import torch
    w = max(args.warmup, 3)
    fn()                                  # first step: one-time setup (module load, allocations)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(w - 1):
        fn()
    torch.cuda.synchronize()
    per = (time.perf_counter() - t0) / (w - 1)
    n = min(200, max(w, int(WARMUP_SECONDS / max(per, 1e-6))))
    if agree is not None:
        n = agree(n)
    for _ in range(n - w):
        fn()
    torch.cuda.synchronize()
    return n


def layer_flops(T: int, S: int) -> float:
    """Algorithmic FLOPs of one fwd+bwd: 18*H*F per kept slot + router 6*T*H*E."""
    return 18.0 * H * F * S + 6.0 * T * H * E


def run_e2e(steps, T, x, dy, step, graphed=False):
    """End-to-end through the public API with HOST buffers: every step copies
    its inputs (x, dy) from pinned host memory and copies its results -- the
    layer output y, the input gradient dx and the aux loss -- back to pinned
    host memory.  Inputs of step i+1 are prefetched on a copy stream while
    step i computes (double-buffered, as a training loop's data prefetch); y
    leaves on a second copy stream as soon as the forward is done (overlapping
    the backward), dx and the loss right after the backward (overlapping the
    next step).  x is copied before dy and a step waits for dy only before its
    backward, so the first step's forward overlaps its dy copy.  Every copy is inside the timed region; the region ends when
    the last D2H copy has landed.  With `graphed`, each of the two input
    buffers has its step captured as a CUDA graph (y's D2H copy is a node of
    it) and the loop replays them; the H2D prefetch and the dx / loss copies
    stay outside, so they overlap the neighbouring steps as in the eager loop."""
    import torch
    xh = x.detach().cpu().pin_memory()
    dyh = dy.cpu().pin_memory()
    res_h = torch.empty(steps + 2, dtype=torch.float32).pin_memory()
    yh = [torch.empty(x.shape, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    dxh = [torch.empty(x.shape, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    bufs = [(torch.empty_like(x), torch.empty_like(dy)) for _ in range(2)]
    cs = torch.cuda.Stream()
    ds = torch.cuda.Stream()
    main = torch.cuda.current_stream()
    copied = [torch.cuda.Event() for _ in range(2)]                  # x landed
    # dy landed: waited on only before the backward (so a step's forward starts
    # as soon as its x is in); external, so that inside a captured graph the
    # wait is a node that honours the record made before each replay
    dy_copied = [torch.cuda.Event(external=True) for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]
    landed = [torch.cuda.Event() for _ in range(2)]     # dx of the buffer's last step copied out
    for ev in consumed + landed + dy_copied:
        ev.record(main)

    def prefetch(i):
        b = i % 2
        with torch.cuda.stream(cs):
            cs.wait_event(consumed[b])
            bufs[b][0].copy_(xh, non_blocking=True)
            copied[b].record(cs)
            bufs[b][1].copy_(dyh, non_blocking=True)
            dy_copied[b].record(cs)

    def fwd_bwd(b):
        cur = torch.cuda.current_stream()
        xin = bufs[b][0].detach().requires_grad_()

        def after_forward(y):
            _d2h(ds, cur, y, yh[b])
            cur.wait_event(dy_copied[b])
        _, aux = step(xin, bufs[b][1], after_forward)
        return xin, aux

    def results(b, slot, xin, aux):
        _d2h(ds, torch.cuda.current_stream(), xin.grad, dxh[b])
        with torch.cuda.stream(ds):
            res_h[slot:slot + 1].copy_(aux.detach().reshape(1), non_blocking=True)
            landed[b].record(ds)

    caps = None
    if graphed:
        from paper_2412_09952_b200.graphs import capture

        def captured(b):
            def fn():
                r = fwd_bwd(b)
                torch.cuda.current_stream().wait_stream(ds)     # join the y copy into the capture
                return r
            return capture(fn, warmup=1)
        for b in range(2):
            bufs[b][0].copy_(x.detach())
            bufs[b][1].copy_(dy)
        caps = [captured(0), captured(1)]

    def run(n):
        prefetch(0)
        for i in range(n):
            if i + 1 < n:
                prefetch(i + 1)
            b = i % 2
            main.wait_event(copied[b])
            if caps is not None:
                main.wait_event(landed[b])       # the graph rewrites this buffer's dx in place
                caps[b].replay()                 # forward + backward, y copied out inside
                r = caps[b].outputs
            else:
                r = fwd_bwd(b)
            consumed[b].record(main)
            results(b, i, *r)                    # dx and the loss leave on the copy stream
        main.wait_stream(ds)

    run(2)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(main)
    run(steps)
    e1.record(main)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / steps
    nb = x.numel() * 2
    return {"value": round(T / (e2e_ms * 1e-3), 1), "unit": "tokens/s",
            "h2d_bytes_per_step": 2 * nb, "d2h_bytes_per_step": 2 * nb + 4,
            "ms_per_step": round(e2e_ms, 4),
            "h2d": "x, dy from pinned host, copy stream double-buffered one step ahead (dy waited for before the backward)",
            "d2h": "y (after the forward, overlapping the backward), dx and the aux loss to pinned host every step",
            "launch": ("CUDA graph per input buffer (y's copy to host is a node of it; dx and the loss are copied "
                       "after the replay, overlapping the next step)") if graphed else "eager"}


def _d2h(ds, main, t, host):
    """Copy device tensor t to pinned `host` on stream ds once `main` has
    produced it; the caching allocator is told t is in use on ds."""
    import torch
    ev = torch.cuda.Event()
    ev.record(main)
    with torch.cuda.stream(ds):
        ds.wait_event(ev)
        host.copy_(t.detach(), non_blocking=True)
        t.record_stream(ds)


# Algorithmic HBM bytes per launch of the layer's non-GEMM kernels (reads +
# writes that the op needs, bf16 activations, fp32 routing tensors; padding
# rows excluded).  T tokens, S kept slots.
def small_kernel_bytes(T: int, S: int) -> dict:
    th, sh, te = T * H * 2, S * H * 2, T * E * 4
    return {
        "router_fwd": th + H * E * 4 + 3 * te,      # x, W_g; logits, gates, probs/noise
        "dispatch": 2 * te + te,                   # gates in; slot_rank out (+ stats)
        "permute": th + sh,                        # x in, kept rows out
        "combine": sh + th + 2 * te,               # expert rows + gates/slots in, y out
        "combine_bwd": th + 2 * sh + 3 * te,       # dy, o in; do, dg out
        "router_bwd": sh + th + 4 * te,            # dxp rows in, dx out (+ dg, gates, dh)
        "router_wgrad": th + te,                   # x, dh in
    }


# CUPTI kernel name -> the layer's C entry point (N=1 path)
_KERNEL_ENTRY = (("moe_gemm_kernel<0,", "expert_fwd1"), ("moe_gemm_kernel<1,", "expert_fwd2"),
                 ("moe_gemm_kernel<2,", "expert_bwd2"), ("moe_gemm_kernel<4,", "expert_wgrad"),
                 ("moe_gemm_kernel<6,", "expert_wgrad"), ("moe_gemm_kernel<3,", "expert_bwd1"),
                 ("router_wsplit_kernel", "router_fwd"), ("router_fwd", "router_fwd"),
                 ("dispatch", "dispatch"), ("combine_bwd_kernel", "combine_bwd"), ("combine_kernel", "combine"),
                 ("permute_kernel", "permute"), ("importance_bwd", "importance_bwd"),
                 ("router_dx_kernel", "router_bwd"), ("router_dh_kernel", "router_bwd"),
                 ("router_wgrad", "router_wgrad"), ("reduce_partials", "router_wgrad"))


def kernel_times(fn, n):
    """{"b200moe_<entry>": (total ms, kernels)} over n calls of fn, from the
    CUPTI kernel records of a torch.profiler pass (the kernels' own device
    durations)."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(n):
            fn()
        torch.cuda.synchronize()
    out = {}
    for e in prof.events():
        if e.device_type != torch.autograd.DeviceType.CUDA or "b200moe::" not in e.name:
            continue
        entry = next((v for k, v in _KERNEL_ENTRY if k in e.name), None)
        if entry is None:
            continue
        t, c = out.get("b200moe_" + entry, (0.0, 0))
        out["b200moe_" + entry] = (t + (e.time_range.end - e.time_range.start) / 1e3, c + 1)
    return out


def run_single(args, dev):
    import torch
    import paper_2412_09952_b200 as B
    from paper_2412_09952_b200 import _lib
    from paper_2412_09952_b200.upcycle import upcycle_experts, router_weights

    T = args.tokens
    if args.gemm_debug:
        _lib.call("b200moe_gemm_set_debug", args.gemm_debug)
    torch.manual_seed(0)
    # upcycled layer: one random-init dense SwiGLU FFN copied into 8 experts (K12)
    w1 = (torch.randn(H, F, device=dev) * 0.02).to(torch.bfloat16)
    w2 = (torch.randn(F, H, device=dev) * 0.02).to(torch.bfloat16)
    w3 = (torch.randn(H, F, device=dev) * 0.02).to(torch.bfloat16)
    W1, W2, W3 = (w.requires_grad_() for w in upcycle_experts(w1, w2, w3, E))
    del w1, w2, w3
    cfg_m = B.ModelConfig(vocab=32, hidden=H, layers=1, heads=32, kv_heads=8, ffn_hidden=F, seq_len=T)
    wg, wn = router_weights(cfg_m, E, 0, 1, torch.float32, dev)
    wg.requires_grad_()
    wn.requires_grad_()
    layer = B.MoELayer.from_stacked(B.RouterParams(wg, wn), W1, W2, W3)
    gate = B.GateConfig(n_experts=E, top_k=K_TOP, router_type=args.router, capacity_factor=args.cf,
                        drop_policy=args.policy)
    x = torch.randn(T, H, device=dev).to(torch.bfloat16).requires_grad_()
    dy = torch.randn(T, H, device=dev).to(torch.bfloat16)
    lam = torch.tensor(0.01, device=dev)
    params = [W1, W2, W3, wg, wn, x]

    def step(xin, dyin, on_forward=None):
        for p in params:
            p.grad = None
        out = B.moe_forward(xin, layer, gate)
        if on_forward is not None:
            on_forward(out.output)
        aux = B.importance_penalty(out.gates)
        torch.autograd.backward([out.output, aux], [dyin, lam])
        return out, aux

    # warmup
    # the clock sampler's process starts (and settles) before the warm-up, so
    # the GPU goes from the warm-up straight into the timed region, without an
    # idle second that would let the clock recover from the power cap
    clk = ClockSampler(dev.index)
    warm = warmup(args, lambda: step(x, dy))
    # (the step's outputs die with this statement: no autograd graph of an eager
    # step may outlive it into a capture -- graphs.py)
    S = int(step(x, dy)[0].stats.assigned.sum())
    warm += 1
    torch.cuda.synchronize()

    # ---- timed region (device time, CUDA events on the launching stream).  The
    # grouped-GEMM time is measured INSIDE the same steps: one event before FWD1
    # and one after FWD2, one before BWD2 and one after BWD1 (the two contiguous
    # GEMM runs of a step; _lib.GEMM_SPANS), 4 events per step.
    # Default launch path: the K timed steps are captured once into a CUDA
    # graph (graphs.capture; the span events become event-record nodes of the
    # graph), replayed once untimed and once timed -- one host call launches
    # all K steps, so the GPU never waits on the Python enqueue.  --eager
    # launches every step from Python.
    prof = _lib.Profiler(spans=_lib.GEMM_SPANS)
    cap = None
    if not args.eager:
        from paper_2412_09952_b200.graphs import capture
        _lib.PROFILER = prof
        try:
            cap = capture(lambda: step(x, dy), repeat=args.steps, warmup=0)
        except Exception as exc:   # noqa: BLE001 -- keep a valid (eager) line rather than none
            print(f"[bench] CUDA-graph capture failed ({exc!r}); timing the eager loop", file=sys.stderr, flush=True)
            torch.cuda.synchronize()
            args.eager = True
            prof = _lib.Profiler(spans=_lib.GEMM_SPANS)
        _lib.PROFILER = None
    if cap is not None:
        cap.replay()
        torch.cuda.synchronize()
        warm += args.steps
    else:
        _lib.PROFILER = prof
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    if args.idle_before:
        torch.cuda.synchronize()
        time.sleep(args.idle_before)
    with clk:
        torch.cuda.synchronize()
        s0.record()
        h0 = time.perf_counter()
        if cap is not None:
            cap.replay()
        else:
            for _ in range(args.steps):
                step(x, dy)
        host_ms = (time.perf_counter() - h0) * 1e3 / args.steps   # host time to enqueue a step
        s1.record()
        torch.cuda.synchronize()
    _lib.PROFILER = None
    del cap
    ms = s0.elapsed_time(s1) / args.steps
    gemm_ms = prof.span_ms() / args.steps
    launches = prof.launches
    assert len(prof.span_pairs) == 2 * args.steps and gemm_ms <= ms, (len(prof.span_pairs), gemm_ms, ms)
    # ---- e2e: through the public API with pinned host buffers, H2D + D2H inside
    # (right after the timed region, before the attribution pass: same thermal state)
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args.steps, T, x, dy, step, graphed=not args.eager)

    # ---- attribution pass: the step split into its kernels from CUPTI kernel
    # records (torch.profiler) of K more steps -- each kernel's own duration,
    # without the launch gaps that CUDA events around every call would add to
    # the short kernels (its GEMM total is reported next to the timed one)
    ktimes = kernel_times(lambda: step(x, dy), args.steps)

    gemm_flops = 18.0 * H * F * S
    achieved_tf = gemm_flops / (gemm_ms * 1e-3) / 1e12
    peak = MEASURED["bf16_tflops"]
    peak_s = MEASURED.get("bf16_tflops_sustained", peak)
    hbm = MEASURED["hbm_gbs"]
    flops = layer_flops(T, S)
    tps = T / (ms * 1e-3)
    mfu_measured = flops / (ms * 1e-3) / (peak * 1e12)
    mfu_spec = flops / (ms * 1e-3) / 2.25e15
    timed_ms = ms * args.steps
    # Roofline denominator (B200_PROFILING.md): the burst figure for a timed
    # region shorter than a second, the sustained (seconds-long loop) one beyond.
    burst = timed_ms < 1000.0
    roof_peak = peak if burst else peak_s
    per_mode = {}
    mode_flops = {"expert_fwd1": 4.0, "expert_fwd2": 2.0, "expert_bwd2": 2.0, "expert_wgrad": 6.0,
                  "expert_bwd1": 4.0}
    for n, f in mode_flops.items():
        t = ktimes.get("b200moe_" + n)
        if t:
            tf = f * H * F * S / (t[0] / args.steps * 1e-3) / 1e12
            per_mode[n] = {"ms": round(t[0] / args.steps, 4), "TFLOPs": round(tf, 1), "frac": round(tf / peak, 4)}
    small = {}
    for n, nbytes in small_kernel_bytes(T, S).items():
        t = ktimes.get("b200moe_" + n)
        if t:
            t_ms = t[0] / args.steps
            gbs = nbytes / (t_ms * 1e-3) / 1e9
            small[n] = {"ms": round(t_ms, 4), "bytes": int(nbytes), "GBps": round(gbs, 1),
                        "frac": round(gbs / hbm, 4)}
    attr_gemm = sum(v[0] for k_, v in ktimes.items() if k_.startswith("b200moe_expert_")) / args.steps

    # ---- CPU baseline (oracle port) on a bounded sample, rank 0 / N=1 only
    cpu = None
    if not args.no_cpu_baseline:
        times, cores = cpu_sample(args.cpu_tokens, args.cf, args.router, args.policy, 2)
        cpu = {"value": round(args.cpu_tokens / min(times), 3), "unit": "tokens/s", "cores": cores, "kind": "port",
               "sample": f"{args.cpu_tokens} tokens per fwd+bwd at the Llama-3 shape (best of 2), numpy/OpenBLAS "
                         f"fp32 on {cores} threads, {cpu_model()}"}

    clocks = clk.summary()
    line = {
        "metric": "E8T2 MoE-layer fwd+bwd tokens/s", "value": round(tps, 1), "unit": "tokens/s", "n_gpus": 1,
        "steps": args.steps, "warmup": warm, "ms_per_step": round(ms, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": "Llama-3-8B-shape E8T2 MoE layer fwd+bwd (configs[1])", "hidden": H, "ffn": F,
                   "experts": E, "top_k": K_TOP, "tokens": T, "capacity_factor": args.cf, "router": args.router,
                   "drop_policy": args.policy, "kept_slots": S, "parallelism": "single GPU",
                   "l2": "inputs > L2, no flush: 2.8 GB of expert weights + ~1.5 GB of activations stream each step",
                   "launch": ("eager (one Python call chain per step)" if args.eager else
                              f"CUDA graph of the {args.steps} timed steps, captured after the warm-up and replayed "
                              f"once untimed before the timed replay")},
        "mfu": {"measured_peak": round(mfu_measured, 4), "spec_2250": round(mfu_spec, 4),
                "flops_per_step": flops},
        "roofline": {"kernel": "moe_gemm (tcgen05 grouped GEMM, all 5 launches/step)", "bound": "tensor",
                     "achieved": round(achieved_tf, 1), "peak": roof_peak, "unit": "TFLOP/s",
                     "frac": round(achieved_tf / roof_peak, 4),
                     "peak_kind": (f"measured {'burst' if burst else 'sustained'} bf16 (MEASURED_PEAKS.json): "
                                   f"timed region {timed_ms:.0f} ms"),
                     "frac_of_sustained": round(achieved_tf / peak_s, 4), "burst_peak": peak,
                     "sustained_peak": peak_s,
                     "traffic": gemm_traffic(),
                     "traffic_unit": "DRAM bytes per step (5 launches), ncu --set full capture, profiles/",
                     "algorithmic_dram_bytes_per_step": gemm_min_bytes(S),
                     "gemm_flops_per_step": gemm_flops,
                     "gemm_ms_per_step": round(gemm_ms, 4), "gemm_share_of_step": round(gemm_ms / ms, 4),
                     "kernel_timing": ("CUDA events on the launching stream around the two contiguous GEMM runs "
                                       "of every timed step (before FWD1 / after FWD2, before BWD2 / after BWD1)")},
        "kernels": {"gemm_modes": per_mode, "hbm_bound": small, "hbm_peak_gbs": hbm,
                    "attribution_gemm_ms_per_step": round(attr_gemm, 4),
                    "timing": f"attribution pass of {args.steps} steps after the timed region, CUPTI kernel records "
                              f"(torch.profiler: each kernel's own device time; TFLOPs/GBps from algorithmic "
                              f"FLOPs/bytes; frac vs burst bf16 / measured HBM)"},
        "kernels_ms_per_step": {n.replace("b200moe_", ""): round(t / args.steps, 4) for n, (t, c) in ktimes.items()},
        "e2e": e2e, "cpu_baseline": cpu, "clocks": clocks, "gpu_launches": launches,
        "host_enqueue_ms_per_step": round(host_ms, 4),
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
