"""CUDA-graph launch path for static-shape layer steps.

The MoE layer makes no host synchronisation in its forward or backward and
keeps every piece of cross-call state on the device -- the dispatch scan's
epoch word, the router-wgrad tickets, the per-expert segment counts the
grouped GEMM reads -- so a whole training step (`moe_forward`,
`importance_penalty`, the backward) can be recorded once and replayed: one
host call launches the step's 13 kernels, and the GPU never waits on the
Python enqueue (a step costs ~0.7 ms of host time eagerly, several ms on a
loaded host).

Rules for a captured step (the same as for any CUDA graph):
  * shapes, the layer object and the input/output tensors are fixed at
    capture; new data goes into the captured input tensors (`copy_`) and
    results are read from the tensors the captured call returned;
  * the process must have run the step eagerly once first (workspaces and
    kernel attributes are set up on first use) -- `capture(warmup=...)` does it;
  * an expert-list layer (`MoELayer(router, [ExpertFFN, ...])`) re-stacks its
    experts inside the graph on every replay, so in-place weight updates
    between replays are seen (the eager path caches the stack by version);
  * routing statistics read after a replay describe the last replayed step;
  * a replay writes its gradients into the tensors `.grad` held when the
    capture ended; an eager step afterwards rebinds `.grad` to new tensors,
    so code that mixes the two keeps references to the captured ones;
  * no output of an earlier eager step may still be alive at capture time:
    its autograd graph keeps the parameters' gradient accumulators bound to
    the stream they were created on (the default stream), which a capture
    cannot wait on.

Expert-parallel layers (`ep.ExpertParallelMoE`) capture the same way on every
rank -- device barriers, peer kernels and the NCCL all_reduce are stream
work -- once the token-count agreement (one host all_reduce per new T) has
run eagerly; their buffer-generation check is evaluated at capture time, so
a captured step must own its buffer slot (one layer, one slot)."""

from __future__ import annotations

from dataclasses import dataclass
from typing import Any, Callable

import torch


@dataclass
class CapturedStep:
    graph: torch.cuda.CUDAGraph
    outputs: Any            # what the last captured call returned (tensors refreshed by every replay)
    repeat: int             # calls recorded back to back in the graph

    def replay(self) -> None:
        self.graph.replay()


def capture(fn: Callable[[], Any], *, repeat: int = 1, warmup: int = 2, pool=None) -> CapturedStep:
    """Record `repeat` back-to-back calls of `fn` into one CUDA graph.

    `fn` is first run `warmup` times eagerly on a side stream (torch's
    recommended pre-capture warm-up), then captured on torch's capture
    stream; the returned graph has not been replayed yet."""
    if warmup:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):
                fn()
        torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    out = None
    with torch.cuda.graph(g, pool=pool):
        for _ in range(repeat):
            out = fn()
    return CapturedStep(graph=g, outputs=out, repeat=repeat)


def capturing() -> bool:
    """True while the current stream is being captured into a CUDA graph."""
    return torch.cuda.is_available() and torch.cuda.is_current_stream_capturing()
