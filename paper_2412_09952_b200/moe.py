"""B200-native drop-in for moefold/moe.py (the E8T2 MoE layer).

Same names, signatures, defaults, dataclasses and error classes as the
reference module; tensors are torch CUDA tensors and every computation runs
in the sm_100a kernels of lib/libb200moe.so (no CPU path):

  router_logits / gate_mixtral / gate_st / top_k_mask   -> K1  (router.cu)
  dispatch / expert_capacity                            -> K1b (router.cu)
  moe_forward:  K1 -> K1b -> permute K2 -> grouped GEMM FWD1 (SwiGLU epilogue)
                -> FWD2 -> combine K5                     (permute.cu, gemm.cu)
  backward:     combine' K6 -> BWD2 (SwiGLU') -> WGRAD -> BWD1 -> router' K10/11
  importance_penalty                                    -> router_bwd.cu

Reference call sites: moe.py:34-283, tensor.py:267-297, 371-403, 503-521.
Numerics: routing (top-k, gates, kept/dropped, slot order) is bit-exact with
the reference in float32 given the same logits; values are bf16 GEMMs with
fp32 accumulation (tolerances in tests/test_gpu_layer.py).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import ConfigError, GateError, ShapeError
from .rng import Rng

ROUTER_TYPES = ("mixtral", "st")
DROP_POLICIES = ("position", "score")
SEG_PAD = 128      # expert segments are zero-padded to this many rows
GEMM_ALIGN = 256   # grouped GEMM needs hidden / ffn multiples of this


# --------------------------------------------------------------------------
# configuration and parameter containers (moe.py:34-128)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class GateConfig:
    """Routing knobs: expert count, fan-out, ordering, noise, capacity."""

    n_experts: int
    top_k: int
    router_type: str = "mixtral"
    noise_enabled: bool = False
    capacity_factor: float | None = None  # None = dropless
    drop_policy: str = "position"

    def __post_init__(self):
        if self.n_experts < 1:
            raise ConfigError(f"n_experts must be >= 1, got {self.n_experts}")
        if not (1 <= self.top_k <= self.n_experts):
            raise ConfigError(f"top_k must be in [1, {self.n_experts}], got {self.top_k}")
        if self.router_type not in ROUTER_TYPES:
            raise ConfigError(f"router_type must be one of {ROUTER_TYPES}, got {self.router_type!r}")
        if self.capacity_factor is not None and not (self.capacity_factor > 0):
            raise ConfigError(f"capacity_factor must be positive or None, got {self.capacity_factor}")
        if self.drop_policy not in DROP_POLICIES:
            raise ConfigError(f"drop_policy must be one of {DROP_POLICIES}, got {self.drop_policy!r}")


@dataclass
class RouterParams:
    """Router weight matrix plus the trainable noise-scale matrix ([H, E])."""

    w_g: torch.Tensor
    w_noise: torch.Tensor

    def __post_init__(self):
        if tuple(self.w_g.shape) != tuple(self.w_noise.shape):
            raise ShapeError(f"router matrices differ in shape: {tuple(self.w_g.shape)} vs {tuple(self.w_noise.shape)}")
        if not bool(torch.isfinite(self.w_g).all() & torch.isfinite(self.w_noise).all()):
            raise ConfigError("router weights must be finite")

    @classmethod
    def trusted(cls, w_g: torch.Tensor, w_noise: torch.Tensor) -> "RouterParams":
        """View over a checkpoint's router tensors without the finiteness scan
        (a host sync); the model forward builds one per MoE layer per step."""
        if tuple(w_g.shape) != tuple(w_noise.shape):
            raise ShapeError(f"router matrices differ in shape: {tuple(w_g.shape)} vs {tuple(w_noise.shape)}")
        obj = cls.__new__(cls)
        obj.w_g, obj.w_noise = w_g, w_noise
        return obj


@dataclass
class ExpertFFN:
    """One expert's SwiGLU parameters in the reference [in, out] shapes:
    w1 (gate) [H, F], w2 (down) [F, H], w3 (up) [H, F].  When the layer is
    built from stacked kernel-layout parameters these are transposed views."""

    w1: torch.Tensor
    w2: torch.Tensor
    w3: torch.Tensor


@dataclass
class MoELayer:
    router: RouterParams
    experts: list
    # Stacked kernel-layout parameters (W1, W2, W3) = ([E,F,H], [E,H,F], [E,F,H]);
    # when present they are the trainable leaves and `experts` holds views.
    stacked: tuple | None = field(default=None, repr=False)

    def __post_init__(self):
        if not self.experts:
            raise ConfigError("MoELayer needs at least one expert")
        s0 = (tuple(self.experts[0].w1.shape), tuple(self.experts[0].w2.shape), tuple(self.experts[0].w3.shape))
        for e in self.experts[1:]:
            s = (tuple(e.w1.shape), tuple(e.w2.shape), tuple(e.w3.shape))
            if s != s0:
                raise ShapeError(f"experts disagree in shape: {s0} vs {s}")

    @classmethod
    def from_stacked(cls, router: RouterParams, W1: torch.Tensor, W2: torch.Tensor, W3: torch.Tensor) -> "MoELayer":
        # detached views: reading an expert shares the stacked storage, its
        # gradient is expert_grad(); an autograd view would keep the stacked
        # parameters' grad accumulators alive (and bound to the stream the
        # layer was built on, which a CUDA-graph capture cannot wait on)
        experts = [ExpertFFN(w1=W1[e].detach().t(), w2=W2[e].detach().t(), w3=W3[e].detach().t())
                   for e in range(W1.shape[0])]
        return cls(router=router, experts=experts, stacked=(W1, W2, W3))

    def stacked_weights(self):
        """(W1, W2, W3) in kernel layout (bf16 for ExpertFFN-list layers);
        differentiable w.r.t. the experts."""
        if self.stacked is not None:
            return self.stacked
        return _StackExperts.apply(self, *[getattr(ex, w) for ex in self.experts for w in ("w1", "w2", "w3")])

    def expert_grad(self, e: int, name: str):
        """Gradient of expert e's `name` ('w1'|'w2'|'w3') in the reference shape."""
        if self.stacked is None:
            return getattr(self.experts[e], name).grad
        W = self.stacked[("w1", "w2", "w3").index(name)]
        return None if W.grad is None else W.grad[e].t()


class _StackExperts(torch.autograd.Function):
    """Per-expert [in, out] parameters (a reference caller's
    MoELayer(router, [ExpertFFN, ...]), model.py:177-188) -> the stacked bf16
    kernel layout W1, W3 [E,F,H], W2 [E,H,F].  The stacks are cached on the
    layer and rebuilt only when an expert tensor changed (its version counter
    moves on every in-place update, e.g. an optimizer step), so repeated
    forwards with the same weights copy nothing.  Backward hands each expert
    the transposed slice of the stacked gradient in its own dtype."""

    @staticmethod
    def forward(ctx, layer, *ws):
        key = tuple((t.data_ptr(), t._version, t.dtype, tuple(t.shape), tuple(t.stride())) for t in ws)
        cache = layer.__dict__.get("_stack_cache")
        if torch.cuda.is_current_stream_capturing():
            # inside a CUDA graph the stack is part of the recorded step, so a
            # replay after an in-place weight update re-stacks (graphs.py)
            n = len(ws) // 3
            cache = (None, tuple(torch.stack([ws[3 * e + j].detach().t() for e in range(n)])
                                 .to(torch.bfloat16).contiguous() for j in range(3)))
        elif cache is None or cache[0] != key:
            n = len(ws) // 3
            stacks = tuple(torch.stack([ws[3 * e + j].detach().t() for e in range(n)]).to(torch.bfloat16).contiguous()
                           for j in range(3))
            cache = (key, stacks)
            layer.__dict__["_stack_cache"] = cache
        ctx.dtypes = [t.dtype for t in ws]
        return tuple(s.detach() for s in cache[1])

    @staticmethod
    def backward(ctx, g1, g2, g3):
        out = [None]
        n = len(ctx.dtypes) // 3
        for e in range(n):
            for j, g in enumerate((g1, g2, g3)):
                out.append(None if g is None else g[e].t().to(ctx.dtypes[3 * e + j]))
        return tuple(out)


@dataclass
class RoutingStats:
    """Per-batch routing outcome for one MoE layer (moe.py:95-116): same
    fields and constructor as the reference."""

    assigned: np.ndarray          # [N] kept slots per expert
    dropped: int                  # slots excluded by capacity
    total_slots: int              # slots with a positive gate
    gate_mass: np.ndarray         # [N] summed gate values of kept slots
    capacity: int | None

    @property
    def drop_rate(self) -> float:
        return self.dropped / self.total_slots if self.total_slots else 0.0

    @property
    def load_entropy(self) -> float:
        """Entropy (nats) of the kept-slot distribution over experts."""
        a = self.assigned
        total = int(a.sum())
        if total == 0:
            return 0.0
        p = a[a > 0] / total
        return float(-(p * np.log(p)).sum())


class DeviceRoutingStats(RoutingStats):
    """RoutingStats backed by the dispatch kernel's device tensors and
    materialised to numpy on first access (one device->host copy), so the
    forward pass never synchronises the host.  A GateError recorded by the
    router (all-masked softmax row) surfaces on that first access."""

    def __init__(self, counts, stats, gate_mass, capacity, err_flag=None):  # noqa: D107 (no dataclass init)
        self._dev = (counts, stats, gate_mass, err_flag)
        self._host = None
        self.capacity = capacity

    def _materialize(self):
        if self._host is None:
            counts, stats, mass, err = self._dev
            st = stats.cpu().numpy()
            if (err is not None and int(err.item()) != 0) or (st.size > 2 and st[2] != 0):
                raise GateError("softmax row with all entries masked")
            self._host = (counts.cpu().numpy().astype(np.int64), int(st[0]), int(st[1]), mass.cpu().numpy())
        return self._host

    @property
    def assigned(self) -> np.ndarray:
        return self._materialize()[0]

    @property
    def dropped(self) -> int:
        return self._materialize()[1]

    @property
    def total_slots(self) -> int:
        return self._materialize()[2]

    @property
    def gate_mass(self) -> np.ndarray:
        return self._materialize()[3]

    def to_host(self) -> RoutingStats:
        """A plain (reference-type) RoutingStats with the same values."""
        return RoutingStats(self.assigned, self.dropped, self.total_slots, self.gate_mass, self.capacity)

    def __repr__(self):
        return (f"RoutingStats(assigned={self.assigned!r}, dropped={self.dropped}, total_slots={self.total_slots}, "
                f"gate_mass={self.gate_mass!r}, capacity={self.capacity})")


@dataclass
class TopKMask:
    """Top-k selection result: original values plus the keep mask."""

    values: torch.Tensor
    keep: torch.Tensor

    def masked_values(self) -> torch.Tensor:
        return torch.where(self.keep, self.values, torch.full_like(self.values, -math.inf))


@dataclass
class DispatchResult:
    kept: torch.Tensor     # [T, N] bool
    dropped: torch.Tensor  # [T, N] bool
    stats: RoutingStats
    slot_rank: torch.Tensor | None = None


@dataclass
class MoEForwardResult:
    output: torch.Tensor
    stats: RoutingStats
    gates: torch.Tensor  # pre-capacity gates, differentiable (aux losses)


# --------------------------------------------------------------------------
# helpers
# --------------------------------------------------------------------------

_CACHE: dict = {}


def _require_cuda(t: torch.Tensor, name: str) -> None:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise RuntimeError(f"{name} must be a CUDA tensor (the B200 build has no CPU path)")


def _ep(E: int) -> int:
    return 4 if E <= 4 else 8 if E <= 8 else 16 if E <= 16 else 32


def _dispatch_ws(device, T: int) -> torch.Tensor:
    """The dispatch kernel's reusable workspace (ticket, tile counter, epoch,
    look-back status words): zeroed once, one per (device, stream), grown for
    larger T (a fresh zeroed buffer)."""
    key = ("disp_ws", device, torch.cuda.current_stream(device).cuda_stream)
    need = int(_lib.load().b200moe_dispatch_workspace_words(int(T)))
    ws = _CACHE.get(key)
    if ws is None or ws.numel() < need:
        ws = torch.zeros(need, dtype=torch.int32, device=device)
        _CACHE[key] = ws
    return ws


def _router_ws(H: int, E: int, device) -> torch.Tensor:
    """Workspace of b200moe_router_fwd (swizzled W tables for the backward +
    the bf16 split table of the tensor-core router)."""
    n = int(_lib.load().b200moe_router_workspace_floats(int(H), int(E)))
    return torch.empty(n, dtype=torch.float32, device=device)


def _wgrad_tickets(device, H: int) -> torch.Tensor:
    """Per-hidden-block tickets of the router weight-gradient kernel (zeroed
    once; each launch leaves them zeroed), one buffer per (device, stream)."""
    key = ("wg_tickets", device, torch.cuda.current_stream(device).cuda_stream)
    t = _CACHE.get(key)
    n = (H + 127) // 128          # one per 128-hidden block (tensor-core kernel; the ring kernel uses half)
    if t is None or t.numel() < n:
        t = torch.zeros(n, dtype=torch.int32, device=device)
        _CACHE[key] = t
    return t


def _arange_i32(n: int, device) -> torch.Tensor:
    key = ("arange", n, device)
    t = _CACHE.get(key)
    if t is None:
        t = torch.arange(n, dtype=torch.int32, device=device)
        _CACHE[key] = t
    return t


def _as_logits(h, keep_graph: bool = False) -> torch.Tensor:
    if isinstance(h, np.ndarray):
        h = torch.from_numpy(np.ascontiguousarray(h, dtype=np.float32)).cuda()
    _require_cuda(h, "logits")
    if h.dim() == 1:
        h = h[None, :]
    if not keep_graph:
        h = h.detach()
    return h.to(torch.float32).contiguous()


def expert_capacity(tokens_per_batch: int, n_experts: int, cf: float | None) -> int | None:
    """Slots per expert: ceil(tokens / N * CF) in host float64 (moe.py:189-196)."""
    if tokens_per_batch < 1:
        raise ConfigError(f"tokens_per_batch must be >= 1, got {tokens_per_batch}")
    if cf is None:
        return None
    return int(math.ceil(tokens_per_batch * cf / n_experts - 1e-9))


def _rows_bound(T: int, E: int, k: int, cap: int | None) -> int:
    kept = T * k if cap is None else min(T * k, E * cap)
    return (kept + E * SEG_PAD + SEG_PAD - 1) // SEG_PAD * SEG_PAD


# --------------------------------------------------------------------------
# routing primitives (forward-only views of K1 / K1b)
# --------------------------------------------------------------------------

def _gate(h: torch.Tensor, k: int, router_type: str, want_topk: bool = False):
    h = _as_logits(h)
    T, E = h.shape
    if not (1 <= k <= E):
        raise ConfigError(f"top-k out of range: k={k}, n={E}")
    gates = torch.empty_like(h)
    probs = torch.empty_like(h) if router_type == "st" else None
    topk = torch.empty(T, E, dtype=torch.uint8, device=h.device) if want_topk else None
    err = torch.zeros(1, dtype=torch.int32, device=h.device)
    _lib.call("b200moe_gate_from_logits", h.data_ptr(), T, E, k, _lib.ROUTER[router_type], gates.data_ptr(),
              _lib.ptr(probs), _lib.ptr(topk), err.data_ptr(), _lib.stream_ptr())
    return gates, probs, topk, err


def top_k_mask(values, k: int) -> torch.Tensor:
    """Boolean keep-mask of the k largest entries per row, lowest index wins ties."""
    squeeze = getattr(values, "ndim", 2) == 1
    _, _, topk, _ = _gate(values, k, "st", want_topk=True)
    m = topk.bool()
    return m[0] if squeeze else m


def keep_top_k(v, k: int) -> TopKMask:
    h = _as_logits(v)
    keep = top_k_mask(h, k)
    squeeze = getattr(v, "ndim", 2) == 1
    return TopKMask(values=h[0] if squeeze else h, keep=keep[0] if squeeze and keep.dim() == 2 else keep)


def _checked(gates, err):
    if int(err.item()) != 0:
        raise GateError("softmax row with all entries masked")
    return gates


class _GateFunction(torch.autograd.Function):
    """gates = gate_{mixtral,st}(h, k) on K1's gate core; backward = the masked
    softmax' of tensor.py:292-295 (b200moe_gate_bwd)."""

    @staticmethod
    def forward(ctx, h, k: int, router_type: str):
        g, probs, _, err = _gate(h, k, router_type)
        _checked(g, err)    # the reference raises GateError at call time (tensor.py:283-284)
        ctx.router_type = router_type
        ctx.save_for_backward(g, probs)
        return g

    @staticmethod
    def backward(ctx, dg):
        g, probs = ctx.saved_tensors
        T, E = g.shape
        dgc = dg.to(torch.float32).contiguous()
        dh = torch.empty_like(g)
        _lib.call("b200moe_gate_bwd", dgc.data_ptr(), g.data_ptr(), _lib.ptr(probs), T, E, _lib.ROUTER[ctx.router_type],
                  dh.data_ptr(), _lib.stream_ptr())
        return dh, None, None


def _gate_fn(h, k: int, router_type: str) -> torch.Tensor:
    squeeze = getattr(h, "ndim", 2) == 1
    g = _GateFunction.apply(_as_logits(h, keep_graph=True), k, router_type)
    return g[0] if squeeze else g


def gate_mixtral(h, k: int) -> torch.Tensor:
    """Top-k mask first, then softmax over the survivors; rows sum to 1
    (moe.py:171-173).  Differentiable w.r.t. h."""
    return _gate_fn(h, k, "mixtral")


def gate_st(h, k: int) -> torch.Tensor:
    """Softmax over all experts, then top-k (on the logits) without
    renormalization (moe.py:176-186).  Differentiable w.r.t. h."""
    return _gate_fn(h, k, "st")


class _RouterLogitsFunction(torch.autograd.Function):
    """h = x.W_g (+ z * softplus(x.W_noise)) on K1 (b200moe_router_fwd); the
    backward (b200moe_router_logits_bwd) gives dx, dW_g and, with noise,
    dW_noise -- the matmul/softplus closures of tensor.py:192-207, 220-227."""

    @staticmethod
    def forward(ctx, xb, wg, wn, z):
        T, H = xb.shape
        E = wg.shape[1]
        dev = xb.device
        logits = torch.empty(T, E, dtype=torch.float32, device=dev)
        gates = torch.empty_like(logits)
        na = torch.empty_like(logits) if z is not None else None
        ws = _router_ws(H, E, dev)
        err = torch.zeros(1, dtype=torch.int32, device=dev)
        _lib.call("b200moe_router_fwd", xb.data_ptr(), wg.data_ptr(), wn.data_ptr(), _lib.ptr(z), T, H, E, 1, 0,
                  logits.data_ptr(), gates.data_ptr(), None, _lib.ptr(na), ws.data_ptr(), err.data_ptr(),
                  _lib.stream_ptr())
        ctx.save_for_backward(xb, wg, wn, z, na)
        return logits

    @staticmethod
    def backward(ctx, dlogits):
        xb, wg, wn, z, na = ctx.saved_tensors
        T, H = xb.shape
        E = wg.shape[1]
        dev = xb.device
        dh = dlogits.to(torch.float32).contiguous()
        want_x, want_g, want_n = ctx.needs_input_grad[0], ctx.needs_input_grad[1], ctx.needs_input_grad[2]
        noise = z is not None
        dx = torch.empty(T, H, dtype=torch.bfloat16, device=dev) if want_x else None
        dwg = torch.empty(H, E, dtype=torch.float32, device=dev) if want_g else None
        dwn = torch.empty(H, E, dtype=torch.float32, device=dev) if (want_n and noise) else None
        dn = torch.empty(T, E, dtype=torch.float32, device=dev) if noise else None
        ws = torch.empty(2 * H * _ep(E) + (T + 63) // 64 * H * E, dtype=torch.float32, device=dev)
        _lib.call("b200moe_router_logits_bwd", xb.data_ptr(), dh.data_ptr(), wg.data_ptr(), wn.data_ptr(),
                  _lib.ptr(z), _lib.ptr(na), T, H, E, _lib.ptr(dx), _lib.ptr(dwg), _lib.ptr(dwn), _lib.ptr(dn),
                  ws.data_ptr(), _lib.stream_ptr())
        return dx, dwg, dwn, None


def router_logits(x: torch.Tensor, p: RouterParams, noise_enabled: bool, rng: Rng | None = None,
                  noise: torch.Tensor | None = None) -> torch.Tensor:
    """Per-token expert logits x @ W_g (+ z * softplus(x @ W_noise)), fp32
    (moe.py:136-149).  Differentiable w.r.t. x, W_g and (with noise) W_noise;
    x enters the kernel as bf16 (the layer's compute dtype)."""
    _require_cuda(x, "x")
    T, H = x.shape
    E = p.w_g.shape[1]
    z = _noise(T, E, x.device, noise_enabled, rng, noise)
    xb = x.to(torch.bfloat16)
    wg = p.w_g.to(torch.float32)
    wn = p.w_noise.to(torch.float32)
    Hp = _pad_to(H, GEMM_ALIGN)
    if Hp != H:   # zero hidden columns add +0 (the router kernels tile H by 256)
        xb = torch.nn.functional.pad(xb, (0, Hp - H))
        wg = torch.nn.functional.pad(wg, (0, 0, 0, Hp - H))
        wn = torch.nn.functional.pad(wn, (0, 0, 0, Hp - H))
    return _RouterLogitsFunction.apply(xb.contiguous(), wg.contiguous(), wn.contiguous(), z)


def _noise(T, E, device, enabled, rng, noise):
    if not enabled:
        return None
    if noise is not None:
        _require_cuda(noise, "noise")
        if tuple(noise.shape) != (T, E):
            raise ShapeError(f"noise must be [{T}, {E}], got {tuple(noise.shape)}")
        return noise.detach().to(torch.float32).contiguous()
    if rng is None:
        raise ConfigError("router noise enabled but no rng supplied")
    if torch.cuda.is_current_stream_capturing():
        raise ConfigError("router noise from a host rng cannot be recorded in a CUDA graph: pass noise= "
                          "(a device tensor refilled before each replay)")
    z = rng.standard_normal((T, E)).astype(np.float32)   # row-major, like moe.py:148
    return torch.from_numpy(z).to(device, non_blocking=False)


def _run_dispatch(gates: torch.Tensor, capacity: int | None, drop_policy: str, layout=_lib.LAYOUT_COMPACT,
                  seg_stride: int = 0):
    if drop_policy not in DROP_POLICIES:
        raise ConfigError(f"drop_policy must be one of {DROP_POLICIES}, got {drop_policy!r}")
    T, E = gates.shape
    dev = gates.device
    slot_rank = torch.empty(T, E, dtype=torch.int32, device=dev)
    counts = torch.empty(E, dtype=torch.int32, device=dev)
    seg_base = torch.empty(E, dtype=torch.int32, device=dev)
    gate_mass = torch.empty(E, dtype=torch.float32, device=dev)
    imp = torch.empty(E, dtype=torch.float32, device=dev)
    stats = torch.empty(3, dtype=torch.int64, device=dev)      # dropped, total slots, gate-error flag
    loss = torch.empty(1, dtype=torch.float32, device=dev)     # importance penalty of these gates
    _lib.call("b200moe_dispatch", gates.data_ptr(), T, E, -1 if capacity is None else int(capacity),
              _lib.POLICY[drop_policy], layout, seg_stride, slot_rank.data_ptr(), counts.data_ptr(),
              seg_base.data_ptr(), gate_mass.data_ptr(), imp.data_ptr(), stats.data_ptr(), loss.data_ptr(), None,
              _dispatch_ws(dev, T).data_ptr(), _lib.stream_ptr())
    return slot_rank, counts, seg_base, gate_mass, (imp, loss), stats


def dispatch(gates, capacity: int | None, drop_policy: str = "position") -> DispatchResult:
    """Resolve per-expert capacity: which (token, expert) slots survive (moe.py:206-240)."""
    if drop_policy not in DROP_POLICIES:
        raise ConfigError(f"drop_policy must be one of {DROP_POLICIES}, got {drop_policy!r}")
    g = _as_logits(gates)
    slot_rank, counts, seg_base, gate_mass, _, stats = _run_dispatch(g, capacity, drop_policy)
    kept = slot_rank >= 0
    dropped = (g > 0) & ~kept
    return DispatchResult(kept=kept, dropped=dropped,
                          stats=DeviceRoutingStats(counts, stats, gate_mass, capacity), slot_rank=slot_rank)


# --------------------------------------------------------------------------
# the fused layer
# --------------------------------------------------------------------------

class _Ctx:
    """Non-tensor forward state shared between forward, backward and stats."""

    def __init__(self, cfg: GateConfig, noise: bool):
        self.cfg = cfg
        self.noise = noise
        self.routing = None


# Gradient-accumulation fusion (opt-in, for training over micro-batches): when
# on and an expert weight leaf already holds a contiguous bf16 .grad, the
# weight-gradient GEMM adds into it (fp32 add, one rounding) and the Function
# returns None for that weight, so no separate gradient and no add pass over
# the ~1.4 G expert parameters per layer exist.  The leaf's post-accumulate
# hooks still fire (autograd runs AccumulateGrad with an undefined gradient),
# after the WGRAD launch on the same stream.  Off by default: moe_forward then
# returns expert gradients to autograd like any other op.  Only for
# .backward()-style accumulation: torch.autograd.grad(...) w.r.t. the expert
# weights would see no gradient while it is on.
_FUSE_GRAD_ACC = False


def set_expert_grad_accumulation_fusion(on: bool) -> None:
    global _FUSE_GRAD_ACC
    _FUSE_GRAD_ACC = bool(on)


def _acc_targets(W1, W2, W3):
    """The expert weight leaves a fused accumulation may add into (or None)."""
    ws = (W1, W2, W3)
    if _FUSE_GRAD_ACC and all(w.is_leaf and w.requires_grad for w in ws):
        return ws
    return None


def _wgrad_call(acc: bool, *args) -> None:
    """The weight-gradient GEMM: plain, or adding into the outputs (acc)."""
    if acc:
        _lib.call("b200moe_expert_wgrad_acc", *args[:-1], 1, args[-1])
    else:
        _lib.call("b200moe_expert_wgrad", *args)


def _wgrad_outputs(targets, W1, W2, W3):
    """(dW1, dW2, dW3, accumulate): the leaves' existing gradients when every one
    can take an in-place add, else fresh buffers."""
    if targets is not None:
        gs = [t.grad for t in targets]
        if all(g is not None and g.dtype == torch.bfloat16 and g.is_contiguous() and g.shape == t.shape
               for g, t in zip(gs, targets)):
            return gs[0], gs[1], gs[2], True
    return torch.empty_like(W1), torch.empty_like(W2), torch.empty_like(W3), False


class _MoEFunction(torch.autograd.Function):
    """y, gates = MoE(x; W_g, W_noise, W1, W2, W3) with the whole forward and
    backward in the sm_100a kernels.  Inputs are already padded/cast:
    x bf16 [T, H]; W_g, W_noise fp32 [H, E]; W1, W3 bf16 [E, F, H];
    W2 bf16 [E, H, F]; z fp32 [T, E] or None."""

    @staticmethod
    def forward(ctx, x, w_g, w_noise, W1, W2, W3, z, st: _Ctx):
        cfg = st.cfg
        T, H = x.shape
        E = w_g.shape[1]
        F = W1.shape[1]
        k = cfg.top_k
        dev = x.device
        s = _lib.stream_ptr()
        rt = _lib.ROUTER[cfg.router_type]
        f32 = dict(dtype=torch.float32, device=dev)
        bf = dict(dtype=torch.bfloat16, device=dev)

        logits = torch.empty(T, E, **f32)
        gates = torch.empty(T, E, **f32)
        probs = torch.empty(T, E, **f32) if cfg.router_type == "st" else None
        noise_act = torch.empty(T, E, **f32) if z is not None else None
        err = None          # gate errors reach the host through the dispatch stats (stats[2])
        ws = _router_ws(H, E, dev)      # left holding the swizzled W_g / W_noise (reused below)
        ctx.router_ws = ws
        _lib.call("b200moe_router_fwd", x.data_ptr(), w_g.data_ptr(), w_noise.data_ptr(), _lib.ptr(z), T, H, E, k,
                  rt, logits.data_ptr(), gates.data_ptr(), _lib.ptr(probs), _lib.ptr(noise_act), ws.data_ptr(),
                  None, s)
        cap = expert_capacity(T, E, cfg.capacity_factor)
        slot_rank, counts, seg_base, gate_mass, (imp, imp_loss), stats = _run_dispatch(gates, cap, cfg.drop_policy)
        R = _rows_bound(T, E, k, cap)
        seg_e = _arange_i32(E, dev)
        xp = torch.empty(R, H, **bf)
        _lib.call("b200moe_permute", x.data_ptr(), slot_rank.data_ptr(), seg_base.data_ptr(), counts.data_ptr(),
                  T, H, E, xp.data_ptr(), s)
        A = torch.empty(R, F, **bf)
        B = torch.empty(R, F, **bf)
        Hh = torch.empty(R, F, **bf)
        _lib.call("b200moe_expert_fwd1", xp.data_ptr(), W1.data_ptr(), W3.data_ptr(), seg_base.data_ptr(),
                  counts.data_ptr(), seg_e.data_ptr(), E, R, H, F, E, A.data_ptr(), B.data_ptr(), Hh.data_ptr(), s)
        O = torch.empty(R, H, **bf)
        _lib.call("b200moe_expert_fwd2", Hh.data_ptr(), W2.data_ptr(), seg_base.data_ptr(), counts.data_ptr(),
                  seg_e.data_ptr(), E, R, H, F, E, O.data_ptr(), s)
        y = torch.empty(T, H, **bf)
        _lib.call("b200moe_combine", O.data_ptr(), gates.data_ptr(), slot_rank.data_ptr(), seg_base.data_ptr(), T,
                  H, E, y.data_ptr(), s)

        st.routing = dict(logits=logits, slot_rank=slot_rank, counts=counts, seg_base=seg_base,
                          gate_mass=gate_mass, importance=imp, importance_loss=imp_loss, stats=stats, err=err,
                          capacity=cap, rows=R,
                          noise_act=noise_act)
        ctx.st = st
        ctx.acc_targets = _acc_targets(W1, W2, W3)
        ctx.save_for_backward(x, w_g, w_noise, W1, W2, W3, z, gates, probs, noise_act, slot_rank, counts,
                              seg_base, xp, A, B, Hh, O)
        return y, gates

    @staticmethod
    def backward(ctx, dy, dgates):
        (x, w_g, w_noise, W1, W2, W3, z, gates, probs, noise_act, slot_rank, counts, seg_base, xp, A, B, Hh,
         O) = ctx.saved_tensors
        st = ctx.st
        cfg = st.cfg
        T, H = x.shape
        E = w_g.shape[1]
        F = W1.shape[1]
        R = xp.shape[0]
        dev = x.device
        s = _lib.stream_ptr()
        f32 = dict(dtype=torch.float32, device=dev)
        bf = dict(dtype=torch.bfloat16, device=dev)
        seg_e = _arange_i32(E, dev)

        if dy is None:
            dy = torch.zeros(T, H, **bf)
        dy = dy.to(torch.bfloat16).contiguous()
        dO = torch.empty(R, H, **bf)
        dg = torch.empty(T, E, **f32)
        _lib.call("b200moe_combine_bwd", dy.data_ptr(), O.data_ptr(), gates.data_ptr(), slot_rank.data_ptr(),
                  seg_base.data_ptr(), counts.data_ptr(), T, H, E, dO.data_ptr(), dg.data_ptr(), s)
        dA = torch.empty(R, F, **bf)
        dB = torch.empty(R, F, **bf)
        dW1, dW2, dW3, acc = _wgrad_outputs(ctx.acc_targets, W1, W2, W3)
        dxp = torch.empty(R, H, **bf)
        seg = (seg_base.data_ptr(), counts.data_ptr(), seg_e.data_ptr(), E, R, H, F, E)
        wg_args = (xp.data_ptr(), Hh.data_ptr(), dO.data_ptr(), dA.data_ptr(), dB.data_ptr()) + seg + \
            (dW1.data_ptr(), dW2.data_ptr(), dW3.data_ptr(), int(acc))
        # serial BWD2 -> WGRAD -> BWD1, each on the whole chip (co-running WGRAD
        # beside BWD1 / dW2 beside BWD2 on split CTA budgets measured slower)
        _lib.call("b200moe_expert_bwd2", dO.data_ptr(), W2.data_ptr(), A.data_ptr(), B.data_ptr(), *seg,
                  dA.data_ptr(), dB.data_ptr(), s)
        _wgrad_call(acc, *wg_args[:-1], s)
        _lib.call("b200moe_expert_bwd1", dA.data_ptr(), dB.data_ptr(), W1.data_ptr(), W3.data_ptr(), *seg,
                  dxp.data_ptr(), s)
        if acc:
            dW1 = dW2 = dW3 = None
        dx = torch.empty(T, H, **bf)
        dh = torch.empty(T, E, **f32)
        dn = torch.empty(T, E, **f32) if z is not None else None
        dgx, sx_t, sx_e = None, 0, 0
        if dgates is not None:
            dgx = dgates.to(torch.float32)
            sx_t, sx_e = dgx.stride()
        ws = torch.empty(2 * H * _ep(E) + T * _ep(E), **f32)
        _lib.call("b200moe_router_bwd", dxp.data_ptr(), slot_rank.data_ptr(), seg_base.data_ptr(), dg.data_ptr(),
                  _lib.ptr(dgx), sx_t, sx_e, gates.data_ptr(), _lib.ptr(probs), w_g.data_ptr(), w_noise.data_ptr(),
                  _lib.ptr(z), _lib.ptr(noise_act), *_swizzled(ctx, H, E, z), T, H, E, cfg.top_k,
                  _lib.ROUTER[cfg.router_type],
                  dx.data_ptr(), dh.data_ptr(), _lib.ptr(dn), ws.data_ptr(), s)
        dwg = torch.empty(H, E, **f32)
        dwn = torch.empty(H, E, **f32) if z is not None else None
        wsw = torch.empty((T + 63) // 64 * H * E, **f32)
        _lib.call("b200moe_router_wgrad", x.data_ptr(), dh.data_ptr(), _lib.ptr(dn), T, H, E, dwg.data_ptr(),
                  _lib.ptr(dwn), wsw.data_ptr(), _wgrad_tickets(dev, H).data_ptr(), s)
        if st.routing is not None:   # router-logit gradients, for inspection (out.routing["dh"])
            st.routing["dh"], st.routing["dn"] = dh, dn
        return dx, dwg, dwn, dW1, dW2, dW3, None, None


def _swizzled(ctx, H: int, E: int, z):
    """Device pointers of the swizzled W_g / W_noise tables the router forward
    left in its workspace (ctx.router_ws), for b200moe_router_bwd."""
    ws = getattr(ctx, "router_ws", None)
    if ws is None:
        return None, None
    return ws.data_ptr(), (ws.data_ptr() + H * _ep(E) * 4 if z is not None else None)


def _pad_to(n: int, a: int) -> int:
    return (n + a - 1) // a * a


def moe_forward(x: torch.Tensor, layer: MoELayer, cfg: GateConfig, rng: Rng | None = None,
                training: bool = False, noise: torch.Tensor | None = None) -> MoEForwardResult:
    """Route tokens, run surviving slots through their experts, combine by gate
    (moe.py:250-283).  Differentiable w.r.t. x, the router and the experts;
    `gates` (pre-capacity) is returned for balance penalties.  Noise applies
    only when cfg.noise_enabled and training (drawn from `rng` on the host, or
    given as `noise` [T, E])."""
    n = cfg.n_experts
    if len(layer.experts) != n:
        raise ConfigError(f"layer has {len(layer.experts)} experts, config says {n}")
    if x.dim() != 2 or x.shape[1] != layer.router.w_g.shape[0]:
        raise ShapeError(f"input width {tuple(x.shape)[-1]} != router input {layer.router.w_g.shape[0]}")
    if n > 32:
        raise ConfigError(f"the B200 router supports up to 32 experts, got {n}")
    _require_cuda(x, "x")
    T, H = x.shape
    z = _noise(T, n, x.device, cfg.noise_enabled and training, rng, noise)
    W1, W2, W3 = layer.stacked_weights()
    F = W1.shape[1]
    Hp, Fp = _pad_to(H, GEMM_ALIGN), _pad_to(F, GEMM_ALIGN)
    xb = x.to(torch.bfloat16)
    wg = layer.router.w_g.to(torch.float32)
    wn = layer.router.w_noise.to(torch.float32)
    W1b, W2b, W3b = (w.to(torch.bfloat16) for w in (W1, W2, W3))
    if Hp != H or Fp != F:
        # zero padding is exact: padded hidden columns / ffn units contribute +0
        xb = torch.nn.functional.pad(xb, (0, Hp - H))
        wg = torch.nn.functional.pad(wg, (0, 0, 0, Hp - H))
        wn = torch.nn.functional.pad(wn, (0, 0, 0, Hp - H))
        W1b = torch.nn.functional.pad(W1b, (0, Hp - H, 0, Fp - F))
        W3b = torch.nn.functional.pad(W3b, (0, Hp - H, 0, Fp - F))
        W2b = torch.nn.functional.pad(W2b, (0, Fp - F, 0, Hp - H))
    st = _Ctx(cfg, z is not None)
    y, gates = _MoEFunction.apply(xb.contiguous(), wg.contiguous(), wn.contiguous(), W1b.contiguous(),
                                  W2b.contiguous(), W3b.contiguous(), z, st)
    if Hp != H:
        y = y[:, :H]
    r = st.routing
    gates._b200_importance = (r["importance"], gates._version, r["importance_loss"])
    stats = DeviceRoutingStats(r["counts"], r["stats"], r["gate_mass"], r["capacity"], r["err"])
    out = MoEForwardResult(output=y, stats=stats, gates=gates)
    out.routing = r  # device-side routing tensors (slot_rank, counts, logits, ...) for inspection
    return out


def ffn_forward(x: torch.Tensor, w1: torch.Tensor, w2: torch.Tensor, w3: torch.Tensor) -> torch.Tensor:
    """SwiGLU feed-forward down(silu(gate(x)) * up(x)) (moe.py:131-133) with the
    reference [in, out] weight shapes, as a one-segment grouped GEMM;
    differentiable (tensor.ffn).  Returns bf16 [T, H]."""
    from .tensor import ffn
    return ffn(x, w1, w2, w3)


# --------------------------------------------------------------------------
# load-balancing auxiliary loss (tensor.py:503-521)
# --------------------------------------------------------------------------

class _ImportanceFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, gates):
        T, E = gates.shape
        loss = None
        cached = getattr(gates, "_b200_importance", None)
        if cached is not None and cached[1] == gates._version:
            # gates straight from moe_forward: the dispatch kernel already reduced
            # them and evaluated the penalty (no launch here)
            imp = cached[0]
            if len(cached) > 2 and cached[2] is not None:
                loss = cached[2]
            else:
                loss = torch.empty(1, dtype=torch.float32, device=gates.device)
                _lib.call("b200moe_importance_loss", imp.data_ptr(), E, loss.data_ptr(), None, _lib.stream_ptr())
        else:
            loss = torch.empty(1, dtype=torch.float32, device=gates.device)
            err = torch.zeros(1, dtype=torch.int32, device=gates.device)
            g = gates.detach().to(torch.float32).contiguous()
            imp = torch.empty(E, dtype=torch.float32, device=g.device)
            _lib.call("b200moe_importance_fwd", g.data_ptr(), T, E, imp.data_ptr(), loss.data_ptr(), err.data_ptr(),
                      _lib.stream_ptr())
            # Arbitrary gates: raise GateError at call time like the reference
            # (tensor.py:512-513), at the cost of one host sync.  Gates straight
            # from moe_forward skip it: every row there holds a positive top-1
            # gate (or the router already flagged the row), so mean > 0.
            if int(err.item()) != 0:
                raise GateError("importance penalty needs positive total gate mass")
        ctx.save_for_backward(imp)
        ctx.shape = (T, E)
        return loss[0]

    @staticmethod
    def backward(ctx, g):
        (imp,) = ctx.saved_tensors
        T, E = ctx.shape
        gs = g.detach().to(torch.float32).reshape(1).contiguous()
        dimp = torch.empty(E, dtype=torch.float32, device=imp.device)
        _lib.call("b200moe_importance_bwd", imp.data_ptr(), gs.data_ptr(), E, dimp.data_ptr(), _lib.stream_ptr())
        return dimp[None, :].expand(T, E)


def importance_penalty(gates: torch.Tensor) -> torch.Tensor:
    """Squared coefficient of variation of per-expert gate mass; zero when
    balanced (tensor.py:503-521).  GateError if the total mass is <= 0."""
    _require_cuda(gates, "gates")
    if gates.dim() != 2:
        raise ShapeError("importance penalty needs a [T, E] gate matrix")
    return _ImportanceFunction.apply(gates)
