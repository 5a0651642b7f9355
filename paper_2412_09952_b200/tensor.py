"""Differentiable ops of the transformer step around the MoE layer, drop-in for
the pieces of moefold/tensor.py the model uses:

  rmsnorm / add_rmsnorm   tensor.py:307-321   -> b200moe_rmsnorm_fwd/bwd (model.cu)
  embedding               tensor.py:324-337   -> b200moe_embedding_fwd/bwd
  cross_entropy           tensor.py:340-364   -> b200moe_cross_entropy_fwd/bwd
  attention               tensor.py:406-500   -> torch SDPA (library flash/cuDNN attention)
  ffn                     moe.py:131-133      -> one-segment tcgen05 grouped GEMMs (gemm.cu)
  importance_penalty      tensor.py:503-521   -> re-exported from moe.py

Residual-stream activations are fp32; everything that feeds a GEMM is bf16.
The row/elementwise passes are the hand-written kernels; the dense
projections are library GEMMs (cuBLAS through torch.matmul).
"""

from __future__ import annotations

import math

import numpy as np
import torch
import torch.nn.functional as F

from . import _lib
from .errors import InputError, ShapeError
from .moe import GEMM_ALIGN, SEG_PAD, _arange_i32, _pad_to, _require_cuda, importance_penalty

RMSNORM_EPS = 1e-5
ROTARY_BASE = 10000.0

__all__ = ["RMSNORM_EPS", "ROTARY_BASE", "rmsnorm", "add_rmsnorm", "embedding", "cross_entropy", "attention", "ffn",
           "importance_penalty"]


# --------------------------------------------------------------------------
# RMSNorm (+ residual add)
# --------------------------------------------------------------------------

def _rms_bwd(ctx, dy, dres):
    x, rstd, gain = ctx.saved_tensors
    T, H = x.shape
    dy = dy.to(torch.bfloat16).contiguous()
    dx = torch.empty(T, H, dtype=torch.float32, device=x.device)
    dx_bf = torch.empty(T, H, dtype=torch.bfloat16, device=x.device) if ctx.want_bf16 else None
    dgain = torch.empty(H, dtype=torch.float32, device=x.device)
    ws = torch.empty((T + 7) // 8 * H, dtype=torch.float32, device=x.device)   # include/b200moe.h
    _lib.call("b200moe_rmsnorm_bwd", dy.data_ptr(), x.data_ptr(), rstd.data_ptr(), gain.data_ptr(), _lib.ptr(dres),
              T, H, dx.data_ptr(), _lib.ptr(dx_bf), dgain.data_ptr(), ws.data_ptr(), _lib.stream_ptr())
    return dx, dx_bf, dgain


class _RMSNorm(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, gain, eps):
        T, H = x.shape
        y = torch.empty(T, H, dtype=torch.bfloat16, device=x.device)
        rstd = torch.empty(T, dtype=torch.float32, device=x.device)
        _lib.call("b200moe_rmsnorm_fwd", x.data_ptr(), None, gain.data_ptr(), T, H, eps, None, y.data_ptr(),
                  rstd.data_ptr(), _lib.stream_ptr())
        ctx.save_for_backward(x, rstd, gain)
        ctx.want_bf16 = False
        return y

    @staticmethod
    def backward(ctx, dy):
        dx, _, dgain = _rms_bwd(ctx, dy, None)
        return dx, dgain, None


class _AddRMSNorm(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, delta, gain, eps):
        T, H = x.shape
        x_out = torch.empty_like(x)
        y = torch.empty(T, H, dtype=torch.bfloat16, device=x.device)
        rstd = torch.empty(T, dtype=torch.float32, device=x.device)
        _lib.call("b200moe_rmsnorm_fwd", x.data_ptr(), delta.data_ptr(), gain.data_ptr(), T, H, eps, x_out.data_ptr(),
                  y.data_ptr(), rstd.data_ptr(), _lib.stream_ptr())
        ctx.save_for_backward(x_out, rstd, gain)
        ctx.want_bf16 = True
        ctx.set_materialize_grads(False)
        return x_out, y

    @staticmethod
    def backward(ctx, dx_out, dy):
        if dy is None:
            dx = dx_out.contiguous()
            return dx, dx.to(torch.bfloat16), None, None
        dres = None if dx_out is None else dx_out.to(torch.float32).contiguous()
        dx, dx_bf, dgain = _rms_bwd(ctx, dy, dres)
        return dx, dx_bf, dgain, None


def _check_norm(x, gain):
    _require_cuda(x, "x")
    if x.dim() != 2 or gain.shape != (x.shape[1],):
        raise ShapeError(f"rmsnorm shapes disagree: x {tuple(x.shape)}, gain {tuple(gain.shape)}")
    if x.shape[1] % 4:
        raise ShapeError(f"rmsnorm hidden width {x.shape[1]} must be a multiple of 4")


def rmsnorm(x: torch.Tensor, gain: torch.Tensor, eps: float = RMSNORM_EPS) -> torch.Tensor:
    """g * x / rms(x) per row; x fp32 [T, H] -> bf16 [T, H] (tensor.py:307-321)."""
    _check_norm(x, gain)
    return _RMSNorm.apply(x.to(torch.float32).contiguous(), gain.to(torch.float32).contiguous(), float(eps))


def add_rmsnorm(x: torch.Tensor, delta: torch.Tensor, gain: torch.Tensor, eps: float = RMSNORM_EPS):
    """(x + delta, rmsnorm(x + delta)): the residual update fused with the next
    norm (model.py:151-156).  x fp32, delta bf16; returns (fp32, bf16)."""
    _check_norm(x, gain)
    if tuple(delta.shape) != tuple(x.shape):
        raise ShapeError(f"residual shapes disagree: {tuple(x.shape)} vs {tuple(delta.shape)}")
    return _AddRMSNorm.apply(x.to(torch.float32).contiguous(), delta.to(torch.bfloat16).contiguous(),
                             gain.to(torch.float32).contiguous(), float(eps))


# --------------------------------------------------------------------------
# embedding
# --------------------------------------------------------------------------

class _Embedding(torch.autograd.Function):
    @staticmethod
    def forward(ctx, table, ids_dev, order, seg_start, seg_id):
        V, H = table.shape
        T = ids_dev.shape[0]
        out = torch.empty(T, H, dtype=torch.float32, device=table.device)
        err = torch.zeros(1, dtype=torch.int32, device=table.device)
        _lib.call("b200moe_embedding_fwd", table.data_ptr(), ids_dev.data_ptr(), T, H, V, out.data_ptr(),
                  err.data_ptr(), _lib.stream_ptr())
        ctx.save_for_backward(order, seg_start, seg_id)
        ctx.shape = (V, H)
        return out

    @staticmethod
    def backward(ctx, g):
        order, seg_start, seg_id = ctx.saved_tensors
        V, H = ctx.shape
        g = g.to(torch.float32).contiguous()
        grad = torch.zeros(V, H, dtype=torch.float32, device=g.device)
        _lib.call("b200moe_embedding_bwd", g.data_ptr(), order.data_ptr(), seg_start.data_ptr(), seg_id.data_ptr(),
                  seg_id.shape[0], H, grad.data_ptr(), _lib.stream_ptr())
        return grad, None, None, None, None


class _EmbeddingDP(torch.autograd.Function):
    """Embedding whose backward produces the gradient of the whole data-parallel
    batch on every rank: all-gather each rank's output gradient [T, H] and ids,
    stable-sort the ids on the device, ordered scatter-add.  Moves world x T x H
    floats instead of all-reducing the [V, H] table gradient, and equals the
    single-GPU np.add.at over the concatenated batch bit for bit."""

    @staticmethod
    def forward(ctx, table, ids_dev, group):
        V, H = table.shape
        T = ids_dev.shape[0]
        out = torch.empty(T, H, dtype=torch.float32, device=table.device)
        err = torch.zeros(1, dtype=torch.int32, device=table.device)
        _lib.call("b200moe_embedding_fwd", table.data_ptr(), ids_dev.data_ptr(), T, H, V, out.data_ptr(),
                  err.data_ptr(), _lib.stream_ptr())
        ctx.save_for_backward(ids_dev)
        ctx.shape = (V, H)
        ctx.group = group
        return out

    @staticmethod
    def backward(ctx, g):
        import torch.distributed as dist
        (ids,) = ctx.saved_tensors
        V, H = ctx.shape
        world = dist.get_world_size(ctx.group)
        g = g.to(torch.float32).contiguous()
        T = ids.shape[0]
        g_all = torch.empty(world * T, H, dtype=torch.float32, device=g.device)
        ids_all = torch.empty(world * T, dtype=torch.int64, device=g.device)
        dist.all_gather_into_tensor(g_all, g, group=ctx.group)
        dist.all_gather_into_tensor(ids_all, ids, group=ctx.group)
        sid, order = torch.sort(ids_all, stable=True)
        grad = torch.zeros(V, H, dtype=torch.float32, device=g.device)
        _lib.call("b200moe_embedding_bwd_sorted", g_all.data_ptr(), order.data_ptr(), sid.data_ptr(), world * T, H,
                  grad.data_ptr(), _lib.stream_ptr())
        return grad, None, None


def embedding(table: torch.Tensor, ids, dp_group=None) -> torch.Tensor:
    """Row gather from an fp32 embedding table; the backward is the ordered
    per-id scatter-add of np.add.at (tensor.py:324-337).  ids: host ints.
    With `dp_group`, the backward returns the gradient of every rank's batch
    (equal on all ranks; no all-reduce of the table gradient needed)."""
    _require_cuda(table, "table")
    ids = np.asarray(ids.cpu() if isinstance(ids, torch.Tensor) else ids, dtype=np.int64).reshape(-1)
    V = table.shape[0]
    if ids.size and (ids.min() < 0 or ids.max() >= V):
        raise InputError(f"token id out of range [0, {V}): min={ids.min()}, max={ids.max()}")
    if table.shape[1] % 4:
        raise ShapeError(f"embedding width {table.shape[1]} must be a multiple of 4")
    if dp_group is not None:
        ids_dev = torch.from_numpy(ids).pin_memory().to(table.device, non_blocking=True)
        return _EmbeddingDP.apply(table.to(torch.float32).contiguous(), ids_dev, dp_group)
    order = np.argsort(ids, kind="stable")
    sid = ids[order]
    starts = np.flatnonzero(np.r_[True, sid[1:] != sid[:-1]]) if ids.size else np.zeros(0, dtype=np.int64)
    seg_id = sid[starts]
    seg_start = np.r_[starts, ids.size]
    dev = table.device
    host = np.concatenate([order, seg_start, seg_id]).astype(np.int32)
    buf = torch.from_numpy(host).pin_memory().to(dev, non_blocking=True)
    n, u = ids.size, seg_id.size
    ids_dev = torch.from_numpy(ids).pin_memory().to(dev, non_blocking=True)
    return _Embedding.apply(table.to(torch.float32).contiguous(), ids_dev, buf[:n], buf[n:n + u + 1],
                            buf[n + u + 1:])


# --------------------------------------------------------------------------
# cross entropy
# --------------------------------------------------------------------------

class _CrossEntropy(torch.autograd.Function):
    @staticmethod
    def forward(ctx, logits, targets):
        T, V = logits.shape
        dev = logits.device
        nll = torch.empty(T, dtype=torch.float32, device=dev)
        lse = torch.empty(T, dtype=torch.float32, device=dev)
        loss = torch.empty(1, dtype=torch.float32, device=dev)
        err = torch.zeros(1, dtype=torch.int32, device=dev)
        _lib.call("b200moe_cross_entropy_fwd", logits.data_ptr(), targets.data_ptr(), T, V, nll.data_ptr(),
                  lse.data_ptr(), loss.data_ptr(), err.data_ptr(), _lib.stream_ptr())
        ctx.save_for_backward(logits, targets, lse)
        return loss[0]

    @staticmethod
    def backward(ctx, g):
        logits, targets, lse = ctx.saved_tensors
        T, V = logits.shape
        gs = g.detach().to(torch.float32).reshape(1).contiguous()
        dlogits = torch.empty_like(logits)
        _lib.call("b200moe_cross_entropy_bwd", logits.data_ptr(), targets.data_ptr(), lse.data_ptr(), gs.data_ptr(),
                  T, V, dlogits.data_ptr(), _lib.stream_ptr())
        return dlogits, None


def cross_entropy(logits: torch.Tensor, targets) -> torch.Tensor:
    """Mean token NLL over rows of logits (tensor.py:340-364); logits are cast
    to bf16 (the lm-head GEMM's output type), math in fp32."""
    _require_cuda(logits, "logits")
    t = np.asarray(targets.cpu() if isinstance(targets, torch.Tensor) else targets, dtype=np.int64)
    if t.size == 0:
        raise InputError("cross_entropy: empty targets")
    if logits.dim() != 2 or t.ndim != 1 or logits.shape[0] != t.shape[0]:
        raise ShapeError(f"cross_entropy shapes disagree: logits {tuple(logits.shape)}, targets {t.shape}")
    V = logits.shape[1]
    if t.min() < 0 or t.max() >= V:
        raise InputError(f"target id out of range [0, {V})")
    td = torch.from_numpy(t).pin_memory().to(logits.device, non_blocking=True)
    return _CrossEntropy.apply(logits.to(torch.bfloat16).contiguous(), td)


# --------------------------------------------------------------------------
# attention (library SDPA; GQA and the reference's interleaved rotary)
# --------------------------------------------------------------------------

def _rotary(x4: torch.Tensor) -> torch.Tensor:
    """Rotate (even, odd) pairs by the per-position angle (tensor.py:383-403);
    x4: [B, S, heads, d] fp32."""
    S, d = x4.shape[1], x4.shape[3]
    half = d // 2
    inv = ROTARY_BASE ** (-torch.arange(0, half, dtype=torch.float32, device=x4.device) * 2.0 / d)
    ang = torch.arange(S, dtype=torch.float32, device=x4.device)[:, None] * inv[None, :]
    c, s = torch.cos(ang)[None, :, None, :], torch.sin(ang)[None, :, None, :]
    x1, x2 = x4[..., 0::2], x4[..., 1::2]
    return torch.stack((x1 * c - x2 * s, x1 * s + x2 * c), dim=-1).flatten(-2)


def attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, n_heads: int, n_kv_heads: int, seq_len: int,
              rotary: bool = False) -> torch.Tensor:
    """Causal grouped-query attention over flattened [batch*seq, width] inputs
    (tensor.py:406-500): query head h reads kv head h // (n_heads/n_kv_heads)."""
    n_tok = q.shape[0]
    if n_tok % seq_len != 0:
        raise ShapeError(f"token count {n_tok} not a multiple of seq_len {seq_len}")
    if n_heads % n_kv_heads != 0:
        raise ShapeError(f"n_heads {n_heads} not divisible by n_kv_heads {n_kv_heads}")
    d = q.shape[1] // n_heads
    if q.shape[1] != n_heads * d or k.shape[1] != n_kv_heads * d or v.shape[1] != n_kv_heads * d:
        raise ShapeError(f"attention projections inconsistent: q {tuple(q.shape)}, k {tuple(k.shape)}, "
                         f"v {tuple(v.shape)}")
    b = n_tok // seq_len
    q4 = q.view(b, seq_len, n_heads, d)
    k4 = k.view(b, seq_len, n_kv_heads, d)
    v4 = v.view(b, seq_len, n_kv_heads, d)
    if rotary:
        q4 = _rotary(q4.float()).to(q.dtype)
        k4 = _rotary(k4.float()).to(k.dtype)
    out = F.scaled_dot_product_attention(q4.transpose(1, 2), k4.transpose(1, 2), v4.transpose(1, 2), is_causal=True,
                                         scale=1.0 / math.sqrt(d), enable_gqa=n_heads != n_kv_heads)
    return out.transpose(1, 2).reshape(n_tok, n_heads * d)


# --------------------------------------------------------------------------
# dense SwiGLU FFN on the grouped-GEMM kernels (one segment)
# --------------------------------------------------------------------------

_SEG_CACHE: dict = {}


def _one_segment(T: int, dev):
    """Device segment table (base [0], count [T]) of a one-segment GEMM, cached."""
    key = (T, dev)
    t = _SEG_CACHE.get(key)
    if t is None:
        t = (torch.zeros(1, dtype=torch.int32, device=dev), torch.full((1,), T, dtype=torch.int32, device=dev))
        _SEG_CACHE[key] = t
    return t


class _FFN(torch.autograd.Function):
    """o = (silu(x W1^T) * (x W3^T)) W2^T with kernel-layout weights
    W1, W3 [1, F, H], W2 [1, H, F] (bf16); x bf16 [T, H], H and F multiples
    of 256."""

    @staticmethod
    def forward(ctx, x, W1, W2, W3):
        T, H = x.shape
        Fd = W1.shape[1]
        dev = x.device
        R = _pad_to(max(T, 1), SEG_PAD)
        bf = dict(dtype=torch.bfloat16, device=dev)
        if R == T and x.dtype == torch.bfloat16 and x.is_contiguous():
            xp = x                      # no padding rows needed: the GEMMs read x in place
        else:
            xp = torch.zeros(R, H, **bf)
            xp[:T] = x
        base, cnt = _one_segment(T, dev)
        seg_e = _arange_i32(1, dev)
        s = _lib.stream_ptr()
        A, B, Hh = (torch.empty(R, Fd, **bf) for _ in range(3))
        _lib.call("b200moe_expert_fwd1", xp.data_ptr(), W1.data_ptr(), W3.data_ptr(), base.data_ptr(), cnt.data_ptr(),
                  seg_e.data_ptr(), 1, R, H, Fd, 1, A.data_ptr(), B.data_ptr(), Hh.data_ptr(), s)
        O = torch.empty(R, H, **bf)
        _lib.call("b200moe_expert_fwd2", Hh.data_ptr(), W2.data_ptr(), base.data_ptr(), cnt.data_ptr(),
                  seg_e.data_ptr(), 1, R, H, Fd, 1, O.data_ptr(), s)
        ctx.save_for_backward(xp, W1, W2, W3, A, B, Hh, base, cnt)
        ctx.T = T
        return O[:T]

    @staticmethod
    def backward(ctx, dy):
        xp, W1, W2, W3, A, B, Hh, base, cnt = ctx.saved_tensors
        T = ctx.T
        R, H = xp.shape
        Fd = W1.shape[1]
        dev = xp.device
        bf = dict(dtype=torch.bfloat16, device=dev)
        seg_e = _arange_i32(1, dev)
        s = _lib.stream_ptr()
        dy = dy.to(torch.bfloat16)
        if R == T and dy.is_contiguous():
            dO = dy
        else:
            dO = torch.zeros(R, H, **bf)
            dO[:T] = dy
        dA = torch.empty(R, Fd, **bf)
        dB = torch.empty(R, Fd, **bf)
        _lib.call("b200moe_expert_bwd2", dO.data_ptr(), W2.data_ptr(), A.data_ptr(), B.data_ptr(), base.data_ptr(),
                  cnt.data_ptr(), seg_e.data_ptr(), 1, R, H, Fd, 1, dA.data_ptr(), dB.data_ptr(), s)
        dW1, dW2, dW3 = torch.empty_like(W1), torch.empty_like(W2), torch.empty_like(W3)
        _lib.call("b200moe_expert_wgrad", xp.data_ptr(), Hh.data_ptr(), dO.data_ptr(), dA.data_ptr(), dB.data_ptr(),
                  base.data_ptr(), cnt.data_ptr(), seg_e.data_ptr(), 1, R, H, Fd, 1, dW1.data_ptr(), dW2.data_ptr(),
                  dW3.data_ptr(), s)
        dxp = torch.empty(R, H, **bf)
        _lib.call("b200moe_expert_bwd1", dA.data_ptr(), dB.data_ptr(), W1.data_ptr(), W3.data_ptr(), base.data_ptr(),
                  cnt.data_ptr(), seg_e.data_ptr(), 1, R, H, Fd, 1, dxp.data_ptr(), s)
        return dxp[:T], dW1, dW2, dW3


def ffn(x: torch.Tensor, w1: torch.Tensor, w2: torch.Tensor, w3: torch.Tensor) -> torch.Tensor:
    """Differentiable SwiGLU FFN with reference [in, out] weights
    (w1, w3 [H, F], w2 [F, H]); returns bf16 [T, H] (moe.py:131-133)."""
    _require_cuda(x, "x")
    T, H = x.shape
    Fd = w1.shape[1]
    if tuple(w1.shape) != (H, Fd) or tuple(w3.shape) != (H, Fd) or tuple(w2.shape) != (Fd, H):
        raise ShapeError(f"ffn shapes disagree: x {tuple(x.shape)}, w1 {tuple(w1.shape)}, w2 {tuple(w2.shape)}, "
                         f"w3 {tuple(w3.shape)}")
    Hp, Fp = _pad_to(H, GEMM_ALIGN), _pad_to(Fd, GEMM_ALIGN)
    xb = F.pad(x.to(torch.bfloat16), (0, Hp - H))
    W1 = F.pad(w1.t().to(torch.bfloat16), (0, Hp - H, 0, Fp - Fd))[None]
    W3 = F.pad(w3.t().to(torch.bfloat16), (0, Hp - H, 0, Fp - Fd))[None]
    W2 = F.pad(w2.t().to(torch.bfloat16), (0, Fp - Fd, 0, Hp - H))[None]
    out = _FFN.apply(xb.contiguous(), W1.contiguous(), W2.contiguous(), W3.contiguous())
    return out[:, :H]


# --------------------------------------------------------------------------
# dense projections (qkv, wo, lm-head) on the tcgen05 kernel
# --------------------------------------------------------------------------

# Persistent-grid cap of the dense projections (0 = one CTA per SM).  A
# multi-GPU training step sets it a little below the SM count
# (set_dense_grid) so the NCCL reductions and the overlapped optimizer updates
# on other streams find free SMs while a projection GEMM runs.
_DENSE_GRID = 0


def set_dense_grid(ctas: int) -> None:
    global _DENSE_GRID
    _DENSE_GRID = int(ctas)


class _Linear(torch.autograd.Function):
    """y = x . w with the reference [in, out] weight layout (tensor.py:192-207
    matmul), bf16 in / out, fp32 accumulation, on the repo's own tcgen05 GEMM
    (b200moe_dense_fwd / _dgrad / _wgrad).  x [M, K], w [K, N] contiguous bf16,
    K and N multiples of 256."""

    @staticmethod
    def forward(ctx, x, w):
        M, K = x.shape
        N = w.shape[1]
        y = torch.empty(M, N, dtype=torch.bfloat16, device=x.device)
        base, cnt = _one_segment(M, x.device)
        e0 = _arange_i32(1, x.device)
        _lib.call("b200moe_dense_fwd", x.data_ptr(), w.data_ptr(), base.data_ptr(), cnt.data_ptr(), e0.data_ptr(),
                  M, K, N, K, N, N, y.data_ptr(), _DENSE_GRID, _lib.stream_ptr())
        ctx.save_for_backward(x, w)
        return y

    @staticmethod
    def backward(ctx, dy):
        x, w = ctx.saved_tensors
        M, K = x.shape
        N = w.shape[1]
        dy = dy.to(torch.bfloat16).contiguous()
        base, cnt = _one_segment(M, x.device)
        e0 = _arange_i32(1, x.device)
        s = _lib.stream_ptr()
        dx = dw = None
        if ctx.needs_input_grad[0]:
            dx = torch.empty(M, K, dtype=torch.bfloat16, device=x.device)
            _lib.call("b200moe_dense_dgrad", dy.data_ptr(), w.data_ptr(), base.data_ptr(), cnt.data_ptr(),
                      e0.data_ptr(), M, K, N, N, N, K, dx.data_ptr(), _DENSE_GRID, s)
        if ctx.needs_input_grad[1]:
            dw = torch.empty(K, N, dtype=torch.bfloat16, device=x.device)
            _lib.call("b200moe_dense_wgrad", x.data_ptr(), dy.data_ptr(), base.data_ptr(), cnt.data_ptr(),
                      e0.data_ptr(), M, K, N, K, N, N, dw.data_ptr(), _DENSE_GRID, s)
        return dx, dw


def linear(x: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    """Differentiable x @ w (reference [in, out] weight layout) on the tcgen05
    dense GEMM; bf16 result.  K / N that are not multiples of 256 are padded
    with zeros (exact)."""
    _require_cuda(x, "x")
    if x.dim() != 2 or w.dim() != 2 or x.shape[1] != w.shape[0]:
        raise ShapeError(f"linear shapes disagree: x {tuple(x.shape)}, w {tuple(w.shape)}")
    K, N = w.shape
    Kp, Np = _pad_to(K, GEMM_ALIGN), _pad_to(N, GEMM_ALIGN)
    xb = x.to(torch.bfloat16)
    wb = w.to(torch.bfloat16)
    if Kp != K or Np != N:
        xb = F.pad(xb, (0, Kp - K))
        wb = F.pad(wb, (0, Np - N, 0, Kp - K))
    y = _Linear.apply(xb.contiguous(), wb.contiguous())
    return y[:, :N] if Np != N else y
