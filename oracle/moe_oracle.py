"""ORACLE -- CPU restatement of the reference MoE-layer hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(`paper_2412_09952_b200/`) imports this module; only `tests/`,
`__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline` leg and
`--impl reference`) may use it, and only as the checker / the CPU arm.

It restates, over plain numpy arrays and in closed form, what the reference
package `moefold` computes with its tape autograd:

  * router logits + learned-scale noise      moefold/moe.py:136-149
  * stable top-k mask                         moefold/moe.py:152-162
  * masked softmax fwd/bwd                    moefold/tensor.py:267-297
  * mixtral / st gate orderings               moefold/moe.py:171-186
  * capacity                                  moefold/moe.py:189-196
  * dispatch (position / score policies)      moefold/moe.py:206-240
  * expert SwiGLU + gate-weighted combine     moefold/moe.py:131-133, 250-283
  * backward of all of the above              moefold/tensor.py:168-227, 371-403
  * importance (CV^2) load-balancing loss     moefold/tensor.py:503-521
  * router init / upcycling copies            moefold/upcycle.py:72-115, 156-227
  * dense init                                moefold/model.py:56-74, 99-113

Numerics follow the reference op for op (same dtype promotion, same numpy
reductions, numpy's own float32 `exp`), so that in float32 the routing bits
(top-k, gates, kept/dropped) are identical to the reference's; this is
pinned against golden vectors produced by the reference itself
(tests/golden/make_golden.py -> tests/test_oracle.py).

The arithmetic lives in numpy (unpinned in the reference, `pkg/pyproject.toml:10-13`;
fixtures were generated with numpy 2.3.5 / OpenBLAS 0.3.30 on an AVX512_SPR host).
"""

from __future__ import annotations

import math
import os
import ctypes
from dataclasses import dataclass, field

import numpy as np

ROUTER_INIT_STD = 0.02   # moefold/upcycle.py:30
INIT_STD = 0.02          # moefold/model.py:22


class OracleGateError(ValueError):
    """Mirror of moefold.errors.GateError raised by the oracle."""


class OracleConfigError(ValueError):
    """Mirror of moefold.errors.ConfigError raised by the oracle."""


# --------------------------------------------------------------------------
# RNG (moefold/rng.py:20-50): numpy Philox4x64-10 keyed by (seed, stream)
# --------------------------------------------------------------------------

def rng(seed: int, stream: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=np.array([seed, stream], dtype=np.uint64)))


# --------------------------------------------------------------------------
# exp: numpy's float32 exp, or the C port of its AVX512F kernel
# --------------------------------------------------------------------------

_NPEXP = None


def _npexp_lib():
    global _NPEXP
    if _NPEXP is None:
        here = os.path.dirname(os.path.abspath(__file__))
        path = os.path.join(here, "build", "libnpexp.so")
        if not os.path.exists(path):
            build_oracle()
        lib = ctypes.CDLL(path)
        lib.npexp_f32_array.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]
        _NPEXP = lib
    return _NPEXP


def build_oracle() -> str:
    """Compile oracle/npexp.c and oracle/crc32c.c (the checkers) into
    oracle/build/libnpexp.so."""
    import subprocess
    here = os.path.dirname(os.path.abspath(__file__))
    os.makedirs(os.path.join(here, "build"), exist_ok=True)
    out = os.path.join(here, "build", "libnpexp.so")
    subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC",
                           os.path.join(here, "npexp.c"), os.path.join(here, "crc32c.c"), "-o", out, "-lm"])
    return out


def exp_port(x: np.ndarray) -> np.ndarray:
    """C port of numpy's AVX512F float32 exp (see npexp.c)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    y = np.empty_like(x)
    _npexp_lib().npexp_f32_array(x.ctypes.data, y.ctypes.data, x.size)
    return y


def _exp(x: np.ndarray, impl: str) -> np.ndarray:
    if impl == "numpy" or x.dtype != np.float32:
        return np.exp(x)
    if impl == "port":
        return exp_port(x)
    raise ValueError(impl)


# --------------------------------------------------------------------------
# elementwise pieces (moefold/tensor.py:210-241)
# --------------------------------------------------------------------------

def sigmoid(x: np.ndarray) -> np.ndarray:
    # tensor.py:239-241 (branch-free stable form)
    e = np.exp(-np.abs(x))
    return np.where(x >= 0, 1.0 / (1.0 + e), e / (1.0 + e))


def softplus(x: np.ndarray) -> np.ndarray:
    # tensor.py:235-236
    return np.maximum(x, 0.0) + np.log1p(np.exp(-np.abs(x)))


# --------------------------------------------------------------------------
# masked softmax (moefold/tensor.py:267-297)
# --------------------------------------------------------------------------

def masked_softmax(x: np.ndarray, mask: np.ndarray | None = None, exp_impl: str = "numpy"):
    """Row softmax over the last axis; returns (p, keep).  Masked and
    non-finite entries get exactly 0; a row with nothing kept raises."""
    keep = np.isfinite(x) if mask is None else (np.asarray(mask, dtype=bool) & np.isfinite(x))
    if not keep.any(axis=-1).all():
        raise OracleGateError("softmax row with all entries masked")
    row_max = np.max(np.where(keep, x, -np.inf), axis=-1, keepdims=True)
    shifted = np.where(keep, x, row_max) - row_max
    e = np.where(keep, _exp(shifted, exp_impl), 0.0)
    p = e / e.sum(axis=-1, keepdims=True)
    return p, keep


def masked_softmax_bwd(p: np.ndarray, keep: np.ndarray, g: np.ndarray) -> np.ndarray:
    # tensor.py:292-295
    g_eff = g * keep
    dot = (p * g_eff).sum(axis=-1, keepdims=True)
    return np.where(keep, p * (g_eff - dot), 0.0)


# --------------------------------------------------------------------------
# top-k and gate orderings (moefold/moe.py:152-186)
# --------------------------------------------------------------------------

def top_k_mask(values: np.ndarray, k: int) -> np.ndarray:
    """k largest per row; ties -> lowest index (stable sort of -v); NaN last."""
    v = np.atleast_2d(np.asarray(values))
    n = v.shape[-1]
    if not (1 <= k <= n):
        raise OracleConfigError(f"top-k out of range: k={k}, n={n}")
    order = np.argsort(-v, axis=-1, kind="stable")[:, :k]
    keep = np.zeros(v.shape, dtype=bool)
    np.put_along_axis(keep, order, True, axis=-1)
    return keep.reshape(np.asarray(values).shape)


@dataclass
class Gating:
    gates: np.ndarray      # [T, E] post-top-k gates (pre-capacity)
    topk: np.ndarray       # [T, E] bool top-k selection on the logits
    probs: np.ndarray      # softmax output feeding the backward
    sm_keep: np.ndarray    # softmax keep mask feeding the backward
    router_type: str


def gate(h: np.ndarray, k: int, router_type: str, exp_impl: str = "numpy") -> Gating:
    topk = top_k_mask(h, k)
    if router_type == "mixtral":
        # moe.py:171-173: mask first, softmax over the survivors
        p, keep = masked_softmax(h, mask=topk, exp_impl=exp_impl)
        return Gating(gates=p, topk=topk, probs=p, sm_keep=keep, router_type=router_type)
    if router_type == "st":
        # moe.py:176-186: softmax over all, then multiply by the logit top-k mask
        s, keep = masked_softmax(h, exp_impl=exp_impl)
        return Gating(gates=s * topk.astype(s.dtype), topk=topk, probs=s, sm_keep=keep,
                      router_type=router_type)
    raise OracleConfigError(router_type)


def gate_bwd(gt: Gating, dg: np.ndarray) -> np.ndarray:
    if gt.router_type == "mixtral":
        return masked_softmax_bwd(gt.probs, gt.sm_keep, dg)
    return masked_softmax_bwd(gt.probs, gt.sm_keep, dg * gt.topk.astype(dg.dtype))


# --------------------------------------------------------------------------
# capacity + dispatch (moefold/moe.py:189-240)
# --------------------------------------------------------------------------

def expert_capacity(tokens: int, n_experts: int, cf: float | None) -> int | None:
    if tokens < 1:
        raise OracleConfigError(f"tokens_per_batch must be >= 1, got {tokens}")
    if cf is None:
        return None
    return int(math.ceil(tokens * cf / n_experts - 1e-9))


@dataclass
class Dispatch:
    kept: np.ndarray       # [T, E] bool
    dropped: np.ndarray    # [T, E] bool
    assigned: np.ndarray   # [E] int64
    n_dropped: int
    total_slots: int
    gate_mass: np.ndarray  # [E]
    capacity: int | None

    def rows(self) -> np.ndarray:
        """[T, E] int64 capacity-slot index of each kept (t, e), -1 elsewhere:
        the rank of t among the kept tokens of expert e in token order."""
        r = np.cumsum(self.kept, axis=0) - 1
        return np.where(self.kept, r, -1)


def dispatch(g: np.ndarray, capacity: int | None, policy: str = "position") -> Dispatch:
    if policy not in ("position", "score"):
        raise OracleConfigError(policy)
    slots = g > 0
    kept = slots.copy()
    if capacity is not None:
        for e in range(g.shape[1]):
            cand = np.flatnonzero(slots[:, e])
            if cand.size <= capacity:
                continue
            if policy == "score":
                cand = cand[np.argsort(-g[cand, e], kind="stable")]
            kept[cand[capacity:], e] = False
    dropped = slots & ~kept
    return Dispatch(kept=kept, dropped=dropped, assigned=kept.sum(axis=0).astype(np.int64),
                    n_dropped=int(dropped.sum()), total_slots=int(slots.sum()),
                    gate_mass=np.where(kept, g, 0.0).sum(axis=0), capacity=capacity)


# --------------------------------------------------------------------------
# importance (CV^2) penalty (moefold/tensor.py:503-521)
# --------------------------------------------------------------------------

def importance_penalty(g: np.ndarray):
    """Returns (loss, dloss/dg as an [E] row broadcast over tokens)."""
    imp = g.sum(axis=0)
    n = imp.shape[0]
    mean = imp.mean()
    if mean <= 0:
        raise OracleGateError("importance penalty needs positive total gate mass")
    var = ((imp - mean) ** 2).mean()
    loss = var / mean ** 2
    dimp = 2.0 * (imp - mean) / (n * mean ** 2) - 2.0 * var / (n * mean ** 3)
    return loss, dimp


# --------------------------------------------------------------------------
# the layer: forward + closed-form backward
# --------------------------------------------------------------------------

@dataclass
class LayerCfg:
    n_experts: int = 8
    top_k: int = 2
    router_type: str = "mixtral"
    noise: bool = False            # noise_enabled AND training
    capacity_factor: float | None = None
    drop_policy: str = "position"


@dataclass
class ForwardCache:
    x: np.ndarray
    wg: np.ndarray
    wn: np.ndarray
    w1: list
    w2: list
    w3: list
    z: np.ndarray | None
    an: np.ndarray | None
    logits: np.ndarray
    gating: Gating
    disp: Dispatch
    per_expert: dict = field(default_factory=dict)


def router_logits(x, wg, wn=None, z=None):
    """moe.py:136-149: clean = x@W_g; with noise h = clean + z*softplus(x@W_noise)."""
    clean = x @ wg
    if z is None:
        return clean, None
    an = x @ wn
    return clean + z.astype(x.dtype) * softplus(an), an


def moe_forward(x, wg, wn, w1, w2, w3, cfg: LayerCfg, z=None, logits=None, exp_impl="numpy"):
    """Forward of moefold.moe.moe_forward (moe.py:250-283).

    x: [T,H]; wg,wn: [H,E]; w1[e],w3[e]: [H,F]; w2[e]: [F,H] (all [in,out]).
    `logits` (optional) overrides x@W_g (+noise): the parity rule feeds the
    device's fp32 logits here so routing is compared from identical inputs.
    Returns (y, gates, cache)."""
    T = x.shape[0]
    E = cfg.n_experts
    if len(w1) != E:
        raise OracleConfigError("expert count mismatch")
    an = None
    if logits is None:
        h, an = router_logits(x, wg, wn, z if cfg.noise else None)
    else:
        h = np.asarray(logits)
        if cfg.noise:
            an = x @ wn
    gt = gate(h, cfg.top_k, cfg.router_type, exp_impl=exp_impl)
    cap = expert_capacity(T, E, cfg.capacity_factor)
    disp = dispatch(gt.gates, cap, cfg.drop_policy)
    cache = ForwardCache(x=x, wg=wg, wn=wn, w1=w1, w2=w2, w3=w3, z=z if cfg.noise else None,
                         an=an, logits=h, gating=gt, disp=disp)
    y = None
    for e in range(E):
        idx = np.flatnonzero(disp.kept[:, e])
        if idx.size == 0:
            continue
        xe = x[idx]
        a = xe @ w1[e]
        b = xe @ w3[e]
        sig = sigmoid(a)
        m = (a * sig) * b
        o = m @ w2[e]
        ge = gt.gates[idx, e:e + 1]
        contrib = np.zeros((T, x.shape[1]), dtype=o.dtype)
        contrib[idx] = o * ge
        y = contrib if y is None else y + contrib
        cache.per_expert[e] = dict(idx=idx, a=a, b=b, sig=sig, m=m, o=o, ge=ge)
    if y is None:
        y = np.zeros_like(x)
    return y, gt.gates, cache


def moe_backward(cache: ForwardCache, dy, dgates=None):
    """Closed-form backward of moe_forward (verified against the
    reference tape to <=2.7e-15 in fp64).  `dgates`: upstream gradient on the
    returned pre-capacity gates (e.g. lambda * importance-penalty grad, a [E]
    row or a full [T,E] array).  Returns dict of gradients."""
    x = cache.x
    T, H = x.shape
    E = len(cache.w1)
    dg = np.zeros_like(cache.gating.gates)
    dx = np.zeros_like(x)
    dW1 = [np.zeros_like(w) for w in cache.w1]
    dW2 = [np.zeros_like(w) for w in cache.w2]
    dW3 = [np.zeros_like(w) for w in cache.w3]
    for e in range(E):
        pe = cache.per_expert.get(e)
        if pe is None:
            continue
        idx = pe["idx"]
        d = dy[idx]
        do = d * pe["ge"]
        dg[idx, e] += (d * pe["o"]).sum(axis=1)
        dW2[e] = pe["m"].T @ do
        dm = do @ cache.w2[e].T
        a, b, sig = pe["a"], pe["b"], pe["sig"]
        dsilu = dm * b
        db = dm * (a * sig)
        da = dsilu * sig * (1.0 + a * (1.0 - sig))
        dW1[e] = x[idx].T @ da
        dW3[e] = x[idx].T @ db
        dx[idx] += da @ cache.w1[e].T + db @ cache.w3[e].T
    if dgates is not None:
        dg = dg + dgates
    dh = gate_bwd(cache.gating, dg)
    dwg = x.T @ dh
    dx = dx + dh @ cache.wg.T
    dwn = np.zeros_like(cache.wg)
    if cache.z is not None:
        dan = dh * cache.z.astype(x.dtype) * sigmoid(cache.an)
        dwn = x.T @ dan
        dx = dx + dan @ cache.wn.T
    return dict(dx=dx, dwg=dwg, dwn=dwn, dw1=dW1, dw2=dW2, dw3=dW3, dh=dh, dg=dg)


# --------------------------------------------------------------------------
# sampled evaluation at full size (the closed form above, restricted to a
# subset of token rows or of ffn columns).  At the Llama shape a whole oracle
# fwd+bwd costs minutes of host time; these pieces recompute exactly the same
# arithmetic for chosen rows / columns so the device can be checked at the
# benchmarked size.  Same formulas as moe_forward / moe_backward
# (moe.py:250-283, tensor.py:192-217, 292-295).
# --------------------------------------------------------------------------

def expert_rows(xe, dye, ge, w1, w2, w3):
    """One expert on a set of its kept rows (moe.py:131-133, 272-280 and the
    matmul/silu backward closures tensor.py:192-217).  xe, dye: [n, H];
    ge: [n] gates.  Returns (ge*o [n,H], dg=<dy,o> [n], dx part [n,H])."""
    ge = np.asarray(ge)[:, None]
    a = xe @ w1
    b = xe @ w3
    sig = sigmoid(a)
    m = (a * sig) * b
    o = m @ w2
    do = dye * ge
    dm = do @ w2.T
    da = dm * b * sig * (1.0 + a * (1.0 - sig))
    db = dm * (a * sig)
    return o * ge, (dye * o).sum(axis=1), da @ w1.T + db @ w3.T


def expert_wgrad_columns(xe, dye, ge, w1_cols, w3_cols, w2_rows):
    """Weight gradients of one expert restricted to a block J of ffn units:
    dW1[:, J], dW3[:, J] ([H, |J|]) and dW2[J, :] ([|J|, H]) over ALL of the
    expert's kept rows xe [M_e, H] (tensor.py:192-207: dB += A^T dC).  Only
    the J columns of a, b, m and dm are needed, so the cost is O(M_e H |J|)."""
    ge = np.asarray(ge)[:, None]
    do = dye * ge
    a = xe @ w1_cols
    b = xe @ w3_cols
    sig = sigmoid(a)
    m = (a * sig) * b
    dm = do @ w2_rows.T
    da = dm * b * sig * (1.0 + a * (1.0 - sig))
    db = dm * (a * sig)
    return xe.T @ da, xe.T @ db, m.T @ do


def router_bwd_rows(logits_rows, k, router_type, dg_rows, x_rows, wg, wn=None, z_rows=None, an_rows=None):
    """Router backward for a subset of token rows (rows are independent):
    softmax' (tensor.py:292-295) on the given gate gradients, then the router
    contribution to dx and, with noise, the softplus-noise branch
    (tensor.py:220-227).  Returns (dh rows, dx part rows, dn rows or None)."""
    sub = gate(logits_rows, k, router_type)
    dh = gate_bwd(sub, dg_rows)
    dx = dh @ wg.T
    dn = None
    if z_rows is not None:
        dn = dh * z_rows.astype(dh.dtype) * sigmoid(an_rows)
        dx = dx + dn @ wn.T
    return dh, dx, dn


# --------------------------------------------------------------------------
# dense init + upcycling (moefold/model.py:56-113, moefold/upcycle.py:46-227)
# --------------------------------------------------------------------------

def dense_schema(vocab, hidden, layers, kv_width, ffn_hidden):
    s = {"embedding": (vocab, hidden), "lm_head": (hidden, vocab), "final_norm": (hidden,)}
    for i in range(layers):
        p = f"layers.{i}"
        s[f"{p}.attn_norm"] = (hidden,)
        s[f"{p}.attn.wq"] = (hidden, hidden)
        s[f"{p}.attn.wk"] = (hidden, kv_width)
        s[f"{p}.attn.wv"] = (hidden, kv_width)
        s[f"{p}.attn.wo"] = (hidden, hidden)
        s[f"{p}.ffn_norm"] = (hidden,)
        s[f"{p}.ffn.w1"] = (hidden, ffn_hidden)
        s[f"{p}.ffn.w2"] = (ffn_hidden, hidden)
        s[f"{p}.ffn.w3"] = (hidden, ffn_hidden)
    return s


def init_dense(schema: dict, seed: int, dtype=np.float64) -> dict:
    """Draw order: sorted tensor names from Rng(seed, 0); norms are ones."""
    g = rng(seed, 0)
    out = {}
    for name, shape in sorted(schema.items()):
        if name.endswith("norm"):
            out[name] = np.ones(shape, dtype=dtype)
        else:
            out[name] = (g.standard_normal(size=shape) * INIT_STD).astype(dtype)
    return out


def router_weights(hidden: int, n_experts: int, layer: int, router_seed: int, dtype):
    w_g = (rng(router_seed, layer).standard_normal(size=(hidden, n_experts)) * ROUTER_INIT_STD).astype(dtype)
    return w_g, np.zeros((hidden, n_experts), dtype=dtype)


# --------------------------------------------------------------------------
# CPU timing helper for bench.py's cpu_baseline / --impl reference
# --------------------------------------------------------------------------

def time_fwd_bwd(T, H, F, E=8, k=2, cf=1.0, router_type="mixtral", policy="position",
                 aux=0.01, seed=0, reps=1, dtype=np.float32):
    """Seconds per oracle fwd+bwd (fp32) at the given shape, best of `reps`.
    Upcycled layer: every expert is the same dense FFN (bitwise copies)."""
    import time
    g = rng(seed, 0)
    w1 = (g.standard_normal((H, F)) * 0.02).astype(dtype)
    w2 = (g.standard_normal((F, H)) * 0.02).astype(dtype)
    w3 = (g.standard_normal((H, F)) * 0.02).astype(dtype)
    wg, wn = router_weights(H, E, 0, 1, dtype)
    x = rng(123, 0).standard_normal((T, H)).astype(dtype)
    dy = rng(124, 0).standard_normal((T, H)).astype(dtype)
    cfg = LayerCfg(n_experts=E, top_k=k, router_type=router_type, capacity_factor=cf, drop_policy=policy)
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        y, gates, cache = moe_forward(x, wg, wn, [w1] * E, [w2] * E, [w3] * E, cfg)
        _, dimp = importance_penalty(gates)
        moe_backward(cache, dy, dgates=aux * dimp)
        best = min(best, time.perf_counter() - t0)
    return best
