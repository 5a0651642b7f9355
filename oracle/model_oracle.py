"""CPU oracle for the transformer step around the MoE layer.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU legs as the checker, never by the product path.

Closed-form numpy restatements of the reference ops, each citing the
reference lines it follows, pinned against tests/golden/model_ops.npz (made
by tests/golden/make_golden_model.py from the reference itself):

  rmsnorm_fwd / rmsnorm_bwd      moefold/tensor.py:307-321
  embedding_fwd / embedding_bwd  moefold/tensor.py:323-337
  cross_entropy_fwd / _bwd       moefold/tensor.py:339-364
  adam_step / sgd_step           moefold/train.py:146-179 (float32 order)
  lr_at                          moefold/train.py:50-65
"""

from __future__ import annotations

import math

import numpy as np

RMSNORM_EPS = 1e-5


def rmsnorm_fwd(x, gain, eps=RMSNORM_EPS):
    """tensor.py:309-312: ms = mean(x^2) + eps; r = ms^-1/2; y = x * r * gain."""
    ms = (x * x).mean(axis=-1, keepdims=True) + eps
    r = ms ** -0.5
    return x * r * gain, r


def rmsnorm_bwd(x, gain, r, g):
    """tensor.py:314-319."""
    h = x.shape[-1]
    gg = g * gain
    dot = (gg * x).sum(axis=-1, keepdims=True)
    dx = r * gg - (r ** 3 / h) * x * dot
    dgain = (g * x * r).reshape(-1, h).sum(axis=0)
    return dx, dgain


def embedding_fwd(table, ids):
    """tensor.py:329."""
    return table[np.asarray(ids, dtype=np.int64)]


def embedding_bwd(table_shape, ids, g, dtype=np.float32):
    """tensor.py:331-335: token-order scatter-add (np.add.at)."""
    out = np.zeros(table_shape, dtype=dtype)
    np.add.at(out, np.asarray(ids, dtype=np.int64), g)
    return out


def cross_entropy_fwd(x, targets):
    """tensor.py:350-358: mean(logsumexp(x) - x[target]); returns (loss, p)."""
    n = targets.shape[0]
    row_max = x.max(axis=1, keepdims=True)
    e = np.exp(x - row_max)
    z = e.sum(axis=1, keepdims=True)
    logz = np.log(z) + row_max
    nll = logz[:, 0] - x[np.arange(n), targets]
    return np.asarray(nll.mean()), e / z


def cross_entropy_bwd(p, targets, g=1.0):
    """tensor.py:360-363."""
    n = targets.shape[0]
    grad = p.copy()
    grad[np.arange(n), targets] -= 1.0
    return grad * (float(g) / n)


def adam_step(p, m, v, g, lr, t, beta1=0.9, beta2=0.999, eps=1e-8):
    """train.py:161-171 on float32 arrays, updated in place (numpy's float32
    evaluation order with Python-float constants rounded to float32)."""
    m *= beta1
    m += (1 - beta1) * g
    v *= beta2
    v += (1 - beta2) * g * g
    mh = m / (1 - beta1 ** t)
    vh = v / (1 - beta2 ** t)
    p -= lr * mh / (np.sqrt(vh) + eps)


def sgd_step(p, buf, g, lr, momentum=0.9):
    """train.py:172-176."""
    buf *= momentum
    buf += g
    p -= lr * buf


def lr_at(step, lr_max, lr_min, warmup, total):
    """train.py:50-65: linear warmup then cosine decay, exact endpoints."""
    if step < warmup:
        return lr_max * step / warmup
    if step == warmup:
        return lr_max
    if step == total:
        return lr_min
    progress = (step - warmup) / (total - warmup)
    return lr_min + 0.5 * (lr_max - lr_min) * (1.0 + math.cos(math.pi * progress))
