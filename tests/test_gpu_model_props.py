"""The reference's own model properties (moefold tests/test_model.py:18-194),
asserted on the B200 model path: exact-zero logits for zero weights, input
validation, causal invariance of position 0, GQA == MHA when kv == heads,
vocabulary-permutation equivariance, rotary positions, the cross-entropy
margin limit and errors, batched == per-sequence, and the same properties
through an MoE checkpoint."""

import math

import numpy as np
import pytest
import torch

import paper_2412_09952_b200 as P
from paper_2412_09952_b200.errors import InputError, SchemaError

pytestmark = pytest.mark.gpu

TINY = dict(vocab=32, hidden=16, layers=2, heads=2, kv_heads=1, ffn_hidden=32, seq_len=16)


@pytest.fixture(scope="module")
def tiny_dense():
    return P.init_dense(P.ModelConfig(**TINY), seed=7)


def logits(ckpt, tokens):
    with torch.no_grad():
        return P.forward_logits(ckpt, tokens).float().cpu()


def test_zero_weight_model_gives_zero_logits():
    ckpt = P.init_dense(P.ModelConfig(**TINY), seed=0)
    for name, t in ckpt.tensors.items():
        if not name.endswith("norm"):
            t.zero_()
    assert torch.count_nonzero(logits(ckpt, np.array([1, 2, 3]))) == 0


def test_input_errors(tiny_dense):
    with pytest.raises(InputError):
        logits(tiny_dense, np.array([TINY["vocab"]]))
    with pytest.raises(InputError):
        logits(tiny_dense, np.zeros(TINY["seq_len"] + 1, dtype=int))
    with pytest.raises(InputError):
        logits(tiny_dense, np.zeros((2, 2, 2), dtype=int))


def test_causal_masking_position_zero_invariant(tiny_dense):
    tokens = np.array([5, 9, 9, 3, 8])
    base = logits(tiny_dense, tokens)
    swapped = tokens.copy()
    swapped[[1, 2]] = swapped[[2, 1]]
    moved = logits(tiny_dense, swapped)
    assert torch.equal(base[0], moved[0])


def test_gqa_equals_mha_when_kv_heads_match_heads():
    from paper_2412_09952_b200.tensor import attention
    r = np.random.default_rng(31)
    t, heads, d = 6, 3, 8
    q, k, v = (r.standard_normal((t, heads * d)) for _ in range(3))

    def reference_mha():
        out = np.zeros((t, heads * d))
        for h in range(heads):
            qh, kh, vh = (a[:, h * d:(h + 1) * d] for a in (q, k, v))
            scores = qh @ kh.T / math.sqrt(d)
            for i in range(t):
                row = scores[i, :i + 1]
                w = np.exp(row - row.max())
                w /= w.sum()
                out[i, h * d:(h + 1) * d] = w @ vh[:i + 1]
        return out

    to = lambda a: torch.from_numpy(a).to("cuda", torch.float32)  # noqa: E731
    got = attention(to(q), to(k), to(v), n_heads=heads, n_kv_heads=heads, seq_len=t).cpu().numpy()
    np.testing.assert_allclose(got, reference_mha(), rtol=2e-5, atol=2e-5)
    # grouped: kv head h serves query heads [h*g, (h+1)*g) (tensor.py:416-419)
    kv = 1
    k1, v1 = k[:, :d], v[:, :d]
    got_g = attention(to(q), to(k1), to(v1), n_heads=heads, n_kv_heads=kv, seq_len=t).cpu().numpy()
    full_k, full_v = np.tile(k1, (1, heads)), np.tile(v1, (1, heads))
    got_m = attention(to(q), to(full_k), to(full_v), n_heads=heads, n_kv_heads=heads, seq_len=t).cpu().numpy()
    np.testing.assert_allclose(got_g, got_m, rtol=2e-5, atol=2e-5)


def test_vocab_permutation_equivariance(tiny_dense):
    cfg = tiny_dense.config
    perm = np.random.default_rng(41).permutation(cfg.vocab)
    tokens = np.array([3, 1, 4, 1, 5])
    base = logits(tiny_dense, tokens)
    t2 = {n: t.clone() for n, t in tiny_dense.tensors.items()}
    pt = torch.from_numpy(perm).cuda()
    t2["embedding"][pt] = tiny_dense.tensors["embedding"]
    t2["lm_head"][:, pt] = tiny_dense.tensors["lm_head"]
    out = logits(P.DenseCheckpoint(config=cfg, tensors=t2), perm[tokens])
    torch.testing.assert_close(out[:, perm], base, rtol=0, atol=0)


def test_rotary_positional_changes_output_but_stays_finite():
    plain = P.init_dense(P.ModelConfig(**TINY), seed=3)
    rot = P.init_dense(P.ModelConfig(**{**TINY, "positional": "rotary"}), seed=3)
    tokens = np.array([1, 2, 3, 4])
    a, b = logits(plain, tokens), logits(rot, tokens)
    assert torch.isfinite(b).all()
    assert not torch.allclose(a, b)
    assert torch.equal(a[0], b[0])     # position 0 is rotated by angle 0


def test_cross_entropy_margin_limit_and_errors():
    prev = None
    for margin in (1.0, 5.0, 20.0, 80.0):
        lg = torch.zeros(2, 8, device="cuda")
        lg[0, 2] = lg[1, 5] = margin
        loss = float(P.cross_entropy(lg, np.array([2, 5])))
        if prev is not None:
            assert loss < prev
        prev = loss
    assert prev < 1e-30
    with pytest.raises(InputError):
        P.cross_entropy(torch.zeros(0, 4, device="cuda"), np.array([], dtype=int))
    with pytest.raises(InputError):
        P.cross_entropy(torch.zeros(2, 4, device="cuda"), np.array([0, 4]))


def test_dense_schema_and_validation(tiny_dense):
    assert set(P.dense_schema(tiny_dense.config)) == set(tiny_dense.tensors)
    tiny_dense.validate()
    broken = P.DenseCheckpoint(config=tiny_dense.config,
                               tensors={k: v for k, v in tiny_dense.tensors.items() if k != "lm_head"})
    with pytest.raises(SchemaError, match="lm_head"):
        broken.validate()


def test_forward_batched_equals_per_sequence(tiny_dense):
    batch = np.random.default_rng(55).integers(0, tiny_dense.config.vocab, (3, 8))
    stacked = logits(tiny_dense, batch)
    rows = torch.cat([logits(tiny_dense, batch[i]) for i in range(3)], 0)
    torch.testing.assert_close(stacked, rows, rtol=0, atol=0)


def test_moe_model_properties():
    """The same invariants through E4T2 MoE layers (dropless, so routing is
    per token and independent of the other tokens)."""
    dense = P.init_dense(P.ModelConfig(**{**TINY, "hidden": 64, "ffn_hidden": 128, "heads": 4, "kv_heads": 2}),
                         seed=5)
    moe = P.upcycle_full(dense, 4, 2, router_seed=2, capacity_factor=None)
    tokens = np.array([5, 9, 9, 3, 8, 1])
    base = logits(moe, tokens)
    swapped = tokens.copy()
    swapped[[1, 2]] = swapped[[2, 1]]
    assert torch.equal(base[0], logits(moe, swapped)[0])
    batch = np.stack([tokens, tokens[::-1]])
    stacked = logits(moe, batch)
    torch.testing.assert_close(stacked[:6], base, rtol=0, atol=0)
    # an upcycled model with identical experts equals the dense model whatever the routing
    # (gates of a token sum to 1 under mixtral top-k; bf16 expert copies of the fp32 FFN)
    dense_bf = {n: (t.to(torch.bfloat16).float() if ".ffn.w" in n else t) for n, t in dense.tensors.items()}
    ref = logits(P.DenseCheckpoint(config=dense.config, tensors=dense_bf), tokens)
    torch.testing.assert_close(base, ref, rtol=2e-2, atol=2e-2)
