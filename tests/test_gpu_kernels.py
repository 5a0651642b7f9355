"""Kernel-level parity on a B200: every C-ABI entry point against the CPU
oracle / golden vectors (routing, bit-exact) or a float32 torch restatement of
the same contraction (grouped GEMMs, tolerance)."""

import os

import numpy as np
import pytest
import torch

from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2412_09952_b200 import _lib
    import paper_2412_09952_b200 as B
from oracle import moe_oracle as O


@pytest.fixture(autouse=True)
def _reset_gemm_knobs():
    """Tests below flip the (thread-local) GEMM diagnostics knobs; put the
    product defaults back after every test, passed or failed."""
    yield
    if torch.cuda.is_available():
        _lib.call("b200moe_gemm_set_cta_group", 2)
        _lib.call("b200moe_gemm_set_debug", 0)
        _lib.call("b200moe_gemm_set_max_ctas", 148)


def bits_equal(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and a.tobytes() == b.tobytes()


def rel(a, b):
    a = a.double()
    b = b.double()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


# --------------------------------------------------------------------------
# grouped GEMMs
# --------------------------------------------------------------------------

def _segments(counts, dev):
    base, acc = [], 0
    for c in counts:
        base.append(acc)
        acc += (c + 127) // 128 * 128
    R = acc + 256
    return (torch.tensor(base, dtype=torch.int32, device=dev), torch.tensor(counts, dtype=torch.int32, device=dev),
            torch.arange(len(counts), dtype=torch.int32, device=dev), R)


def _rows(base, counts, e):
    return torch.arange(int(base[e]), int(base[e]) + int(counts[e]), device=base.device)


def _fill_rows(R, C, base, counts, dev, scale=1.0, seed=0):
    g = torch.Generator(device=dev).manual_seed(seed)
    t = torch.zeros(R, C, dtype=torch.bfloat16, device=dev)
    for e in range(len(counts)):
        r = _rows(base, counts, e)
        t[r] = (torch.randn(len(r), C, generator=g, device=dev) * scale).to(torch.bfloat16)
    return t


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("H,F,counts", [(256, 512, [300, 129]), (512, 768, [1, 0, 513]), (256, 256, [1024])])
def test_grouped_gemm_all_modes(cg, H, F, counts):
    dev = torch.device("cuda")
    _lib.call("b200moe_gemm_set_cta_group", cg)
    E = len(counts)
    base, cnt, sege, R = _segments(counts, dev)
    s = _lib.stream_ptr()
    g = torch.Generator(device=dev).manual_seed(1)
    W1 = (torch.randn(E, F, H, generator=g, device=dev) * 0.05).to(torch.bfloat16)
    W3 = (torch.randn(E, F, H, generator=g, device=dev) * 0.05).to(torch.bfloat16)
    W2 = (torch.randn(E, H, F, generator=g, device=dev) * 0.05).to(torch.bfloat16)
    xp = _fill_rows(R, H, base, cnt, dev, seed=2)
    bf = dict(dtype=torch.bfloat16, device=dev)
    A, Bm, Hh = (torch.full((R, F), float("nan"), **bf) for _ in range(3))
    _lib.call("b200moe_expert_fwd1", xp.data_ptr(), W1.data_ptr(), W3.data_ptr(), base.data_ptr(), cnt.data_ptr(),
              sege.data_ptr(), E, R, H, F, E, A.data_ptr(), Bm.data_ptr(), Hh.data_ptr(), s)
    Oo = torch.full((R, H), float("nan"), **bf)
    _lib.call("b200moe_expert_fwd2", Hh.data_ptr(), W2.data_ptr(), base.data_ptr(), cnt.data_ptr(), sege.data_ptr(),
              E, R, H, F, E, Oo.data_ptr(), s)
    dO = _fill_rows(R, H, base, cnt, dev, seed=3)
    dA, dB = (torch.full((R, F), float("nan"), **bf) for _ in range(2))
    _lib.call("b200moe_expert_bwd2", dO.data_ptr(), W2.data_ptr(), A.data_ptr(), Bm.data_ptr(), base.data_ptr(),
              cnt.data_ptr(), sege.data_ptr(), E, R, H, F, E, dA.data_ptr(), dB.data_ptr(), s)
    # BWD2 that also rebuilds h = silu(a) * b (callers that dropped the forward's h)
    dA2, dB2, H2 = (torch.full((R, F), float("nan"), **bf) for _ in range(3))
    _lib.call("b200moe_expert_bwd2_h", dO.data_ptr(), W2.data_ptr(), A.data_ptr(), Bm.data_ptr(), base.data_ptr(),
              cnt.data_ptr(), sege.data_ptr(), E, R, H, F, E, dA2.data_ptr(), dB2.data_ptr(), H2.data_ptr(), 0, s)
    dW1, dW3 = (torch.full((E, F, H), float("nan"), **bf) for _ in range(2))
    dW2 = torch.full((E, H, F), float("nan"), **bf)
    _lib.call("b200moe_expert_wgrad", xp.data_ptr(), Hh.data_ptr(), dO.data_ptr(), dA.data_ptr(), dB.data_ptr(),
              base.data_ptr(), cnt.data_ptr(), sege.data_ptr(), E, R, H, F, E, dW1.data_ptr(), dW2.data_ptr(),
              dW3.data_ptr(), s)
    dxp = torch.full((R, H), float("nan"), **bf)
    _lib.call("b200moe_expert_bwd1", dA.data_ptr(), dB.data_ptr(), W1.data_ptr(), W3.data_ptr(), base.data_ptr(),
              cnt.data_ptr(), sege.data_ptr(), E, R, H, F, E, dxp.data_ptr(), s)
    torch.cuda.synchronize()
    for e in range(E):
        r = _rows(base, cnt, e)
        pad = torch.arange(int(base[e]) + counts[e], int(base[e]) + (counts[e] + 127) // 128 * 128, device=dev)
        x = xp[r].float()
        a = x @ W1[e].float().t()
        b = x @ W3[e].float().t()
        if len(r):
            assert rel(A[r].float(), a) < 1e-2, ("fwd1 a", e)
            assert rel(Bm[r].float(), b) < 1e-2, ("fwd1 b", e)
            h = torch.nn.functional.silu(A[r].float()) * Bm[r].float()
            assert rel(Hh[r].float(), h) < 1e-2, ("fwd1 h", e)
            o = Hh[r].float() @ W2[e].float().t()
            assert rel(Oo[r].float(), o) < 1e-2, ("fwd2", e)
            dm = dO[r].float() @ W2[e].float()
            av, bv = A[r].float(), Bm[r].float()
            sg = torch.sigmoid(av)
            assert rel(dA[r].float(), dm * bv * sg * (1 + av * (1 - sg))) < 1e-2, ("bwd2 da", e)
            assert rel(dB[r].float(), dm * av * sg) < 1e-2, ("bwd2 db", e)
            assert torch.equal(dA2[r], dA[r]) and torch.equal(dB2[r], dB[r]), ("bwd2_h da/db", e)
            assert rel(H2[r].float(), torch.nn.functional.silu(av) * bv) < 1e-2, ("bwd2_h h", e)
            assert rel(H2[r].float(), Hh[r].float()) < 1e-2, ("bwd2_h h vs forward h", e)
            dx = dA[r].float() @ W1[e].float() + dB[r].float() @ W3[e].float()
            assert rel(dxp[r].float(), dx) < 1e-2, ("bwd1", e)
        if len(pad):  # padded rows must come out exactly zero
            for t, n in ((A, "A"), (Hh, "H"), (dA, "dA"), (dB, "dB"), (Oo, "O"), (dxp, "dxp"), (H2, "H2")):
                assert bool((t[pad] == 0).all()), ("pad", n, e)
        gw1 = dA[r].float().t() @ x
        gw3 = dB[r].float().t() @ x
        gw2 = dO[r].float().t() @ Hh[r].float()
        if len(r):
            assert rel(dW1[e].float(), gw1) < 1e-2, ("wgrad dW1", e)
            assert rel(dW3[e].float(), gw3) < 1e-2, ("wgrad dW3", e)
            assert rel(dW2[e].float(), gw2) < 1e-2, ("wgrad dW2", e)
        else:
            assert bool((dW1[e] == 0).all() and (dW2[e] == 0).all() and (dW3[e] == 0).all()), ("empty expert", e)
    _lib.call("b200moe_gemm_set_cta_group", 2)


@pytest.mark.parametrize("H,F,counts,owners", [
    (256, 1024, [1, 0, 513], [0, 1, 2]),
    (512, 512, [300, 129, 700, 64], [0, 1, 0, 1]),      # EP layout: two source segments per expert
    (256, 512, [1024, 1024], [0, 1]),
])
def test_wgrad_wide_tiles_match_one_accumulator_tiles(H, F, counts, owners):
    """The opt-in wide WGRAD tiles (debug bit 256: dW1/dW3 sharing xp, dW2 column pairs sharing do)
    issue the same MMA sequence into each accumulator as the one-accumulator
    tiles, so the weight gradients must be bit-identical; both are also checked
    against an fp32 reference."""
    dev = torch.device("cuda")
    _lib.call("b200moe_gemm_set_cta_group", 2)
    E = max(owners) + 1
    base, cnt, _, R = _segments(counts, dev)
    sege = torch.tensor(owners, dtype=torch.int32, device=dev)
    nseg = len(counts)
    xp = _fill_rows(R, H, base, cnt, dev, seed=1)
    Hh = _fill_rows(R, F, base, cnt, dev, seed=2)
    dO = _fill_rows(R, H, base, cnt, dev, seed=3)
    dA = _fill_rows(R, F, base, cnt, dev, seed=4)
    dB = _fill_rows(R, F, base, cnt, dev, seed=5)
    bf = dict(dtype=torch.bfloat16, device=dev)
    s = _lib.stream_ptr()
    outs = []
    for debug in (0, 256):
        _lib.call("b200moe_gemm_set_debug", debug)
        dW1, dW3 = (torch.full((E, F, H), float("nan"), **bf) for _ in range(2))
        dW2 = torch.full((E, H, F), float("nan"), **bf)
        _lib.call("b200moe_expert_wgrad", xp.data_ptr(), Hh.data_ptr(), dO.data_ptr(), dA.data_ptr(),
                  dB.data_ptr(), base.data_ptr(), cnt.data_ptr(), sege.data_ptr(), nseg, R, H, F, E,
                  dW1.data_ptr(), dW2.data_ptr(), dW3.data_ptr(), s)
        torch.cuda.synchronize()
        outs.append((dW1, dW2, dW3))
    _lib.call("b200moe_gemm_set_debug", 0)
    for w, n in zip(range(3), ("dW1", "dW2", "dW3")):
        assert torch.equal(outs[0][w], outs[1][w]), n
    dW1, dW2, dW3 = outs[0]
    for e in range(E):
        r = torch.cat([_rows(base, cnt, s_) for s_ in range(nseg) if owners[s_] == e])
        if len(r) == 0:
            assert bool((dW1[e] == 0).all() and (dW2[e] == 0).all() and (dW3[e] == 0).all()), e
            continue
        x = xp[r].float()
        assert rel(dW1[e].float(), dA[r].float().t() @ x) < 1e-2, ("dW1", e)
        assert rel(dW3[e].float(), dB[r].float().t() @ x) < 1e-2, ("dW3", e)
        assert rel(dW2[e].float(), dO[r].float().t() @ Hh[r].float()) < 1e-2, ("dW2", e)


@pytest.mark.parametrize("cg", [1, 2])
def test_wgrad_accumulate_into_existing_gradients(cg):
    """b200moe_expert_wgrad_acc: accumulate=0 is the plain WGRAD (bitwise);
    accumulate=1 adds the new gradient to the bf16 values already in the
    outputs (fp32 add, one rounding), empty experts keep their old values."""
    dev = torch.device("cuda")
    _lib.call("b200moe_gemm_set_cta_group", cg)
    H, F, counts = 256, 512, [300, 0, 700]
    E = len(counts)
    base, cnt, sege, R = _segments(counts, dev)
    xp = _fill_rows(R, H, base, cnt, dev, seed=1)
    Hh = _fill_rows(R, F, base, cnt, dev, seed=2)
    dO = _fill_rows(R, H, base, cnt, dev, seed=3)
    dA = _fill_rows(R, F, base, cnt, dev, seed=4)
    dB = _fill_rows(R, F, base, cnt, dev, seed=5)
    bf = dict(dtype=torch.bfloat16, device=dev)
    s = _lib.stream_ptr()
    g = torch.Generator(device=dev).manual_seed(9)
    old = [torch.randn(E, F, H, generator=g, device=dev).to(torch.bfloat16),
           torch.randn(E, H, F, generator=g, device=dev).to(torch.bfloat16),
           torch.randn(E, F, H, generator=g, device=dev).to(torch.bfloat16)]

    def run(outs, acc):
        _lib.call("b200moe_expert_wgrad_acc", xp.data_ptr(), Hh.data_ptr(), dO.data_ptr(), dA.data_ptr(),
                  dB.data_ptr(), base.data_ptr(), cnt.data_ptr(), sege.data_ptr(), E, R, H, F, E,
                  outs[0].data_ptr(), outs[1].data_ptr(), outs[2].data_ptr(), acc, s)

    plain = [torch.full_like(o, float("nan")) for o in old]
    _lib.call("b200moe_expert_wgrad", xp.data_ptr(), Hh.data_ptr(), dO.data_ptr(), dA.data_ptr(), dB.data_ptr(),
              base.data_ptr(), cnt.data_ptr(), sege.data_ptr(), E, R, H, F, E, plain[0].data_ptr(),
              plain[1].data_ptr(), plain[2].data_ptr(), s)
    fresh = [torch.full_like(o, float("nan")) for o in old]
    run(fresh, 0)
    acc = [o.clone() for o in old]
    run(acc, 1)
    torch.cuda.synchronize()
    _lib.call("b200moe_gemm_set_cta_group", 2)
    for i in range(3):
        assert torch.equal(fresh[i], plain[i]), i
    for e in range(E):
        r = _rows(base, cnt, e)
        if len(r) == 0:
            for i in range(3):
                assert torch.equal(acc[i][e], old[i][e]), ("empty expert keeps its gradient", i)
            continue
        x = xp[r].float()
        new = [dA[r].float().t() @ x, dO[r].float().t() @ Hh[r].float(), dB[r].float().t() @ x]
        for i in range(3):
            want = old[i][e].float() + new[i]
            assert rel(acc[i][e].float(), want) < 1e-2, (i, e)


# --------------------------------------------------------------------------
# router: gate arithmetic bit-exact vs the reference goldens
# --------------------------------------------------------------------------

def _gate_dev(h, k, rt):
    g, p, topk, err = B.moe._gate(torch.from_numpy(np.ascontiguousarray(h)).cuda(), k, rt, want_topk=True)
    return g.cpu().numpy(), topk.cpu().numpy().astype(bool), int(err.item())


@pytest.mark.parametrize("rt", ["mixtral", "st"])
def test_gate_from_reference_logits_bit_exact(rt):
    cfg1 = np.load(os.path.join(GOLDEN, "routing_cfg1.npz"))
    g, topk, err = _gate_dev(cfg1["logits"], 2, rt)
    assert err == 0
    assert bits_equal(g, cfg1[f"{rt}_gates"])
    assert np.array_equal(topk, O.top_k_mask(cfg1["logits"], 2))


@pytest.mark.parametrize("rt", ["mixtral", "st"])
@pytest.mark.parametrize("k", [1, 2, 3, 4, 8])
def test_gate_edge_rows_bit_exact(rt, k):
    edge = np.load(os.path.join(GOLDEN, "routing_edge.npz"))
    g, topk, err = _gate_dev(edge["logits"], k, rt)
    assert err == 0
    ref = edge[f"{rt}_k{k}_gates"]
    bad = np.nonzero((g.view(np.uint32) != ref.view(np.uint32)).any(axis=1))[0]
    assert bad.size == 0, (bad[:5], edge["logits"][bad[:3]], g[bad[:3]], ref[bad[:3]])
    assert np.array_equal(topk, O.top_k_mask(edge["logits"], k))


@pytest.mark.parametrize("rt", ["mixtral", "st"])
def test_gate_nonfinite_rows(rt):
    edge = np.load(os.path.join(GOLDEN, "routing_edge.npz"))
    for row, ref in zip(edge["nonfinite_logits"], edge[f"nonfinite_{rt}_gates"]):
        g, _, err = _gate_dev(row[None, :], 2, rt)
        if (ref == -1).all():
            assert err == 1
        else:
            assert err == 0 and bits_equal(g[0], ref)


def test_exp_exhaustive_slice_on_device():
    """The device exp reproduces numpy's f32 exp: drive it through mixtral k=2
    rows [0, d] whose second gate is e/(1+e) with e = exp(d), d in [-104, 0]."""
    rng = np.random.default_rng(3)
    d = np.concatenate([-rng.uniform(0, 104, 200_000), -np.linspace(0, 104, 100_000)]).astype(np.float32)
    h = np.zeros((d.size, 2), dtype=np.float32)
    h[:, 1] = d
    g, _, _ = _gate_dev(h, 2, "mixtral")
    ref = O.gate(h, 2, "mixtral").gates
    assert bits_equal(g, ref)


# --------------------------------------------------------------------------
# router forward + dispatch on config 1 vs the oracle
# --------------------------------------------------------------------------

@pytest.mark.parametrize("rt", ["mixtral", "st"])
def test_router_fwd_cfg1(rt):
    x = O.rng(123, 0).standard_normal((2048, 256)).astype(np.float32)
    wg, wn = O.router_weights(256, 8, 0, 1, np.float32)
    xd = torch.from_numpy(x).cuda().to(torch.bfloat16)
    p = B.RouterParams(w_g=torch.from_numpy(wg).cuda(), w_noise=torch.from_numpy(wn).cuda())
    h = B.router_logits(xd, p, noise_enabled=False).cpu().numpy()
    # values: fp32 logits of the bf16-rounded input
    xr = xd.float().cpu().numpy()
    href = xr @ wg
    assert np.max(np.abs(h - href)) < 1e-4 * max(1.0, np.abs(href).max())
    # routing from the device logits is bit-exact
    g = B.gate_mixtral(torch.from_numpy(h).cuda(), 2) if rt == "mixtral" else B.gate_st(torch.from_numpy(h).cuda(), 2)
    assert bits_equal(g.cpu().numpy(), O.gate(h, 2, rt).gates)


@pytest.mark.parametrize("rt", ["mixtral", "st"])
@pytest.mark.parametrize("cf", [0.5, 1.0, 2.0, None])
@pytest.mark.parametrize("pol", ["position", "score"])
def test_dispatch_cfg1_bit_exact(rt, cf, pol):
    cfg1 = np.load(os.path.join(GOLDEN, "routing_cfg1.npz"))
    g = cfg1[f"{rt}_gates"]
    cap = O.expert_capacity(2048, 8, cf)
    res = B.dispatch(torch.from_numpy(g).cuda(), cap, pol)
    ref = O.dispatch(g, cap, pol)
    assert np.array_equal(res.kept.cpu().numpy(), ref.kept)
    assert np.array_equal(res.dropped.cpu().numpy(), ref.dropped)
    assert np.array_equal(res.stats.assigned, ref.assigned)
    assert (res.stats.dropped, res.stats.total_slots) == (ref.n_dropped, ref.total_slots)
    assert np.allclose(res.stats.gate_mass, ref.gate_mass, rtol=1e-5)
    assert np.array_equal(res.slot_rank.cpu().numpy(), ref.rows())


def test_dispatch_prefix_rule_and_score_ties():
    g = O.gate(np.array([[0, 2, 1], [0, 1, 2]], dtype=np.float32), 2, "mixtral").gates
    res = B.dispatch(torch.from_numpy(g).cuda(), 1, "position")
    assert res.kept.cpu().numpy().tolist() == O.dispatch(g, 1, "position").kept.tolist()
    gates = np.zeros((3, 1), dtype=np.float32)
    gates[:, 0] = 0.5
    res = B.dispatch(torch.from_numpy(gates).cuda(), 2, "score")
    assert res.kept[:, 0].cpu().tolist() == [True, True, False]
    gates = np.zeros((3, 2), dtype=np.float32)
    gates[:, 0] = [0.9, 0.5, 0.7]
    assert B.dispatch(torch.from_numpy(gates).cuda(), 2, "score").kept[:, 0].cpu().tolist() == [True, False, True]


@pytest.mark.parametrize("T", [1, 5, 8192, 8193, 20000])   # one-chunk single-scan path up to 8192
@pytest.mark.parametrize("pol", ["position", "score"])
def test_dispatch_random_sizes(T, pol):
    rng = np.random.default_rng(T)
    h = (rng.standard_normal((T, 8)) * 1.3).astype(np.float32)
    g = O.gate(h, 2, "mixtral").gates
    for cf in (0.3, 1.0, None):
        cap = O.expert_capacity(T, 8, cf)
        res = B.dispatch(torch.from_numpy(g).cuda(), cap, pol)
        ref = O.dispatch(g, cap, pol)
        assert np.array_equal(res.kept.cpu().numpy(), ref.kept), cf
        assert np.array_equal(res.slot_rank.cpu().numpy(), ref.rows()), cf


# --------------------------------------------------------------------------
# upcycling: bitwise against the reference copy after the dtype cast
# --------------------------------------------------------------------------

def test_upcycle_copy_bitwise():
    schema = O.dense_schema(32, 256, 1, 128, 512)
    dense = O.init_dense(schema, seed=7, dtype=np.float32)
    w1, w2, w3 = (torch.from_numpy(dense[f"layers.0.ffn.{w}"]).cuda() for w in ("w1", "w2", "w3"))
    from paper_2412_09952_b200.upcycle import upcycle_experts
    W1, W2, W3 = upcycle_experts(w1, w2, w3, 8)
    for e in range(8):
        assert torch.equal(W1[e].t(), w1.to(torch.bfloat16))
        assert torch.equal(W2[e].t(), w2.to(torch.bfloat16))
        assert torch.equal(W3[e].t(), w3.to(torch.bfloat16))
    W1b, _, _ = upcycle_experts(w1.to(torch.bfloat16), w2.to(torch.bfloat16), w3.to(torch.bfloat16), 3)
    assert torch.equal(W1b[2].t(), w1.to(torch.bfloat16))


@pytest.mark.parametrize("E,noise", [(4, False), (8, False), (8, True), (16, True), (6, True)])
def test_router_fwd_tensor_core_matches_fp64_and_cuda_core_path(E, noise):
    """K1 on tcgen05 (x . W with W split into three bf16 parts, fp32
    accumulation) against an fp64 reference of x . W (+ z softplus(x . W_n))
    and against the CUDA-core K1: logits agree to fp32 accumulation slack
    (|dh| <= 2e-6 * sum |x w| + 1e-7), and the gates each path produces from its
    own logits are the oracle's gates for those logits (bit-exact)."""
    T, H = 1000, 1024
    g = O.rng(60, E)
    x = torch.from_numpy(g.standard_normal((T, H)).astype(np.float32)).cuda().to(torch.bfloat16)
    wg = torch.from_numpy((g.standard_normal((H, E)) * 0.05).astype(np.float32)).cuda()
    wn = torch.from_numpy((g.standard_normal((H, E)) * 0.05).astype(np.float32)).cuda()
    z = torch.from_numpy(g.standard_normal((T, E)).astype(np.float32)).cuda() if noise else None
    out = {}
    for fma in (0, 1):
        _lib.call("b200moe_router_set_fma", fma)
        try:
            logits = torch.empty(T, E, device="cuda")
            gates = torch.empty(T, E, device="cuda")
            na = torch.empty(T, E, device="cuda") if noise else None
            ws = B.moe._router_ws(H, E, torch.device("cuda"))
            _lib.call("b200moe_router_fwd", x.data_ptr(), wg.data_ptr(), wn.data_ptr(), _lib.ptr(z), T, H, E, 2, 0,
                      logits.data_ptr(), gates.data_ptr(), None, _lib.ptr(na), ws.data_ptr(), None, _lib.stream_ptr())
            torch.cuda.synchronize()
        finally:
            _lib.call("b200moe_router_set_fma", 0)
        out[fma] = (logits.cpu().numpy(), gates.cpu().numpy())
    xd = x.double().cpu().numpy()
    wgd, wnd = wg.double().cpu().numpy(), wn.double().cpu().numpy()
    ref = xd @ wgd
    slack = np.abs(xd) @ np.abs(wgd)
    if noise:
        an = xd @ wnd
        zd = z.double().cpu().numpy()
        ref = ref + zd * (np.maximum(an, 0) + np.log1p(np.exp(-np.abs(an))))
        slack = slack + np.abs(zd) * (np.abs(xd) @ np.abs(wnd) + 1.0)
    for fma in (0, 1):
        h, gts = out[fma]
        assert np.all(np.abs(h - ref) <= 2e-6 * slack + 1e-7), (fma, np.abs(h - ref).max())
        assert gts.tobytes() == O.gate(h, 2, "mixtral").gates.tobytes()
