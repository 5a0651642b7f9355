"""Pin the CPU oracle (oracle/moe_oracle.py) against golden vectors produced by
the reference itself (tests/golden/make_golden.py) and against the reference's
own known-answer tests (moefold pkg/tests/test_moe.py, test_tensor.py)."""

import hashlib
import json
import math
import os

import numpy as np
import pytest

from oracle import moe_oracle as O
from tests.conftest import GOLDEN

CFS = (0.5, 1.0, 2.0, None)


def cf_key(cf):
    return "none" if cf is None else str(cf).replace(".", "p")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def bits_equal(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and a.tobytes() == b.tobytes()


@pytest.fixture(scope="module")
def cfg1():
    return np.load(os.path.join(GOLDEN, "routing_cfg1.npz"))


# --------------------------------------------------------------------------
# numpy float32 exp port (device exp is ported from the same algorithm)
# --------------------------------------------------------------------------

def test_exp_port_matches_numpy_on_this_host():
    rng = np.random.default_rng(5)
    x = np.concatenate([rng.uniform(-110, 90, 300_000), rng.uniform(-104, 0, 300_000),
                        [0.0, -0.0, -103.97208404541015625, -103.9720764, 88.72283935546875]]).astype(np.float32)
    with np.errstate(over="ignore"):
        ref = np.exp(x)
    assert bits_equal(O.exp_port(x), ref)


# --------------------------------------------------------------------------
# routing vs the reference's config-1 goldens
# --------------------------------------------------------------------------

@pytest.mark.parametrize("rt", ["mixtral", "st"])
def test_cfg1_gates_bit_exact(cfg1, rt):
    h = cfg1["logits"]
    for impl in ("numpy", "port"):
        g = O.gate(h, 2, rt, exp_impl=impl).gates
        assert bits_equal(g, cfg1[f"{rt}_gates"]), impl


@pytest.mark.parametrize("rt", ["mixtral", "st"])
@pytest.mark.parametrize("cf", CFS)
@pytest.mark.parametrize("pol", ["position", "score"])
def test_cfg1_dispatch_bit_exact(cfg1, rt, cf, pol):
    g = cfg1[f"{rt}_gates"]
    cap = O.expert_capacity(2048, 8, cf)
    d = O.dispatch(g, cap, pol)
    k = f"{rt}_{cf_key(cf)}_{pol}"
    assert np.array_equal(np.packbits(d.kept), cfg1[k + "_kept"])
    assert np.array_equal(np.packbits(d.dropped), cfg1[k + "_dropped"])
    assert np.array_equal(d.assigned, cfg1[k + "_assigned"])
    assert bits_equal(d.gate_mass, cfg1[k + "_gate_mass"])
    st = cfg1[k + "_stats"]
    assert (d.n_dropped, d.total_slots, -1 if cap is None else cap) == tuple(st)


def test_cfg1_inputs_regenerate_bitwise(cfg1):
    """Dense init + router init restated from seeds reproduce the reference bits."""
    dig = json.load(open(os.path.join(GOLDEN, "upcycle.json")))["digests"]
    schema = O.dense_schema(32, 256, 1, 2 * 64, 512)
    dense = O.init_dense(schema, seed=7, dtype=np.float32)
    for w in ("w1", "w2", "w3"):
        assert sha(dense[f"layers.0.ffn.{w}"]) == dig["cfg1_f32_ffn"][w]
    wg, wn = O.router_weights(256, 8, 0, 1, np.float32)
    assert sha(wg) == dig["cfg1_f32_router_wg"] and sha(wn) == dig["cfg1_f32_router_wn"]
    assert bits_equal(wg, cfg1["wg"])
    x = O.rng(123, 0).standard_normal((2048, 256)).astype(np.float32)
    assert bits_equal(x @ wg, cfg1["logits"])


# --------------------------------------------------------------------------
# edge-case routing rows
# --------------------------------------------------------------------------

@pytest.fixture(scope="module")
def edge():
    return np.load(os.path.join(GOLDEN, "routing_edge.npz"))


@pytest.mark.parametrize("rt", ["mixtral", "st"])
@pytest.mark.parametrize("k", [1, 2, 3, 4, 8])
def test_edge_gates_bit_exact(edge, rt, k):
    with np.errstate(over="ignore", invalid="ignore"):
        for impl in ("numpy", "port"):
            g = O.gate(edge["logits"], k, rt, exp_impl=impl).gates
            assert bits_equal(g, edge[f"{rt}_k{k}_gates"]), impl


@pytest.mark.parametrize("rt", ["mixtral", "st"])
def test_edge_nonfinite_rows(edge, rt):
    for row, ref in zip(edge["nonfinite_logits"], edge[f"nonfinite_{rt}_gates"]):
        if (ref == -1).all():
            with pytest.raises(O.OracleGateError):
                O.gate(row[None, :], 2, rt)
        else:
            with np.errstate(invalid="ignore"):
                assert bits_equal(O.gate(row[None, :], 2, rt).gates[0], ref)


def test_prefix_capacity_example(edge):
    g = O.gate(np.array([[0, 2, 1], [0, 1, 2]], dtype=np.float32), 2, "mixtral").gates
    assert bits_equal(g, edge["prefix_example_gates"])
    d = O.dispatch(g, 1, "position")
    assert np.array_equal(d.kept, edge["prefix_example_kept"])
    assert not d.kept[1].any()   # token 1 fully dropped by token 0's 2nd choice


# --------------------------------------------------------------------------
# full layer fwd+bwd vs the reference autograd
# --------------------------------------------------------------------------

def _small_inputs(T, H, F, E, dt):
    g = O.rng(10, 0)
    wg = (g.standard_normal((H, E)) * 0.5).astype(dt)
    wn = (g.standard_normal((H, E)) * 0.1).astype(dt)
    w1, w2, w3 = [], [], []
    for _ in range(E):
        w1.append((g.standard_normal((H, F)) * 0.3).astype(dt))
        w2.append((g.standard_normal((F, H)) * 0.3).astype(dt))
        w3.append((g.standard_normal((H, F)) * 0.3).astype(dt))
    x = O.rng(11, 0).standard_normal((T, H)).astype(dt)
    dy = O.rng(12, 0).standard_normal((T, H)).astype(dt)
    z = O.rng(13, 0).standard_normal((T, E))
    return wg, wn, w1, w2, w3, x, dy, z


def _rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-30))


@pytest.fixture(scope="module")
def small():
    return np.load(os.path.join(GOLDEN, "layer_small.npz"))


def _small_cases():
    out = []
    for dt in ("f32", "f64"):
        for rt in ("mixtral", "st"):
            for pol in ("position", "score"):
                for cf in CFS:
                    for noise in (False, True):
                        if dt == "f64" and (cf != 1.0 or pol != "position"):
                            continue
                        out.append((dt, rt, pol, cf, noise))
    return out


@pytest.mark.parametrize("dt,rt,pol,cf,noise", _small_cases())
def test_small_layer_fwd_bwd(small, dt, rt, pol, cf, noise):
    T, H, F, E = (int(v) for v in small["shape"])
    lam = float(small["lam"])
    dtype = np.float32 if dt == "f32" else np.float64
    wg, wn, w1, w2, w3, x, dy, z = _small_inputs(T, H, F, E, dtype)
    key = f"{dt}_{rt}_{pol}_{cf_key(cf)}_{'noise' if noise else 'clean'}"
    cfg = O.LayerCfg(n_experts=E, top_k=2, router_type=rt, noise=noise, capacity_factor=cf, drop_policy=pol)
    y, gates, cache = O.moe_forward(x, wg, wn, w1, w2, w3, cfg, z=z if noise else None)
    assert bits_equal(gates, small[key + "_gates"])
    assert np.array_equal(cache.disp.assigned, small[key + "_assigned"])
    assert cache.disp.n_dropped == int(small[key + "_dropped"])
    tol_y = 1e-6 if dt == "f32" else 1e-13
    tol_g = 1e-5 if dt == "f32" else 1e-11
    assert _rel(y, small[key + "_y"]) <= tol_y
    _, dimp = O.importance_penalty(gates)
    gr = O.moe_backward(cache, dy, dgates=lam * dimp)
    assert _rel(gr["dx"], small[key + "_dx"]) <= tol_g
    assert _rel(gr["dwg"], small[key + "_dwg"]) <= tol_g
    assert _rel(gr["dwn"], small[key + "_dwn"]) <= tol_g if noise else np.all(small[key + "_dwn"] == 0)
    for w in ("w1", "w2", "w3"):
        assert _rel(np.stack(gr["d" + w]), small[key + f"_d{w}"]) <= tol_g, w


@pytest.mark.parametrize("rt", ["mixtral", "st"])
def test_cfg1_layer_summaries(rt):
    ref = np.load(os.path.join(GOLDEN, "layer_cfg1.npz"))
    schema = O.dense_schema(32, 256, 1, 128, 512)
    dense = O.init_dense(schema, seed=7, dtype=np.float32)
    w1, w2, w3 = (dense[f"layers.0.ffn.{w}"] for w in ("w1", "w2", "w3"))
    wg, wn = O.router_weights(256, 8, 0, 1, np.float32)
    x = O.rng(123, 0).standard_normal((2048, 256)).astype(np.float32)
    dy = O.rng(124, 0).standard_normal((2048, 256)).astype(np.float32)
    cfg = O.LayerCfg(router_type=rt, capacity_factor=1.0)
    y, gates, cache = O.moe_forward(x, wg, wn, [w1] * 8, [w2] * 8, [w3] * 8, cfg)
    assert np.array_equal(cache.disp.assigned, ref[f"{rt}_assigned"])
    assert np.allclose(np.linalg.norm(y.astype(np.float64), axis=1), ref[f"{rt}_y_rownorm"], rtol=1e-5, atol=1e-7)
    _, dimp = O.importance_penalty(gates)
    gr = O.moe_backward(cache, dy, dgates=0.01 * dimp)
    assert np.allclose(np.linalg.norm(gr["dx"].astype(np.float64), axis=1), ref[f"{rt}_dx_rownorm"], rtol=1e-4)
    assert _rel(gr["dwg"], ref[f"{rt}_dwg"]) < 1e-5
    for w in ("w1", "w2", "w3"):
        n = np.array([np.linalg.norm(d.astype(np.float64)) for d in gr["d" + w]])
        assert np.allclose(n, ref[f"{rt}_d{w}_norm"], rtol=1e-4), w


# --------------------------------------------------------------------------
# known-answer tests restated from the reference suite (pkg/tests/test_moe.py)
# --------------------------------------------------------------------------

def test_known_answers():
    assert O.top_k_mask(np.array([1.0, 3.0, 2.0, 0.0]), 2).tolist() == [False, True, True, False]
    assert O.top_k_mask(np.array([5.0, 5.0, 5.0, 5.0]), 2).tolist() == [True, True, False, False]
    for k in (0, 5):
        with pytest.raises(O.OracleConfigError):
            O.top_k_mask(np.zeros(4), k)
    g = O.gate(np.array([[1.0, 3.0, 2.0, 0.0]]), 2, "mixtral").gates
    assert g[0, 1] == pytest.approx(math.e / (math.e + 1), abs=1e-12)
    assert g[0, 2] == pytest.approx(1 / (math.e + 1), abs=1e-12)
    g = O.gate(np.zeros((1, 8)), 2, "st").gates
    assert np.allclose(g[0, :2], 0.125) and g.sum() == pytest.approx(0.25)
    assert O.expert_capacity(64, 8, 2) == 16
    assert O.expert_capacity(100, 8, 1) == 13
    assert O.expert_capacity(64, 8, None) is None
    assert O.expert_capacity(10, 7, 0.7) == 1
    gates = np.zeros((6, 2)); gates[:, 0] = 0.9; gates[:, 1] = 0.1
    assert O.dispatch(gates, 3, "position").kept[:, 0].tolist() == [True] * 3 + [False] * 3
    gates = np.zeros((3, 2)); gates[:, 0] = [0.9, 0.5, 0.7]
    assert O.dispatch(gates, 2, "score").kept[:, 0].tolist() == [True, False, True]
    gates = np.zeros((3, 1)); gates[:, 0] = 0.5
    assert O.dispatch(gates, 2, "score").kept[:, 0].tolist() == [True, True, False]
    loss, dimp = O.importance_penalty(np.full((6, 4), 0.25))
    assert loss == pytest.approx(0.0, abs=1e-15) and np.allclose(dimp, 0)


def test_identical_experts_mixtral_dropless_equals_dense():
    g = O.rng(6, 0)
    H, F, E, T = 8, 16, 4, 10
    w1, w2, w3 = (g.standard_normal(s) * 0.3 for s in ((H, F), (F, H), (H, F)))
    wg = g.standard_normal((H, E)) * 0.5
    x = g.standard_normal((T, H))
    y, _, cache = O.moe_forward(x, wg, np.zeros_like(wg), [w1] * E, [w2] * E, [w3] * E, O.LayerCfg(n_experts=E))
    a = x @ w1
    dense = ((a * O.sigmoid(a)) * (x @ w3)) @ w2
    assert np.max(np.abs(y - dense) / np.maximum(np.abs(dense), 1e-30)) <= 1e-12
    assert cache.disp.n_dropped == 0


@pytest.mark.parametrize("rt,pol,cf,noise", [("mixtral", "position", 1.0, True), ("st", "score", 2.0, False),
                                             ("mixtral", "score", None, True)])
def test_sampled_oracle_pieces_equal_full_oracle(rt, pol, cf, noise):
    """The row / column pieces the bench-shape GPU test uses (expert_rows,
    expert_wgrad_columns, router_bwd_rows) reproduce the pinned full oracle
    (moe_forward / moe_backward) on the rows and columns they cover."""
    T, H, F, E, k = 96, 16, 24, 8, 2
    g = O.rng(77, 1)
    wg = (g.standard_normal((H, E)) * 0.5).astype(np.float64)
    wn = (g.standard_normal((H, E)) * 0.2).astype(np.float64)
    w1 = [g.standard_normal((H, F)) * 0.3 for _ in range(E)]
    w2 = [g.standard_normal((F, H)) * 0.3 for _ in range(E)]
    w3 = [g.standard_normal((H, F)) * 0.3 for _ in range(E)]
    x = g.standard_normal((T, H))
    dy = g.standard_normal((T, H))
    z = g.standard_normal((T, E))
    cfg = O.LayerCfg(n_experts=E, top_k=k, router_type=rt, noise=noise, capacity_factor=cf, drop_policy=pol)
    y, gates, cache = O.moe_forward(x, wg, wn, w1, w2, w3, cfg, z=z if noise else None)
    _, dimp = O.importance_penalty(gates)
    gr = O.moe_backward(cache, dy, dgates=0.3 * dimp)
    kept = cache.disp.kept
    idx = np.arange(0, T, 3)
    y_s = np.zeros((idx.size, H))
    dx_s = np.zeros((idx.size, H))
    dg = np.zeros((idx.size, E))
    cols = np.array([0, 5, 11, 23])
    for e in range(E):
        rows = np.flatnonzero(kept[idx, e])
        if rows.size:
            yc, dgc, dxc = O.expert_rows(x[idx[rows]], dy[idx[rows]], gates[idx[rows], e], w1[e], w2[e], w3[e])
            y_s[rows] += yc
            dg[rows, e] = dgc
            dx_s[rows] += dxc
        allr = np.flatnonzero(kept[:, e])
        if allr.size:
            d1, d3, d2 = O.expert_wgrad_columns(x[allr], dy[allr], gates[allr, e], w1[e][:, cols], w3[e][:, cols],
                                                w2[e][cols, :])
            np.testing.assert_allclose(d1, gr["dw1"][e][:, cols], rtol=1e-10, atol=1e-12)
            np.testing.assert_allclose(d3, gr["dw3"][e][:, cols], rtol=1e-10, atol=1e-12)
            np.testing.assert_allclose(d2, gr["dw2"][e][cols, :], rtol=1e-10, atol=1e-12)
    dh, dxr, dn = O.router_bwd_rows(cache.logits[idx], k, rt, dg + 0.3 * dimp[None, :], x[idx], wg, wn,
                                    z[idx] if noise else None, cache.an[idx] if noise else None)
    np.testing.assert_allclose(y_s, y[idx], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(dh, gr["dh"][idx], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(dx_s + dxr, gr["dx"][idx], rtol=1e-10, atol=1e-12)
