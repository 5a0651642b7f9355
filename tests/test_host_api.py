"""CPU-side checks of the boundary: the C-ABI library loads and exports every
symbol include/b200moe.h declares; host-side validation mirrors the reference
(moefold/moe.py:45-55, 189-196, upcycle.py:62-69) and raises the same classes;
the product path refuses CPU tensors instead of falling back."""

import ctypes
import os
import re

import numpy as np
import pytest
import torch

import paper_2412_09952_b200 as B
from paper_2412_09952_b200 import _lib
from paper_2412_09952_b200.errors import ConfigError, ShapeError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "b200moe.h")).read()
    return sorted(set(re.findall(r"\b(b200moe_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    declared = header_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.exported_symbols())


def test_version_and_error_strings():
    lib = _lib.load()
    assert lib.b200moe_version() == 1
    assert isinstance(lib.b200moe_last_error(), bytes)


def test_argument_errors_map_to_reference_exceptions():
    # invalid arguments are rejected before any device work (no GPU needed)
    with pytest.raises(ConfigError):
        _lib.call("b200moe_dispatch", None, 4, 8, 1, 7, 0, 0, None, None, None, None, None, None, None, None, None,
                  None)
    with pytest.raises(ConfigError):
        _lib.call("b200moe_router_fwd", None, None, None, None, 4, 64, 8, 9, 0, None, None, None, None, None, None,
                  None)
    with pytest.raises(ShapeError):
        _lib.call("b200moe_router_fwd", None, None, None, None, 4, 63, 8, 2, 0, None, None, None, None, None, None,
                  None)
    with pytest.raises(ShapeError):
        _lib.call("b200moe_expert_fwd1", None, None, None, None, None, None, 8, 1024, 4000, 14336, 8, None, None,
                  None, None)
    with pytest.raises(ConfigError):
        _lib.call("b200moe_expert_fwd1", None, None, None, None, None, None, 0, 1024, 4096, 14336, 8, None, None,
                  None, None)


def test_gate_config_validation_matches_reference():
    B.GateConfig(n_experts=8, top_k=2)
    for kw in (dict(n_experts=0, top_k=1), dict(n_experts=4, top_k=5), dict(n_experts=4, top_k=0),
               dict(n_experts=4, top_k=2, router_type="switch"), dict(n_experts=4, top_k=2, capacity_factor=0.0),
               dict(n_experts=4, top_k=2, drop_policy="random")):
        with pytest.raises(ConfigError):
            B.GateConfig(**kw)


def test_expert_capacity_reference_examples():
    assert B.expert_capacity(64, 8, 2) == 16
    assert B.expert_capacity(100, 8, 1) == 13
    assert B.expert_capacity(64, 8, None) is None
    assert B.expert_capacity(10, 7, 0.7) == 1
    assert B.expert_capacity(8192, 8, 1.0) == 1024
    with pytest.raises(ConfigError):
        B.expert_capacity(0, 8, 1.0)


def test_router_params_validation():
    with pytest.raises(ShapeError):
        B.RouterParams(torch.zeros(4, 8), torch.zeros(4, 7))
    with pytest.raises(ConfigError):
        B.RouterParams(torch.full((4, 8), float("nan")), torch.zeros(4, 8))


def test_moe_layer_validation_and_views():
    W1, W2, W3 = torch.zeros(3, 32, 16), torch.zeros(3, 16, 32), torch.zeros(3, 32, 16)
    layer = B.MoELayer.from_stacked(B.RouterParams(torch.zeros(16, 3), torch.zeros(16, 3)), W1, W2, W3)
    assert tuple(layer.experts[1].w1.shape) == (16, 32) and tuple(layer.experts[1].w2.shape) == (32, 16)
    with pytest.raises(ConfigError):
        B.MoELayer(router=layer.router, experts=[])
    bad = [B.ExpertFFN(torch.zeros(16, 32), torch.zeros(32, 16), torch.zeros(16, 32)),
           B.ExpertFFN(torch.zeros(16, 8), torch.zeros(8, 16), torch.zeros(16, 8))]
    with pytest.raises(ShapeError):
        B.MoELayer(router=layer.router, experts=bad)


def test_moe_forward_validation_and_no_cpu_fallback():
    layer = B.MoELayer.from_stacked(B.RouterParams(torch.zeros(16, 4), torch.zeros(16, 4)),
                                    torch.zeros(4, 32, 16), torch.zeros(4, 16, 32), torch.zeros(4, 32, 16))
    with pytest.raises(ConfigError):
        B.moe_forward(torch.zeros(2, 16), layer, B.GateConfig(n_experts=8, top_k=2))
    with pytest.raises(ShapeError):
        B.moe_forward(torch.zeros(2, 15), layer, B.GateConfig(n_experts=4, top_k=2))
    with pytest.raises(RuntimeError, match="CUDA"):
        B.moe_forward(torch.zeros(2, 16), layer, B.GateConfig(n_experts=4, top_k=2))
    with pytest.raises(ConfigError):   # noise on without an rng (moe.py:146-147)
        B.moe._noise(2, 4, "cpu", True, None, None)


def test_rng_matches_numpy_philox():
    a = B.Rng(123, 4).standard_normal((3, 5))
    g = np.random.Generator(np.random.Philox(key=np.array([123, 4], dtype=np.uint64)))
    assert np.array_equal(a, g.standard_normal(size=(3, 5)))
    with pytest.raises(ValueError):
        B.Rng(-1)


def test_moe_schema_and_dense_schema():
    cfg = B.ModelConfig(vocab=32, hidden=16, layers=2, heads=2, kv_heads=1, ffn_hidden=32, seq_len=16)
    gate = B.GateConfig(n_experts=4, top_k=2)
    s = B.moe_schema(cfg, gate, (1,))
    assert "layers.0.ffn.w1" in s and "layers.1.ffn.w1" not in s
    assert s["layers.1.moe.experts.003.w2"] == (32, 16)
    assert s["layers.1.moe.router.wg"] == (16, 4)


def test_routing_stats_reference_constructor_and_properties():
    """RoutingStats keeps the reference dataclass constructor (moe.py:95-116);
    the device-backed variant the layer returns is a subclass of it."""
    import dataclasses
    from paper_2412_09952_b200 import RoutingStats
    from paper_2412_09952_b200.moe import DeviceRoutingStats
    s = RoutingStats(assigned=np.array([3, 1, 0, 0]), dropped=2, total_slots=6,
                     gate_mass=np.array([1.5, 0.5, 0.0, 0.0], np.float32), capacity=3)
    assert [f.name for f in dataclasses.fields(RoutingStats)] == ["assigned", "dropped", "total_slots", "gate_mass",
                                                                   "capacity"]
    assert s.drop_rate == 2 / 6
    assert abs(s.load_entropy - float(-(0.75 * np.log(0.75) + 0.25 * np.log(0.25)))) < 1e-15
    assert RoutingStats(np.zeros(4, np.int64), 0, 0, np.zeros(4), None).drop_rate == 0.0
    assert RoutingStats(np.zeros(4, np.int64), 0, 0, np.zeros(4), None).load_entropy == 0.0
    assert issubclass(DeviceRoutingStats, RoutingStats)
