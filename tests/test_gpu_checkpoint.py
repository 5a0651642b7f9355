"""GPU parity for SURVEY 8(f) row 3: the CRC32C kernel against the oracle, and
checkpoints written by the B200 build byte-identical to the reference's files
(manifest text and weights.bin digest), round-tripping through load."""

import hashlib
import json
import os

import numpy as np
import pytest
import torch

from oracle import checkpoint_oracle as CO
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu

CK = json.load(open(os.path.join(GOLDEN, "ckpt.json")))


@pytest.mark.parametrize("n", [0, 1, 3, 4, 15, 16, 17, 63, 64, 65, 1000, 16383, 16384, 16385, 16400, 65536 * 3 + 5,
                               1_000_003, 40_000_017])
def test_crc32c_kernel_matches_oracle(n):
    from paper_2412_09952_b200.checkpoint import crc32c
    data = np.random.default_rng(n).integers(0, 256, n, dtype=np.uint8)
    assert crc32c(data) == CO.crc32c(data.tobytes())


def test_crc32c_known_values_and_chaining():
    from paper_2412_09952_b200.checkpoint import crc32c
    k = CK["crc_known"]
    assert crc32c(b"123456789") == k["123456789"] == 0xE3069283
    assert crc32c(b"") == 0
    assert crc32c(bytes(range(256))) == k["bytes_0_255"]
    assert crc32c(b"\x00" * 1000) == k["zeros_1000"]
    assert crc32c(b"56789", crc32c(b"1234")) == 0xE3069283
    t = torch.randn(1 << 20, device="cuda")     # device tensors are checksummed in place
    assert crc32c(t) == CO.crc32c(t.cpu().numpy().tobytes())


def _dir_case(path, shard=False):
    out = {"manifest": open(os.path.join(path, "manifest.json")).read(),
           "weights_sha256": hashlib.sha256(open(os.path.join(path, "weights.bin"), "rb").read()).hexdigest()}
    if shard:
        out["shard"] = open(os.path.join(path, "shard.json")).read()
    return out


def _rounded_dense():
    import paper_2412_09952_b200 as P
    d = P.init_dense(P.ModelConfig(**CK["tiny"]), seed=7)
    for name, t in d.tensors.items():
        if ".ffn.w" in name:
            t.copy_(t.to(torch.bfloat16).float())
    return d


@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_dense_checkpoint_bytes_match_reference(tmp_path, dt):
    import paper_2412_09952_b200 as P
    from paper_2412_09952_b200.checkpoint import load_checkpoint, save_checkpoint
    d = P.init_dense(P.ModelConfig(**CK["tiny"]), seed=7, dtype=torch.float32 if dt == "f32" else torch.float64)
    save_checkpoint(d, str(tmp_path / "a"))
    assert _dir_case(tmp_path / "a") == CK["cases"][f"dense_{dt}"]
    back = load_checkpoint(str(tmp_path / "a"))
    assert P.verify_equivalence(d, back).equal
    save_checkpoint(back, str(tmp_path / "b"))
    assert _dir_case(tmp_path / "b") == CK["cases"][f"dense_{dt}"]


def test_moe_checkpoint_bytes_match_reference_and_round_trip(tmp_path):
    import paper_2412_09952_b200 as P
    from paper_2412_09952_b200.checkpoint import load_checkpoint, save_checkpoint
    u = CK["upcycle"]
    moe = P.upcycle_full(_rounded_dense(), u["n_experts"], u["top_k"], moe_layers=tuple(u["moe_layers"]),
                         router_seed=u["router_seed"], capacity_factor=u["capacity_factor"])
    save_checkpoint(moe, str(tmp_path / "m"))
    assert _dir_case(tmp_path / "m") == CK["cases"]["moe"]
    back = load_checkpoint(str(tmp_path / "m"))
    assert P.verify_equivalence(moe, back).equal
    for a, b in zip(moe.stacked[1], back.stacked[1]):       # kernel-layout stacks rebuilt bit-exactly
        assert torch.equal(a, b)
    x = torch.randn(64, CK["tiny"]["hidden"], device="cuda")
    y0 = P.moe_forward(x, moe.layer(1), moe.gate).output
    y1 = P.moe_forward(x, back.layer(1), back.gate).output
    assert torch.equal(y0, y1)


@pytest.mark.parametrize("case,dt", [("moe_f64", torch.float64), ("moe_f32_raw", torch.float32)])
def test_full_precision_moe_checkpoint_bytes_and_round_trip(tmp_path, case, dt):
    """Experts the bf16 stacks cannot hold exactly (f64, unrounded f32): the
    checkpoint keeps full-precision expert copies and a router in the source
    dtype, like the reference (upcycle.py:104-112), so the files match its bytes;
    load -> save reproduces them (the stacks are separate bf16 compute copies)."""
    import paper_2412_09952_b200 as P
    from paper_2412_09952_b200.checkpoint import load_checkpoint, save_checkpoint
    u = CK["upcycle"]
    dense = P.init_dense(P.ModelConfig(**CK["tiny"]), seed=7, dtype=dt)
    moe = P.upcycle_full(dense, u["n_experts"], u["top_k"], moe_layers=tuple(u["moe_layers"]),
                         router_seed=u["router_seed"], capacity_factor=u["capacity_factor"])
    assert moe.tensors["layers.1.moe.router.wg"].dtype == dt
    save_checkpoint(moe, str(tmp_path / "m"))
    assert _dir_case(tmp_path / "m") == CK["cases"][case]
    with pytest.warns(RuntimeWarning, match="bf16"):
        back = load_checkpoint(str(tmp_path / "m"))
    assert P.verify_equivalence(moe, back).equal
    save_checkpoint(back, str(tmp_path / "b"))
    assert _dir_case(tmp_path / "b") == CK["cases"][case]
    x = torch.randn(64, CK["tiny"]["hidden"], device="cuda")
    assert torch.equal(P.moe_forward(x, moe.layer(1), moe.gate).output,
                       P.moe_forward(x, back.layer(1), back.gate).output)


def test_shards_bytes_match_reference_and_gather(tmp_path):
    import paper_2412_09952_b200 as P
    from paper_2412_09952_b200.checkpoint import load_shard, save_shard
    u = CK["upcycle"]
    dense = _rounded_dense()
    loaded = []
    for s in P.shard_dense(dense, 2, 2):
        ms = P.upcycle_shard(s, u["n_experts"], u["top_k"], moe_layers=tuple(u["moe_layers"]),
                             router_seed=u["router_seed"], capacity_factor=u["capacity_factor"])
        p = tmp_path / f"s{s.rank}"
        save_shard(ms, str(p))
        assert _dir_case(p, shard=True) == CK["cases"][f"moe_shard_r{s.rank}"]
        loaded.append(load_shard(str(p)))
    full = P.upcycle_full(dense, u["n_experts"], u["top_k"], moe_layers=tuple(u["moe_layers"]),
                          router_seed=u["router_seed"], capacity_factor=u["capacity_factor"])
    assert P.verify_equivalence(P.gather_moe(loaded), full).equal
    plain = P.init_dense(P.ModelConfig(**CK["tiny"]), seed=7)
    for s in P.shard_dense(plain, 2, 2):
        p = tmp_path / f"d{s.rank}"
        save_shard(s, str(p))
        assert _dir_case(p, shard=True) == CK["cases"][f"dense_shard_r{s.rank}"]


def test_corrupted_payload_raises_checksum_error(tmp_path):
    import paper_2412_09952_b200 as P
    from paper_2412_09952_b200.checkpoint import load_checkpoint, save_checkpoint
    from paper_2412_09952_b200.errors import ChecksumError
    d = P.init_dense(P.ModelConfig(**CK["tiny"]), seed=7)
    save_checkpoint(d, str(tmp_path / "a"))
    man = json.loads((tmp_path / "a" / "manifest.json").read_text())
    rec = next(r for r in man["tensors"] if r["name"] == "layers.1.attn.wk")
    raw = bytearray((tmp_path / "a" / "weights.bin").read_bytes())
    raw[rec["offset"] + 5] ^= 0x10
    (tmp_path / "a" / "weights.bin").write_bytes(bytes(raw))
    with pytest.raises(ChecksumError, match="layers.1.attn.wk"):
        load_checkpoint(str(tmp_path / "a"))
    assert load_checkpoint(str(tmp_path / "a"), verify=False) is not None


# --------------------------------------------------------------------------
# gather_moe integrity errors (reference tests/test_upcycle.py:152-168,
# behaviour upcycle.py:240-254, 273-283)
# --------------------------------------------------------------------------

def _tiny_shards(tp, ep):
    import paper_2412_09952_b200 as P
    dense = P.init_dense(P.ModelConfig(**CK["tiny"]), seed=7)
    return [P.upcycle_shard(s, 4, 2, router_seed=5) for s in P.shard_dense(dense, tp, ep)]


def test_gather_missing_tile_names_rank():
    import paper_2412_09952_b200 as P
    from paper_2412_09952_b200.errors import IntegrityError
    shards = _tiny_shards(2, 2)
    with pytest.raises(IntegrityError, match="rank 2"):
        P.gather_moe([s for s in shards if s.rank != 2])


def test_gather_replica_mismatch():
    import paper_2412_09952_b200 as P
    from paper_2412_09952_b200.errors import IntegrityError
    shards = _tiny_shards(1, 2)
    shards[1].tensors["layers.0.moe.router.wg"].data[0, 0] += 1.0
    with pytest.raises(IntegrityError, match="replica mismatch"):
        P.gather_moe(shards)


def test_gather_duplicate_rank():
    import paper_2412_09952_b200 as P
    from paper_2412_09952_b200.errors import IntegrityError
    shards = _tiny_shards(1, 2)
    with pytest.raises(IntegrityError, match="duplicate"):
        P.gather_moe([shards[0], shards[0]])


def test_gather_equals_full_bitwise_grid():
    """Reference test_upcycle.py:140-148 over tp {1,2} x ep {1,2,4}."""
    import paper_2412_09952_b200 as P
    dense = P.init_dense(P.ModelConfig(**CK["tiny"]), seed=7)
    full = P.upcycle_full(dense, n_experts=4, top_k=2, router_seed=5)
    for tp in (1, 2):
        for ep in (1, 2, 4):
            shards = [P.upcycle_shard(s, n_experts=4, top_k=2, router_seed=5) for s in P.shard_dense(dense, tp, ep)]
            rep = P.verify_equivalence(full, P.gather_moe(shards))
            assert rep.equal, (tp, ep, str(rep))
