"""CPU tests for SURVEY 8(f) row 3 (checkpoint format): the CRC32C / layout
oracle pinned against the reference's own files, and the manifest checks of
the loader that run before any GPU work."""

import json
import os

import numpy as np
import pytest
import torch

from oracle import checkpoint_oracle as CO
from tests.conftest import GOLDEN

CK = json.load(open(os.path.join(GOLDEN, "ckpt.json")))


def test_crc_oracle_known_values():
    k = CK["crc_known"]
    assert CO.crc32c(b"123456789") == k["123456789"] == 0xE3069283
    assert CO.crc32c(b"") == k["empty"] == 0
    assert CO.crc32c(bytes(range(256))) == k["bytes_0_255"]
    assert CO.crc32c(b"\x00" * 1000) == k["zeros_1000"]
    r = np.random.default_rng(1).integers(0, 256, 5000, dtype=np.uint8).tobytes()
    assert CO.crc32c(r) == CO.crc32c_py(r)


@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_layout_oracle_reproduces_reference_dense_files(dt):
    import hashlib
    import paper_2412_09952_b200 as P
    cfg = P.ModelConfig(**CK["tiny"])
    d = P.init_dense(cfg, seed=7, dtype=torch.float32 if dt == "f32" else torch.float64, device="cpu")
    records, blob = CO.layout({k: v.numpy() for k, v in d.tensors.items()})
    ref = json.loads(CK["cases"][f"dense_{dt}"]["manifest"])
    assert records == ref["tensors"]
    assert hashlib.sha256(blob).hexdigest() == CK["cases"][f"dense_{dt}"]["weights_sha256"]


def _write(tmp_path, manifest, payload=b"\x00" * 64):
    (tmp_path / "manifest.json").write_text(json.dumps(manifest))
    (tmp_path / "weights.bin").write_bytes(payload)


def _manifest(**over):
    m = json.loads(CK["cases"]["dense_f32"]["manifest"])
    m.update(over)
    return m


def test_loader_manifest_errors(tmp_path):
    from paper_2412_09952_b200 import checkpoint as C
    from paper_2412_09952_b200.errors import ManifestError, TruncatedFileError, UnknownVersionError
    _write(tmp_path, _manifest(format_version=2))
    with pytest.raises(UnknownVersionError):
        C._read_manifest(str(tmp_path))
    (tmp_path / "manifest.json").write_text("{not json")
    with pytest.raises(ManifestError):
        C._read_manifest(str(tmp_path))
    rec = {"name": "a", "dtype": "f32", "shape": [4], "offset": 0, "length": 16, "crc32c": 0}
    for bad, exc in ((dict(rec, dtype="f16"), ManifestError), (dict(rec, length=12), ManifestError),
                     (dict(rec, offset=60), TruncatedFileError)):
        _write(tmp_path, _manifest(tensors=[bad]))
        with pytest.raises(exc):
            C._check_records(str(tmp_path), C._read_manifest(str(tmp_path)))
    _write(tmp_path, _manifest(tensors=[rec, rec]))
    with pytest.raises(ManifestError):
        C._check_records(str(tmp_path), C._read_manifest(str(tmp_path)))


def test_crc_shift_matrix_combines_like_zlib():
    from paper_2412_09952_b200.checkpoint import _shift_matrix
    a, b = b"hello, ", b"checkpoint world"
    m, apply = _shift_matrix(len(b))
    assert apply(m, CO.crc32c(a)) ^ CO.crc32c(b) == CO.crc32c(a + b)
