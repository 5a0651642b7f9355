"""On-disk checkpoints in the reference format, drop-in for moefold/checkpoint.py
(SURVEY 8(f) row 3), so GPU-upcycled weights round-trip through the files the
reference reads and writes and can be checked with verify_equivalence.

A checkpoint is a directory with `manifest.json` (format_version, kind,
model / gate config, moe_layers and one record per tensor: name, dtype
f32|f64, shape, 64-byte-aligned offset, length, CRC32C of the payload;
records sorted by name) and `weights.bin` (little-endian payloads, zero
padding between records); shards add `shard.json` (rank, tp, ep).  Saving is
deterministic: the bytes equal the reference's for the same tensor values.

B200 specifics: payload checksums are computed on the GPU
(b200moe_crc32c, crc32c.cu) on device tensors -- before the device->host copy
on save and after the host->device copy on load -- instead of the reference's
pure-Python slicing-by-8 loop.  bf16 expert weights are written as f32 (an
exact widening; the format has no bf16) and loaded back into the stacked bf16
kernel layout with the K12 copy kernel.
"""

from __future__ import annotations

import json
import os
import warnings
from dataclasses import asdict

import numpy as np
import torch

from . import _lib
from .errors import (ChecksumError, ConfigError, ManifestError, TruncatedFileError, UnknownVersionError)
from .model import DenseCheckpoint, ModelConfig
from .moe import GateConfig
from .upcycle import EXPERT_DTYPE, DenseShard, MoECheckpoint, MoEShard, _bf16_exact

FORMAT_VERSION = 1
ALIGNMENT = 64

_DTYPES = {"f32": (torch.float32, "<f4", 4), "f64": (torch.float64, "<f8", 8)}
_TORCH_TO_NAME = {torch.float32: "f32", torch.float64: "f64", torch.bfloat16: "f32"}


# --------------------------------------------------------------------------
# CRC32C on the GPU
# --------------------------------------------------------------------------

_POLY = 0x82F63B78


def _shift_matrix(nbytes: int) -> list:
    """Columns of the GF(2) matrix that runs the CRC register over nbytes zeros."""
    def apply(m, c):
        r = 0
        for j in range(32):
            if (c >> j) & 1:
                r ^= m[j]
        return r

    base = []
    for j in range(32):
        c = 1 << j
        for _ in range(8):
            c = (c >> 1) ^ _POLY if c & 1 else c >> 1
        base.append(c)
    m = [1 << j for j in range(32)]
    while nbytes:
        if nbytes & 1:
            m = [apply(base, col) for col in m]
        base = [apply(base, col) for col in base]
        nbytes >>= 1
    return m, apply


def _as_bytes_tensor(data) -> torch.Tensor:
    if isinstance(data, torch.Tensor):
        t = data.detach()
    else:
        buf = data.tobytes() if isinstance(data, np.ndarray) else bytes(data)
        t = torch.frombuffer(bytearray(buf), dtype=torch.uint8) if buf else torch.zeros(0, dtype=torch.uint8)
    t = t.contiguous().reshape(-1).view(torch.uint8)
    if not t.is_cuda:
        t = t.pin_memory().to("cuda", non_blocking=True) if t.numel() else t.to("cuda")
    if t.numel() and t.data_ptr() % 16:
        t = t.clone()
    return t


_WS: dict = {}


def _crc_workspace(device) -> torch.Tensor:
    """Per-device, per-stream workspace holding the kernel's lookup tables."""
    dev = torch.device(device)
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    key = (dev, torch.cuda.current_stream(dev).cuda_stream)
    ws = _WS.get(key)
    if ws is None:
        ws = torch.empty(_lib.load().b200moe_crc32c_workspace_bytes(), dtype=torch.uint8, device=dev)
        _lib.call("b200moe_crc32c_init", ws.data_ptr(), _lib.stream_ptr())
        _WS[key] = ws
    return ws


class _CRC:
    """Batches device CRCs: one uint32 slot per payload, one D2H at the end."""

    def __init__(self, n: int, device="cuda"):
        self.out = torch.zeros(max(n, 1), dtype=torch.int64, device=device)
        self._ws = _crc_workspace(device)
        self._keep = []

    def add(self, i: int, t: torch.Tensor) -> None:
        b = _as_bytes_tensor(t)
        self._keep.append(b)
        _lib.call("b200moe_crc32c", b.data_ptr() if b.numel() else None, b.numel(), self.out[i:i + 1].data_ptr(),
                  self._ws.data_ptr(), _lib.stream_ptr())

    def values(self) -> list:
        return [int(v) & 0xFFFFFFFF for v in self.out.cpu().tolist()]


def crc32c(data, crc: int = 0) -> int:
    """CRC32C of bytes / a numpy array / a tensor, computed on the GPU;
    `crc` continues a previous checksum (crc32c(b, crc32c(a)) == crc32c(a+b))."""
    b = _as_bytes_tensor(data)
    c = _CRC(1)
    c.add(0, b)
    v = c.values()[0]
    if crc:
        m, apply = _shift_matrix(b.numel())
        v ^= apply(m, crc)
    return v


# --------------------------------------------------------------------------
# save
# --------------------------------------------------------------------------

def _payload(t: torch.Tensor):
    if t.dtype not in _TORCH_TO_NAME:
        raise ConfigError(f"tensor has unsupported dtype {t.dtype}")
    name = _TORCH_TO_NAME[t.dtype]
    dev = t.detach()
    if not dev.is_cuda:
        dev = dev.to("cuda")
    dev = dev.to(_DTYPES[name][0]).contiguous()
    return name, dev


def _write_payload(path: str, kind: str, model: ModelConfig, tensors: dict, gate: GateConfig | None = None,
                   moe_layers=None) -> None:
    os.makedirs(path, exist_ok=True)
    names = sorted(tensors)
    payloads = [_payload(tensors[n]) for n in names]
    crc = _CRC(len(names))
    for i, (_, dev) in enumerate(payloads):
        crc.add(i, dev)
    records, offset = [], 0
    with open(os.path.join(path, "weights.bin"), "wb") as f:
        for name, (dt, dev) in zip(names, payloads):
            pad = (-offset) % ALIGNMENT
            if pad:
                f.write(b"\x00" * pad)
            offset += pad
            host = dev.cpu()
            nbytes = host.numel() * host.element_size()
            f.write(host.reshape(-1).view(torch.uint8).numpy().tobytes())
            records.append({"name": name, "dtype": dt, "shape": list(dev.shape), "offset": offset,
                            "length": nbytes, "crc32c": None})
            offset += nbytes
    for rec, v in zip(records, crc.values()):
        rec["crc32c"] = v
    manifest = {"format_version": FORMAT_VERSION, "kind": kind, "model": asdict(model),
                "gate": None if gate is None else asdict(gate),
                "moe_layers": list(moe_layers) if moe_layers is not None else None, "tensors": records}
    with open(os.path.join(path, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=2, sort_keys=True)
        f.write("\n")


def save_checkpoint(ckpt, path: str) -> None:
    """Write a dense or MoE checkpoint (checkpoint.py:138-148)."""
    if isinstance(ckpt, MoECheckpoint):
        ckpt.validate()
        _write_payload(path, "moe", ckpt.config, ckpt.tensors, gate=ckpt.gate, moe_layers=ckpt.moe_layers)
    elif isinstance(ckpt, DenseCheckpoint):
        ckpt.validate()
        _write_payload(path, "dense", ckpt.config, ckpt.tensors)
    else:
        raise ConfigError(f"cannot save object of type {type(ckpt).__name__}")


def save_shard(shard, path: str) -> None:
    """Write one rank's shard plus its shard.json sidecar (checkpoint.py:151-168)."""
    if isinstance(shard, MoEShard):
        _write_payload(path, "moe_shard", shard.config, shard.tensors, gate=shard.gate, moe_layers=shard.moe_layers)
    elif isinstance(shard, DenseShard):
        _write_payload(path, "dense_shard", shard.config, shard.tensors)
    else:
        raise ConfigError(f"cannot save object of type {type(shard).__name__}")
    with open(os.path.join(path, "shard.json"), "w") as f:
        json.dump({"rank": shard.rank, "tp": [shard.tp_index, shard.tp_size], "ep": [shard.ep_index, shard.ep_size]},
                  f, indent=2, sort_keys=True)
        f.write("\n")


# --------------------------------------------------------------------------
# load
# --------------------------------------------------------------------------

def _read_manifest(path: str) -> dict:
    mp = os.path.join(path, "manifest.json")
    try:
        with open(mp) as f:
            manifest = json.load(f)
    except json.JSONDecodeError as e:
        raise ManifestError(f"manifest is not valid JSON: {mp}: {e}") from e
    version = manifest.get("format_version")
    if version != FORMAT_VERSION:
        raise UnknownVersionError(f"unsupported checkpoint format version {version!r} (expected {FORMAT_VERSION})")
    return manifest


def _check_records(path: str, manifest: dict) -> list:
    size = os.path.getsize(os.path.join(path, "weights.bin"))
    seen, out = set(), []
    for rec in manifest["tensors"]:
        name = rec["name"]
        if name in seen:
            raise ManifestError(f"duplicate tensor record: {name}")
        seen.add(name)
        if rec["dtype"] not in _DTYPES:
            raise ManifestError(f"tensor {name}: unknown dtype {rec['dtype']!r}")
        tdt, _, isz = _DTYPES[rec["dtype"]]
        shape = tuple(rec["shape"])
        expected = int(np.prod(shape, dtype=np.int64)) * isz
        if expected != rec["length"]:
            raise ManifestError(f"tensor {name}: manifest length {rec['length']} does not match shape {shape} x "
                                f"{isz} bytes = {expected}")
        if rec["offset"] + rec["length"] > size:
            raise TruncatedFileError(f"weights.bin truncated: tensor {name} needs bytes "
                                     f"[{rec['offset']}, {rec['offset'] + rec['length']}) of {size}")
        out.append((name, tdt, shape, rec))
    return out


def _read_tensors(path: str, manifest: dict, verify: bool = True, device="cuda") -> dict:
    recs = _check_records(path, manifest)
    tensors = {}
    crc = _CRC(len(recs), device) if verify else None
    with open(os.path.join(path, "weights.bin"), "rb") as f:
        for i, (name, tdt, shape, rec) in enumerate(recs):
            f.seek(rec["offset"])
            raw = f.read(rec["length"])
            if len(raw) != rec["length"]:
                raise TruncatedFileError(f"weights.bin truncated while reading tensor {name}")
            host = torch.frombuffer(bytearray(raw), dtype=torch.uint8) if raw else torch.zeros(0, dtype=torch.uint8)
            dev = host.pin_memory().to(device, non_blocking=True) if raw else host.to(device)
            if crc is not None:
                crc.add(i, dev)
            tensors[name] = dev.view(tdt).reshape(shape)
    if crc is not None:
        for (name, _, _, rec), v in zip(recs, crc.values()):
            if v != rec["crc32c"]:
                raise ChecksumError(f"checksum mismatch for tensor {name}")
    return tensors


def _gate_from_json(d):
    if d is None:
        return None
    try:
        return GateConfig(**d)
    except TypeError as e:
        raise ManifestError(f"bad gate config in manifest: {e}") from e


def _model_from_json(d) -> ModelConfig:
    try:
        return ModelConfig(**d)
    except TypeError as e:
        raise ManifestError(f"bad model config in manifest: {e}") from e


def _stack_experts(tensors: dict, layers, experts, device) -> dict:
    """Rebuild the bf16 kernel-layout stacks (W1, W3 [E,F,H], W2 [E,H,F]) from
    per-expert [in, out] tensors with the K12 transpose kernel.  When every
    expert tensor of a layer is f32 holding bf16-representable values (what
    upcycle_full / save_checkpoint of this build produce) the per-expert entries
    become views of the stacks, exactly as upcycle_full returns them.
    Otherwise (f64 experts, or f32 values a bf16 copy would round) the loaded
    full-precision tensors stay the checkpoint values -- load -> save
    reproduces the file bytes -- and the stacks are separate bf16 compute
    copies (a warning says so)."""
    stacked = {}
    experts = list(experts)
    for i in layers:
        p = f"layers.{i}.moe.experts"
        exact = all(_bf16_exact(tensors[f"{p}.{e:03d}.{w}"]) for e in experts for w in ("w1", "w2", "w3"))
        if not exact:
            warnings.warn(f"layer {i}: expert weights are not bf16-representable f32; the B200 kernels compute "
                          f"on bf16 copies, the checkpoint keeps the original values", RuntimeWarning, stacklevel=3)
        w1 = tensors[f"{p}.{experts[0]:03d}.w1"]
        H, F = w1.shape
        n = len(experts)
        W1 = torch.empty(n, F, H, dtype=EXPERT_DTYPE, device=device)
        W3 = torch.empty(n, F, H, dtype=EXPERT_DTYPE, device=device)
        W2 = torch.empty(n, H, F, dtype=EXPERT_DTYPE, device=device)
        for j, e in enumerate(experts):
            src = [tensors[f"{p}.{e:03d}.{w}"] for w in ("w1", "w2", "w3")]
            fp32 = int(src[0].dtype != torch.bfloat16)
            src = [s.to(torch.float32 if fp32 else torch.bfloat16).contiguous() for s in src]
            _lib.call("b200moe_upcycle_copy", src[0].data_ptr(), src[1].data_ptr(), src[2].data_ptr(), fp32, H, F, 1,
                      W1[j].data_ptr(), W2[j].data_ptr(), W3[j].data_ptr(), _lib.stream_ptr())
            if not exact:
                continue
            tensors[f"{p}.{e:03d}.w1"] = W1[j].t()
            tensors[f"{p}.{e:03d}.w2"] = W2[j].t()
            tensors[f"{p}.{e:03d}.w3"] = W3[j].t()
        stacked[i] = (W1, W2, W3)
    return stacked


def load_checkpoint(path: str, verify: bool = True, device="cuda"):
    """Read a dense or MoE checkpoint (checkpoint.py:222-239); MoE experts come
    back as bf16 kernel-layout stacks (views in `tensors`)."""
    manifest = _read_manifest(path)
    kind = manifest.get("kind")
    if kind not in ("dense", "moe"):
        raise ManifestError(f"not a whole-model checkpoint (kind={kind!r}); use load_shard")
    model = _model_from_json(manifest["model"])
    tensors = _read_tensors(path, manifest, verify=verify, device=device)
    if kind == "dense":
        ckpt = DenseCheckpoint(config=model, tensors=tensors)
        ckpt.validate()
        return ckpt
    gate = _gate_from_json(manifest.get("gate"))
    if gate is None or manifest.get("moe_layers") is None:
        raise ManifestError("moe checkpoint missing gate config or moe_layers")
    layers = tuple(manifest["moe_layers"])
    ckpt = MoECheckpoint(config=model, gate=gate, moe_layers=layers, tensors=tensors)
    ckpt.validate()
    ckpt.stacked = _stack_experts(tensors, layers, range(gate.n_experts), device)
    return ckpt


def load_shard(path: str, verify: bool = True, device="cuda"):
    """Read one rank's shard (checkpoint.py:242-258)."""
    manifest = _read_manifest(path)
    kind = manifest.get("kind")
    if kind not in ("dense_shard", "moe_shard"):
        raise ManifestError(f"not a shard checkpoint (kind={kind!r}); use load_checkpoint")
    with open(os.path.join(path, "shard.json")) as f:
        sidecar = json.load(f)
    model = _model_from_json(manifest["model"])
    tensors = _read_tensors(path, manifest, verify=verify, device=device)
    common = dict(rank=sidecar["rank"], tp_index=sidecar["tp"][0], tp_size=sidecar["tp"][1],
                  ep_index=sidecar["ep"][0], ep_size=sidecar["ep"][1], config=model, tensors=tensors)
    if kind == "dense_shard":
        return DenseShard(**common)
    gate = _gate_from_json(manifest.get("gate"))
    if gate is None or manifest.get("moe_layers") is None:
        raise ManifestError("moe shard missing gate config or moe_layers")
    layers = tuple(manifest["moe_layers"])
    block = gate.n_experts // sidecar["ep"][1]
    owned = tuple(range(sidecar["ep"][0] * block, (sidecar["ep"][0] + 1) * block))
    shard = MoEShard(gate=gate, moe_layers=layers, owned=owned, **common)
    shard.stacked = _stack_experts(tensors, layers, owned, device)
    return shard


__all__ = ["FORMAT_VERSION", "ALIGNMENT", "crc32c", "save_checkpoint", "save_shard", "load_checkpoint", "load_shard"]
