"""CPU oracle for the checkpoint format.

TEST INFRASTRUCTURE ONLY: imported by tests/ as the checker of the GPU CRC32C
kernel and of the on-disk layout, never by the product path.

  crc32c        moefold/checkpoint.py:40-78 (C restatement in crc32c.c)
  crc32c_py     the same algorithm bit-serially in Python, for tiny inputs
  layout        moefold/checkpoint.py:101-135: sorted records, 64-byte aligned
                offsets, zero padding, manifest json (indent 2, sorted keys)
"""

from __future__ import annotations

import ctypes

import numpy as np

from .moe_oracle import _npexp_lib

ALIGNMENT = 64


def crc32c(data, crc: int = 0) -> int:
    b = np.frombuffer(bytes(data), dtype=np.uint8) if not isinstance(data, np.ndarray) else \
        np.ascontiguousarray(data).view(np.uint8).reshape(-1)
    lib = _npexp_lib()
    fn = lib.oracle_crc32c
    fn.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint32]
    fn.restype = ctypes.c_uint32
    return int(fn(b.ctypes.data, b.size, crc))


def crc32c_py(data: bytes, crc: int = 0) -> int:
    c = crc ^ 0xFFFFFFFF
    for byte in data:
        c ^= byte
        for _ in range(8):
            c = (c >> 1) ^ 0x82F63B78 if c & 1 else c >> 1
    return c ^ 0xFFFFFFFF


def layout(named_arrays: dict) -> tuple[list, bytes]:
    """(records, weights.bin bytes) for name -> little-endian f32/f64 array."""
    records, blobs, offset = [], [], 0
    for name in sorted(named_arrays):
        a = np.ascontiguousarray(named_arrays[name])
        dt = {np.dtype(np.float32): ("f32", "<f4"), np.dtype(np.float64): ("f64", "<f8")}[a.dtype]
        raw = a.astype(dt[1], copy=False).tobytes()
        pad = (-offset) % ALIGNMENT
        offset += pad
        blobs.append(b"\x00" * pad + raw)
        records.append({"name": name, "dtype": dt[0], "shape": list(a.shape), "offset": offset, "length": len(raw),
                        "crc32c": crc32c(raw)})
        offset += len(raw)
    return records, b"".join(blobs)
