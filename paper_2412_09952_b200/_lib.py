"""ctypes binding of the b200moe C ABI (include/b200moe.h).

The product path has exactly one implementation: the sm_100a CUDA library
built in-tree at paper_2412_09952_b200/lib/libb200moe.so.  If it is missing or
no CUDA device is present, every op raises -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import ConfigError, GateError, ShapeError

_HERE = os.path.dirname(os.path.abspath(__file__))
# B200MOE_LIB overrides the library path (A/B experiments with variant builds).
LIB_PATH = os.environ.get("B200MOE_LIB") or os.path.join(_HERE, "lib", "libb200moe.so")

OK, ERR_SHAPE, ERR_CONFIG, ERR_GATE, ERR_CUDA = 0, -1, -2, -3, -4
ROUTER = {"mixtral": 0, "st": 1}
POLICY = {"position": 0, "score": 1}
LAYOUT_COMPACT, LAYOUT_FIXED = 0, 1

_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_F = ctypes.c_float

# name -> argtypes (every function returns int status)
SIGNATURES = {
    "b200moe_router_fwd": [_P, _P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P],
    "b200moe_gate_from_logits": [_P, _I, _I, _I, _I, _P, _P, _P, _P, _P],
    "b200moe_gate_bwd": [_P, _P, _P, _I, _I, _I, _P, _P],
    "b200moe_router_logits_bwd": [_P, _P, _P, _P, _P, _P, _I, _I, _I, _P, _P, _P, _P, _P, _P],
    "b200moe_dispatch": [_P, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "b200moe_dispatch_workspace_words": [_I],
    "b200moe_router_workspace_floats": [_I, _I],
    "b200moe_router_set_fma": [_I],
    "b200moe_permute": [_P, _P, _P, _P, _I, _I, _I, _P, _P],
    "b200moe_combine": [_P, _P, _P, _P, _I, _I, _I, _P, _P],
    "b200moe_combine_bwd": [_P, _P, _P, _P, _P, _P, _I, _I, _I, _P, _P, _P],
    "b200moe_router_bwd": [_P, _P, _P, _P, _P, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I,
                           _P, _P, _P, _P, _P],
    "b200moe_router_wgrad": [_P, _P, _P, _I, _I, _I, _P, _P, _P, _P, _P],
    "b200moe_permute_peer": [_P, _P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P],
    "b200moe_combine_peer": [_P, _I, _P, _P, _P, _I, _I, _I, _P, _P, _I, _P],
    "b200moe_combine_bwd_peer": [_P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _P, _P, _P, _I, _P],
    "b200moe_router_bwd_peer": [_P, _I, _P, _P, _P, _P, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I,
                                _I, _P, _P, _P, _P, _P],
    "b200moe_importance_fwd": [_P, _I, _I, _P, _P, _P, _P],
    "b200moe_importance_bwd": [_P, _P, _I, _P, _P],
    "b200moe_importance_loss": [_P, _I, _P, _P, _P],
    "b200moe_expert_fwd1": [_P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P, _P],
    "b200moe_expert_fwd2": [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _P, _P],
    "b200moe_expert_bwd2": [_P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P],
    "b200moe_expert_bwd1": [_P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _P, _P],
    "b200moe_expert_wgrad": [_P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P, _P],
    "b200moe_expert_wgrad_acc": [_P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P, _I, _P],
    "b200moe_expert_bwd2_ex": [_P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _I, _P],
    "b200moe_expert_bwd2_h": [_P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P, _I, _P],
    "b200moe_expert_fwd2_peer": [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _P, _I, _I, _I, _I, _P],
    "b200moe_expert_bwd1_peer": [_P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _P, _I, _I, _I, _I, _P],
    "b200moe_expert_bwd1_ex": [_P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _P, _I, _P],
    "b200moe_expert_wgrad_ex": [_P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P, _I, _I, _I, _P],
    "b200moe_dense_fwd": [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _P, _I, _P],
    "b200moe_dense_dgrad": [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _P, _I, _P],
    "b200moe_dense_wgrad": [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _P, _I, _P],
    "b200moe_gemm_set_cta_group": [_I],
    "b200moe_gemm_set_max_ctas": [_I],
    "b200moe_gemm_set_debug": [_I],
    "b200moe_upcycle_copy": [_P, _P, _P, _I, _I, _I, _I, _P, _P, _P, _P],
    "b200moe_version": [],
    "b200moe_rmsnorm_fwd": [_P, _P, _P, _I, _I, _F, _P, _P, _P, _P],
    "b200moe_rmsnorm_bwd": [_P, _P, _P, _P, _P, _I, _I, _P, _P, _P, _P, _P],
    "b200moe_embedding_fwd": [_P, _P, _I, _I, _I, _P, _P, _P],
    "b200moe_embedding_bwd": [_P, _P, _P, _P, _I, _I, _P, _P],
    "b200moe_embedding_bwd_sorted": [_P, _P, _P, _I, _I, _P, _P],
    "b200moe_cross_entropy_fwd": [_P, _P, _I, _I, _P, _P, _P, _P, _P],
    "b200moe_cross_entropy_bwd": [_P, _P, _P, _P, _I, _I, _P, _P],
    "b200moe_optimizer_chunk": [],
    "b200moe_optimizer_step": [_P, _P, _P, _I, _I, _F, _F, _F, _F, _F, _F, _F, _F, _F, _P],
    "b200moe_crc32c_workspace_bytes": [],
    "b200moe_crc32c_init": [_P, _P],
    "b200moe_crc32c": [_P, _I64, _P, _P, _P],
}

_lib = None
_lock = threading.Lock()


class NativeLibraryMissing(RuntimeError):
    """The CUDA library was not built (run __graft_entry__.build())."""


def load() -> ctypes.CDLL:
    """Load (once) and type the native library; raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryMissing(
                    f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
            lib = ctypes.CDLL(LIB_PATH)
            for name, argtypes in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = argtypes
                fn.restype = ctypes.c_int
            lib.b200moe_crc32c_workspace_bytes.restype = ctypes.c_longlong
            lib.b200moe_dispatch_workspace_words.restype = ctypes.c_size_t
            lib.b200moe_router_workspace_floats.restype = ctypes.c_size_t
            lib.b200moe_last_error.argtypes = []
            lib.b200moe_last_error.restype = ctypes.c_char_p
            _lib = lib
    return _lib


def exported_symbols() -> list[str]:
    return sorted(list(SIGNATURES) + ["b200moe_last_error"])


# Kernel launches issued by each entry point (for the bench's gpu_launches).
KERNELS_PER_CALL = {
    "b200moe_router_fwd": 2, "b200moe_gate_from_logits": 1, "b200moe_gate_bwd": 1, "b200moe_router_logits_bwd": 6, "b200moe_dispatch": 1, "b200moe_permute": 1,
    "b200moe_combine": 1, "b200moe_combine_bwd": 1, "b200moe_router_bwd": 1, "b200moe_router_wgrad": 1,
    "b200moe_importance_fwd": 1, "b200moe_importance_bwd": 1, "b200moe_importance_loss": 1, "b200moe_expert_fwd1": 1, "b200moe_expert_fwd2": 1,
    "b200moe_expert_bwd2": 1, "b200moe_expert_bwd1": 1, "b200moe_expert_wgrad": 1, "b200moe_expert_wgrad_acc": 1,
    "b200moe_expert_bwd1_ex": 1, "b200moe_expert_wgrad_ex": 1, "b200moe_expert_bwd2_ex": 1, "b200moe_expert_bwd2_h": 1, "b200moe_expert_fwd2_peer": 1,
    "b200moe_expert_bwd1_peer": 1,
    "b200moe_dense_fwd": 1, "b200moe_dense_dgrad": 1, "b200moe_dense_wgrad": 1,
    "b200moe_upcycle_copy": 3,
    "b200moe_permute_peer": 1, "b200moe_combine_peer": 1, "b200moe_combine_bwd_peer": 1, "b200moe_router_bwd_peer": 1,
    "b200moe_rmsnorm_fwd": 1, "b200moe_rmsnorm_bwd": 2, "b200moe_embedding_fwd": 1, "b200moe_embedding_bwd": 1,
    "b200moe_embedding_bwd_sorted": 1,
    "b200moe_cross_entropy_fwd": 2, "b200moe_cross_entropy_bwd": 1, "b200moe_optimizer_step": 1,
    "b200moe_crc32c": 2, "b200moe_crc32c_init": 1,
}


class Profiler:
    """Optional per-entry-point accounting: launch counts and, with
    `events=True`, CUDA events recorded on the current stream around each call
    (the stream the kernels are launched on).  With `spans=(starts, ends)`
    only two events per contiguous group of calls are recorded -- one before a
    call named in `starts`, one after a call named in `ends` -- so a timed
    region can carry the GEMM time of its own steps at 4 events per step."""

    def __init__(self, events: bool = False, spans: tuple | None = None):
        self.events = events
        self.spans = spans
        self.launches = 0
        self.calls: dict = {}
        self._pending: list = []
        self._open = None
        self.span_pairs: list = []

    def record(self, name, fn):
        self.launches += KERNELS_PER_CALL.get(name, 0)
        self.calls[name] = self.calls.get(name, 0) + 1
        if self.spans is not None:
            import torch
            # inside a CUDA-graph capture the events become event-record nodes
            # of the graph (external), so every replay re-times the spans
            ext = torch.cuda.is_current_stream_capturing()
            if name in self.spans[0] and self._open is None:
                self._open = torch.cuda.Event(enable_timing=True, external=ext)
                self._open.record()
            rc = fn()
            if name in self.spans[1] and self._open is not None:
                b = torch.cuda.Event(enable_timing=True, external=ext)
                b.record()
                self.span_pairs.append((self._open, b))
                self._open = None
            return rc
        if not self.events:
            return fn()
        import torch
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        rc = fn()
        b.record()
        self._pending.append((name, a, b))
        return rc

    def times_ms(self) -> dict:
        """Sum of event durations per entry point (synchronises)."""
        out: dict = {}
        for name, a, b in self._pending:
            b.synchronize()
            t, n = out.get(name, (0.0, 0))
            out[name] = (t + a.elapsed_time(b), n + 1)
        return out

    def span_ms(self) -> float:
        """Sum of the recorded span durations (synchronises)."""
        tot = 0.0
        for a, b in self.span_pairs:
            b.synchronize()
            tot += a.elapsed_time(b)
        return tot


# The grouped-GEMM launches of one layer step form two contiguous runs on the
# stream: FWD1 -> FWD2 and BWD2 -> WGRAD -> BWD1.
GEMM_SPANS = (("b200moe_expert_fwd1", "b200moe_expert_bwd2", "b200moe_expert_bwd2_ex", "b200moe_expert_bwd2_h",
               "b200moe_expert_wgrad_ex"),
              ("b200moe_expert_fwd2", "b200moe_expert_bwd1", "b200moe_expert_bwd1_ex", "b200moe_expert_fwd2_peer",
               "b200moe_expert_bwd1_peer"))


PROFILER: Profiler | None = None


def call(name: str, *args) -> None:
    """Invoke a C entry point and map its status onto the reference exceptions."""
    lib = load()
    fn = getattr(lib, name)
    if PROFILER is not None:
        rc = PROFILER.record(name, lambda: fn(*args))
    else:
        rc = fn(*args)
    if rc == OK:
        return
    msg = (lib.b200moe_last_error() or b"").decode(errors="replace")
    if rc == ERR_SHAPE:
        raise ShapeError(msg)
    if rc == ERR_CONFIG:
        raise ConfigError(msg)
    if rc == ERR_GATE:
        raise GateError(msg)
    raise RuntimeError(f"{name}: {msg} (status {rc})")


def host_u64(vals):
    """(ctypes uint64 array, its address) for a C entry point taking a HOST
    array of 64-bit values (e.g. per-rank device pointers); keep the array
    referenced until the call returns."""
    import ctypes
    arr = (ctypes.c_uint64 * len(vals))(*vals)
    return arr, ctypes.addressof(arr)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream
