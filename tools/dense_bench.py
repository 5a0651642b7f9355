"""Dense projection GEMMs of the model step (qkv, wo, lm-head at T=8192,
hidden 4096, vocab 128256): the repo's tcgen05 dense GEMM (tensor.linear)
against torch.matmul (cuBLAS) on the same box, fwd + dgrad + wgrad, CUDA
events, best of interleaved reps.  Prints one JSON line."""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_09952_b200.tensor import linear  # noqa: E402


def timeit(fn, reps=10):
    ts = []
    for _ in range(3):
        fn()
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    dev = torch.device("cuda")
    M = 8192
    out = {}
    for name, (K, N) in {"qkv": (4096, 6144), "wo": (4096, 4096), "lm_head": (4096, 128256)}.items():
        x = torch.randn(M, K, device=dev).to(torch.bfloat16).requires_grad_()
        w = (torch.randn(K, N, device=dev) * 0.02).to(torch.bfloat16).requires_grad_()
        dy = torch.randn(M, N, device=dev).to(torch.bfloat16)

        def ours():
            x.grad = w.grad = None
            linear(x, w).backward(dy)

        def cublas():
            x.grad = w.grad = None
            (x @ w).backward(dy)

        from paper_2412_09952_b200 import _lib
        from paper_2412_09952_b200.tensor import _one_segment
        from paper_2412_09952_b200.moe import _arange_i32
        xb, wb = x.detach(), w.detach()
        base, cnt = _one_segment(M, dev)
        e0 = _arange_i32(1, dev)
        y = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
        dx = torch.empty(M, K, dtype=torch.bfloat16, device=dev)
        dw = torch.empty(K, N, dtype=torch.bfloat16, device=dev)
        s = lambda: _lib.stream_ptr()  # noqa: E731
        phases = {
            "fwd": (lambda: _lib.call("b200moe_dense_fwd", xb.data_ptr(), wb.data_ptr(), base.data_ptr(),
                                      cnt.data_ptr(), e0.data_ptr(), M, K, N, K, N, N, y.data_ptr(), 0, s()),
                    lambda: torch.matmul(xb, wb, out=y)),
            "dgrad": (lambda: _lib.call("b200moe_dense_dgrad", dy.data_ptr(), wb.data_ptr(), base.data_ptr(),
                                        cnt.data_ptr(), e0.data_ptr(), M, K, N, N, N, K, dx.data_ptr(), 0, s()),
                      lambda: torch.matmul(dy, wb.t(), out=dx)),
            "wgrad": (lambda: _lib.call("b200moe_dense_wgrad", xb.data_ptr(), dy.data_ptr(), base.data_ptr(),
                                        cnt.data_ptr(), e0.data_ptr(), M, K, N, K, N, N, dw.data_ptr(), 0, s()),
                      lambda: torch.matmul(xb.t(), dy, out=dw)),
            "fwd+bwd": (ours, cublas),
        }
        fl1 = 2.0 * M * K * N
        out[name] = {}
        for ph, (fo, fc) in phases.items():
            res = {}
            for _ in range(2):
                for nm, fn in (("ours", fo), ("cublas", fc)):
                    res.setdefault(nm, []).append(timeit(fn))
            fl = fl1 * (3 if ph == "fwd+bwd" else 1)
            out[name][ph] = {nm: {"ms": round(min(v), 4), "TFLOPs": round(fl / (min(v) * 1e-3) / 1e12, 1)}
                             for nm, v in res.items()}
        del y, dx, dw
        del x, w, dy
        torch.cuda.empty_cache()
    print(json.dumps({"dense_fwd_dgrad_wgrad": out, "tokens": M}))


if __name__ == "__main__":
    main()
