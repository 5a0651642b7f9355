"""The dense projections of the model step (qkv, wo, lm-head; reference
model.py:135-169 through the matmul closure tensor.py:192-207) on the repo's
tcgen05 GEMM (tensor.linear -> b200moe_dense_fwd / _dgrad / _wgrad): y, dx
and dw against an fp32 reference on the same bf16-rounded operands."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


@pytest.mark.parametrize("M,K,N", [(8192, 4096, 6144), (8192, 4096, 4096), (1000, 4096, 128256 // 4),
                                   (300, 256, 512), (1, 512, 256), (129, 768, 1024), (77, 40, 24)])
def test_linear_matches_fp32(M, K, N):
    from paper_2412_09952_b200.tensor import linear
    g = torch.Generator(device="cuda").manual_seed(M + K + N)
    x = (torch.randn(M, K, generator=g, device="cuda")).to(torch.bfloat16).requires_grad_()
    w = (torch.randn(K, N, generator=g, device="cuda") * K ** -0.5).to(torch.bfloat16).requires_grad_()
    dy = torch.randn(M, N, generator=g, device="cuda").to(torch.bfloat16)
    y = linear(x, w)
    y.backward(dy)
    xf, wf, dyf = x.detach().float(), w.detach().float(), dy.float()
    assert y.dtype == torch.bfloat16 and tuple(y.shape) == (M, N)
    assert rel(y.float(), xf @ wf) < 5e-3
    assert rel(x.grad.float(), dyf @ wf.t()) < 5e-3
    assert rel(w.grad.float(), xf.t() @ dyf) < 5e-3


def test_linear_lm_head_vocab():
    """The lm-head shape: N = 128256 = 501 x 256 columns."""
    from paper_2412_09952_b200.tensor import linear
    M, K, N = 512, 4096, 128256
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(M, K, generator=g, device="cuda").to(torch.bfloat16).requires_grad_()
    w = (torch.randn(K, N, generator=g, device="cuda") * 0.02).to(torch.bfloat16).requires_grad_()
    dy = (torch.randn(M, N, generator=g, device="cuda") * 1e-3).to(torch.bfloat16)
    y = linear(x, w)
    y.backward(dy)
    xf, wf, dyf = x.detach().float(), w.detach().float(), dy.float()
    assert rel(y.float(), xf @ wf) < 5e-3
    assert rel(x.grad.float(), dyf @ wf.t()) < 5e-3
    assert rel(w.grad.float(), xf.t() @ dyf) < 5e-3


def test_dense_entry_points_strided_outputs_and_grid_cap():
    """The C entry points directly: the forward writing into a column block of a
    wider output (ldy > N, as a fused qkv buffer would), dgrad into a wider dx,
    and a capped persistent grid (2 and 38 CTAs) giving bit-identical results."""
    from paper_2412_09952_b200 import _lib
    from paper_2412_09952_b200.moe import _arange_i32
    from paper_2412_09952_b200.tensor import _one_segment
    M, K, N, LD = 300, 512, 256, 768
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(3)
    x = torch.randn(M, K, generator=g, device=dev).to(torch.bfloat16)
    w = (torch.randn(K, N, generator=g, device=dev) * 0.05).to(torch.bfloat16)
    dy = torch.randn(M, N, generator=g, device=dev).to(torch.bfloat16)
    base, cnt = _one_segment(M, dev)
    e0 = _arange_i32(1, dev)
    s = _lib.stream_ptr()
    outs = []
    for grid in (0, 2, 38):
        y = torch.full((M, LD), float("nan"), dtype=torch.bfloat16, device=dev)
        dx = torch.full((M, LD), float("nan"), dtype=torch.bfloat16, device=dev)
        dw = torch.empty(K, N, dtype=torch.bfloat16, device=dev)
        _lib.call("b200moe_dense_fwd", x.data_ptr(), w.data_ptr(), base.data_ptr(), cnt.data_ptr(), e0.data_ptr(),
                  M, K, N, K, N, LD, y[:, 256:].data_ptr(), grid, s)
        _lib.call("b200moe_dense_dgrad", dy.data_ptr(), w.data_ptr(), base.data_ptr(), cnt.data_ptr(),
                  e0.data_ptr(), M, K, N, N, N, LD, dx.data_ptr(), grid, s)
        _lib.call("b200moe_dense_wgrad", x.data_ptr(), dy.data_ptr(), base.data_ptr(), cnt.data_ptr(),
                  e0.data_ptr(), M, K, N, K, N, N, dw.data_ptr(), grid, s)
        torch.cuda.synchronize()
        assert torch.isnan(y[:, :256].float()).all() and torch.isnan(y[:, 512:].float()).all()   # untouched
        assert torch.isnan(dx[:, K:].float()).all()
        outs.append((y[:, 256:512].clone(), dx[:, :K].clone(), dw))
    assert rel(outs[0][0].float(), x.float() @ w.float()) < 5e-3
    assert rel(outs[0][1].float(), dy.float() @ w.float().t()) < 5e-3
    assert rel(outs[0][2].float(), x.float().t() @ dy.float()) < 5e-3
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            assert torch.equal(a, b)


def test_wgrad_subproblem_mask_and_grid_cap():
    """b200moe_expert_wgrad_ex: computing dW2 alone and dW1/dW3 alone on capped
    grids gives the same bits as the one-launch WGRAD, and leaves the other
    outputs untouched."""
    from paper_2412_09952_b200 import _lib
    H, F, counts = 256, 512, [300, 0, 129]
    E = len(counts)
    dev = torch.device("cuda")
    base, acc = [], 0
    for c in counts:
        base.append(acc)
        acc += (c + 127) // 128 * 128
    R = acc
    base_t = torch.tensor(base, dtype=torch.int32, device=dev)
    cnt_t = torch.tensor(counts, dtype=torch.int32, device=dev)
    seg_e = torch.arange(E, dtype=torch.int32, device=dev)
    g = torch.Generator(device=dev).manual_seed(4)
    mk = lambda C: torch.randn(R, C, generator=g, device=dev).to(torch.bfloat16)  # noqa: E731
    xp, Hh, dO, dA, dB = mk(H), mk(F), mk(H), mk(F), mk(F)
    for t in (xp, Hh, dO, dA, dB):   # zero the pad rows like the layer does
        for e, c in enumerate(counts):
            t[base[e] + c: base[e] + (c + 127) // 128 * 128] = 0
    bf = dict(dtype=torch.bfloat16, device=dev)
    s = _lib.stream_ptr()

    def run(subs, grid):
        outs = [torch.full((E, F, H), float("nan"), **bf), torch.full((E, H, F), float("nan"), **bf),
                torch.full((E, F, H), float("nan"), **bf)]
        _lib.call("b200moe_expert_wgrad_ex", xp.data_ptr(), Hh.data_ptr(), dO.data_ptr(), dA.data_ptr(),
                  dB.data_ptr(), base_t.data_ptr(), cnt_t.data_ptr(), seg_e.data_ptr(), E, R, H, F, E,
                  outs[0].data_ptr(), outs[1].data_ptr(), outs[2].data_ptr(), 0, subs, grid, s)
        torch.cuda.synchronize()
        return outs

    full = run(7, 0)
    w2 = run(4, 20)
    w13 = run(3, 38)
    assert torch.equal(w2[1], full[1]) and torch.isnan(w2[0].float()).all() and torch.isnan(w2[2].float()).all()
    assert torch.equal(w13[0], full[0]) and torch.equal(w13[2], full[2]) and torch.isnan(w13[1].float()).all()
