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
