"""The block's row-wise kernels (csrc/block.cu) against plain PyTorch fp32
references of the same ops: fused residual + layernorm (layers.py:106-110),
exact GELU (layers.py:113-127), forward and backward."""

import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu


def L():
    from paper_2309_14509_b200 import layer
    return layer


def _tol(dtype):
    return 1e-5 if dtype == torch.float32 else 2e-2


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("rows,d", [(1, 64), (37, 1000), (256, 2048), (8, 4096)])
def test_add_layernorm_fwd_bwd(dtype, rows, d):
    g = torch.Generator(device="cuda")
    g.manual_seed(rows + d)
    mk = lambda *s: torch.randn(*s, generator=g, device="cuda")
    x, r, dy, ds = mk(rows, d), mk(rows, d), mk(rows, d), mk(rows, d)
    gain, bias = 1 + 0.1 * mk(d), 0.1 * mk(d)
    # reference: fp32 torch on the same (rounded) inputs
    xs = [t.to(dtype).float().requires_grad_(True) for t in (x, r, gain, bias)]
    s_ref = xs[0] + xs[1]
    y_ref = F.layer_norm(s_ref, (d,), xs[2], xs[3], eps=1e-5)
    torch.autograd.backward([s_ref, y_ref], [ds.to(dtype).float(), dy.to(dtype).float()])
    ins = [t.to(dtype).requires_grad_(True) for t in (x, r, gain, bias)]
    s, y = L().add_layernorm(*ins)
    torch.autograd.backward([s, y], [ds.to(dtype), dy.to(dtype)])
    tol = _tol(dtype)
    rel = lambda a, b: float((a.float() - b).abs().max() / b.abs().max())
    assert rel(s, s_ref.detach()) <= tol and rel(y, y_ref.detach()) <= tol
    for a, b in zip(ins, xs):
        assert rel(a.grad, b.grad) <= tol * (5 if dtype == torch.bfloat16 else 10)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_layernorm_and_gelu_fwd_bwd(dtype):
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    x = torch.randn(300, 512, generator=g, device="cuda") * 3
    dy = torch.randn(300, 512, generator=g, device="cuda")
    xr = x.to(dtype).float().requires_grad_(True)
    yr = F.gelu(xr, approximate="none")
    yr.backward(dy.to(dtype).float())
    xi = x.to(dtype).requires_grad_(True)
    y = L().gelu(xi)
    y.backward(dy.to(dtype))
    tol = _tol(dtype)
    assert float((y.float() - yr).abs().max() / yr.abs().max()) <= tol
    assert float((xi.grad.float() - xr.grad).abs().max() / xr.grad.abs().max()) <= tol
    gain, bias = torch.ones(512, device="cuda", dtype=dtype), torch.zeros(512, device="cuda", dtype=dtype)
    a = L().layernorm(x.to(dtype), gain, bias)
    b = F.layer_norm(x.to(dtype).float(), (512,), eps=1e-5)
    assert float((a.float() - b).abs().max()) <= (1e-5 if dtype == torch.float32 else 3e-2)
