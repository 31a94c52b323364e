"""cuDNN SDPA forward + backward at config 2 (library anchor; ncu capture
target for comparing its kernels' counters with ours -- never product)."""
import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

g = torch.Generator(device="cuda")
g.manual_seed(2024)
q, k, v, do = (torch.randn((1, 16, 8192, 128), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
    for _ in range(3):
        qq, kk, vv = (t.detach().requires_grad_(True) for t in (q, k, v))
        o = F.scaled_dot_product_attention(qq, kk, vv, is_causal=True)
        o.backward(do)
torch.cuda.synchronize()
