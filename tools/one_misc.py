"""One launch sequence of the non-attention kernels for ncu captures:
the P = 1 seq->head exchange (a2a_copy_kernel on 3 x [8192, 1, 16, 128] bf16)
and the fused Q/K/V projection GEMM (qkv_proj, d = 2048, 8192 tokens).
    python tools/one_misc.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_14509_b200 as U  # noqa: E402

g = torch.Generator(device="cuda")
g.manual_seed(1)
xs = [torch.randn((8192, 1, 16, 128), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3)]
g1 = U.SequenceGroup.single()
d = 2048
x = torch.randn((8192, d), generator=g, device="cuda").to(torch.bfloat16)
w = torch.randn((d, 3 * d), generator=g, device="cuda").to(torch.bfloat16) / d ** 0.5
for _ in range(3):
    g1.all_to_all(xs, 2, 0)
    g1.qkv_projection(x, w, 1, 16, 16)
torch.cuda.synchronize()
