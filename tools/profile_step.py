"""Minimal workload for ncu: W warm-up + K layer steps (config 2 shape) with
no flushes, e2e or sweeps -- so `ncu --metrics gpu__time_duration.sum` lists
exactly the kernels of a step.

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python tools/profile_step.py 1 2
"""
import sys

import torch

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_14509_b200 as U  # noqa: E402

warm, steps = (int(a) for a in (sys.argv[1:3] if len(sys.argv) > 2 else (1, 2)))
dev = torch.device("cuda", 0)
n, H, hd = int(os.environ.get("PS_N", 8192)), int(os.environ.get("PS_H", 16)), 128   # shape override for long-N captures
g = torch.Generator(device=dev)
g.manual_seed(2024)
mk = lambda: torch.randn((n, 1, H, hd), generator=g, device=dev).to(torch.bfloat16)
q, k, v, do = mk(), mk(), mk(), mk()
layer = U.DistributedAttention(U.FlashAttention("causal"), U.SequenceGroup.single())
for i in range(warm + steps):
    qq, kk, vv = (t.detach().requires_grad_(True) for t in (q, k, v))
    o = layer(qq, kk, vv)
    torch.autograd.backward([o], [do])
torch.cuda.synchronize()
print("done")
