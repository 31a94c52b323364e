"""A/B of the bench step's timing harness (config 2): the same fwd+bwd step
timed with CUDA events per step, L2 flushed by reading 1 GiB (bench
default), by zero_() (round 1), or not at all; the per-kernel sum beside it.
python tools/step_ab.py [steps]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_14509_b200 as U  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
n, h = 8192, 16
g = torch.Generator(device="cuda")
g.manual_seed(2024)
q, k, v, do = (torch.randn((n, 1, h, 128), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
layer = U.DistributedAttention(U.FlashAttention("causal"), U.SequenceGroup.single())
flush = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")


def step():
    qq, kk, vv = (x.detach().requires_grad_(True) for x in (q, k, v))
    o = layer(qq, kk, vv)
    torch.autograd.backward([o], [do])


def run(mode):
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        if mode == "read":
            flush.view(torch.int64).sum()
        elif mode == "zero":
            flush.zero_()
        elif mode == "read+cover":
            flush.view(torch.int64).sum()
            flush[: 256 << 20].view(torch.int64).sum()
        ev[i][0].record()
        step()
        ev[i][1].record()
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in ev)
    return {"mean_ms": round(sum(ts) / len(ts), 4), "median_ms": round(ts[len(ts) // 2], 4), "min_ms": round(ts[0], 4)}


out = [(m, run(m)) for m in ("read", "none", "zero", "read+cover", "read")]
print(json.dumps(out))
