"""Diagnostic: where does the end-to-end (host-buffer) step time go?"""
import torch

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_14509_b200 as U  # noqa: E402

dev = torch.device("cuda", 0)
n, H, hd = 8192, 16, 128
mk = lambda: torch.randn((n, 1, H, hd), device=dev).to(torch.bfloat16)
q, k, v, do = mk(), mk(), mk(), mk()
hq = [t.cpu().pin_memory() for t in (q, k, v, do)]
print("pinned:", [t.is_pinned() for t in hq])
layer = U.DistributedAttention(U.FlashAttention("causal"), U.SequenceGroup.single())


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


bufs = [torch.empty_like(t, device=dev) for t in hq]


def h2d():
    for d_, s_ in zip(bufs, hq):
        d_.copy_(s_, non_blocking=True)


def compute():
    qq, kk, vv = (t.detach().requires_grad_(True) for t in (q, k, v))
    o = layer(qq, kk, vv)
    torch.autograd.backward([o], [do])


def seq_e2e():
    h2d()
    qq, kk, vv, dd = (t.detach() for t in bufs)
    for t in (qq, kk, vv):
        t.requires_grad_(True)
    o = layer(qq, kk, vv)
    torch.autograd.backward([o], [dd])
    (o.float() * dd.float()).sum().item()


print("h2d 128MB ms", timeit(h2d), "GB/s", 134217728 / timeit(h2d) / 1e6)
print("compute ms", timeit(compute))
print("sequential e2e ms", timeit(seq_e2e))
