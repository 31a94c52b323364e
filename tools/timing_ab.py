"""A/B of the kernel-timing method: event pairs with vs without a device
sleep in front (does the lead change the measured kernel time?)."""
import statistics

import torch

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_14509_b200 as U  # noqa: E402

dev = torch.device("cuda", 0)
n, H, hd = 8192, 16, 128
mk = lambda: torch.randn((n, 1, H, hd), device=dev).to(torch.bfloat16)
q, k, v, do = mk(), mk(), mk(), mk()
attn = U.FlashAttention("causal")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def run(lead, reps=20, back_to_back=1):
    ts = []
    for i in range(reps + 3):
        flush.zero_()
        if lead:
            torch.cuda._sleep(lead)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(back_to_back):
            attn.forward_with_lse(q, k, v)
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b) / back_to_back)
    return statistics.median(ts), min(ts)


for lead in (0, 50_000, 400_000, 2_000_000):
    print("lead", lead, "fwd ms (median, min)", run(lead))
print("back-to-back x10, no flush between", run(0, back_to_back=10))
