"""Device timeline of the bench step (config 2 by default): kernel start /
end stamps from the torch profiler (CUPTI), idle gaps between consecutive
kernels on the step's stream, and the host time to issue one step.
python tools/step_gaps.py [n] [heads]"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_14509_b200 as U  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
h = int(sys.argv[2]) if len(sys.argv) > 2 else 16
g = torch.Generator(device="cuda")
g.manual_seed(2024)
q, k, v, do = (torch.randn((n, 1, h, 128), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
layer = U.DistributedAttention(U.FlashAttention("causal"), U.SequenceGroup.single())


def step():
    qq, kk, vv = (x.detach().requires_grad_(True) for x in (q, k, v))
    o = layer(qq, kk, vv)
    torch.autograd.backward([o], [do])


for _ in range(5):
    step()
torch.cuda.synchronize()
# host issue time per step (GPU kept busy by a long kernel in front)
big = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
big.view(torch.int64).sum()
t0 = time.perf_counter()
for _ in range(5):
    step()
host_ms = (time.perf_counter() - t0) / 5 * 1e3
torch.cuda.synchronize()

from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        step()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ker = sorted(((e.time_range.start, e.time_range.end, e.name) for e in evs), key=lambda x: x[0])
rows = []
prev_end = None
for s, e, nm in ker:
    gap = None if prev_end is None else s - prev_end
    rows.append({"name": nm[:48], "us": round(e - s, 1), "gap_before_us": None if gap is None else round(gap, 1)})
    prev_end = e
print(json.dumps({"host_issue_ms_per_step": round(host_ms, 3), "timeline": rows}, indent=0))
