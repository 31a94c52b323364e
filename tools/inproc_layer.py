"""Exposed exchange of the DistributedAttention layer with P in-process ranks
on one B200 (all traffic in local HBM, all ranks' kernels sharing the GPU):
fwd+bwd of every rank issued on its own stream, timed first launch to last
completion, against the same ranks' attention kernels alone (no exchange),
for the unpipelined (pipeline=1) and pipelined (pipeline=2) layer.

    python tools/inproc_layer.py [P] [heads] [N]
"""
import json
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_14509_b200 as U  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
H = int(sys.argv[2]) if len(sys.argv) > 2 else 32
N = int(sys.argv[3]) if len(sys.argv) > 3 else 32768
hd, nl = 128, N // P
g = torch.Generator(device="cuda")
g.manual_seed(7)
mk = lambda *s: torch.randn(s, generator=g, device="cuda").to(torch.bfloat16)
flush = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")


def run_group(fns, streams, reps=5):
    """Issue fns[r] on streams[r] (GPU kept busy by a flush read while the
    host enqueues), time first start to last end, mean of reps."""
    ts = []
    for it in range(2 + reps):
        torch.cuda.synchronize()
        flush.view(torch.int64).sum()
        flush.view(torch.int64).sum()
        start = torch.cuda.Event(enable_timing=True)
        start.record()
        ends = []
        for f, s in zip(fns, streams):
            s.wait_event(start)
            with torch.cuda.stream(s):
                f()
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                ends.append(e)
        torch.cuda.synchronize()
        if it >= 2:
            ts.append(max(start.elapsed_time(e) for e in ends))
    return sum(ts) / len(ts)


out = {"P": P, "heads": H, "N": N}
groups = U.SequenceGroup.local_group(P)
streams = [gr.stream for gr in groups]
# warm every rank stream's allocator (in-process groups: no cudaMalloc while ranks are issued)
for s in streams + [gr.channel.stream for gr in groups]:
    with torch.cuda.stream(s):
        torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
ins = [[mk(nl, 1, H, hd) for _ in range(4)] for _ in range(P)]
for pipe in (1, 2):
    layers = [U.DistributedAttention(U.FlashAttention("causal"), gr, pipeline=pipe) for gr in groups]

    def step(r, layers=layers):
        q, k, v, do = ins[r]
        qq, kk, vv = (x.detach().requires_grad_(True) for x in (q, k, v))
        torch.autograd.backward([layers[r](qq, kk, vv)], [do])
    out[f"layer_ms_pipeline{pipe}"] = round(run_group([lambda r=r: step(r) for r in range(P)], streams), 3)
    for gr in groups:
        gr.check()
# the same ranks' attention alone: each rank's head-sharded problem
att = U.FlashAttention("causal")
heads = [[mk(N, 1, H // P, hd) for _ in range(4)] for _ in range(P)]


def attn_only(r):
    q, k, v, do = heads[r]
    o, lse = att.forward_with_lse(q, k, v)
    att.backward(q, k, v, o, lse, do)
out["attention_only_ms"] = round(run_group([lambda r=r: attn_only(r) for r in range(P)], streams), 3)
for pipe in (1, 2):
    t = out[f"layer_ms_pipeline{pipe}"]
    out[f"exposed_pct_pipeline{pipe}"] = round(100.0 * (t - out["attention_only_ms"]) / t, 2)
print(json.dumps(out))
