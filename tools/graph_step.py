"""Config-2 step (DistributedAttention fwd + bwd at P = 1) eager vs captured
in a CUDA graph and replayed: same results, device time per step, and the
gap between the step and its kernels (tool)."""
import json
import os
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_14509_b200 as U  # noqa: E402

n, h, hd = 8192, 16, 128
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(2024)
mk = lambda: torch.randn((n, 1, h, hd), generator=g, device=dev).to(torch.bfloat16)
q, k, v, do = mk(), mk(), mk(), mk()
layer = U.DistributedAttention(U.FlashAttention("causal"), U.SequenceGroup.single(0))
flush = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
sq, sk, sv = (x.detach().clone().requires_grad_(True) for x in (q, k, v))


def step():
    for t in (sq, sk, sv):
        t.grad = None
    o = layer(sq, sk, sv)
    torch.autograd.backward([o], [do])
    return o


def timed(fn, reps=20):
    ts = []
    for it in range(3 + reps):
        flush.view(torch.int64).sum()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        e.record()
        if it >= 3:
            ts.append((a, e))
    torch.cuda.synchronize()
    return sum(a.elapsed_time(e) for a, e in ts) / len(ts)


o_e = step()
ref = [o_e.detach().clone()] + [t.grad.detach().clone() for t in (sq, sk, sv)]
eager = timed(step)
s = torch.cuda.Stream(dev)
s.wait_stream(torch.cuda.current_stream(dev))
with torch.cuda.stream(s):
    # fresh leaves: their AccumulateGrad nodes live on the capture stream
    cq, ck, cv = (x.detach().clone().requires_grad_(True) for x in (q, k, v))
    for _ in range(3):
        for t in (cq, ck, cv):
            t.grad = None
        o_w = layer(cq, ck, cv)
        torch.autograd.backward([o_w], [do])
    del o_w
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    for t in (cq, ck, cv):
        t.grad = None
    with torch.cuda.graph(graph, stream=s):
        o_g = layer(cq, ck, cv)
        torch.autograd.backward([o_g], [do])
torch.cuda.current_stream(dev).wait_stream(s)
graph.replay()
torch.cuda.synchronize()
got = [o_g.detach()] + [t.grad.detach() for t in (cq, ck, cv)]
diff = [float((a.float() - b.float()).abs().max()) for a, b in zip(got, ref)]
replay = timed(graph.replay)
print(json.dumps({"eager_ms": round(eager, 4), "graph_ms": round(replay, 4), "max_abs_diff_o_dq_dk_dv": diff}))
