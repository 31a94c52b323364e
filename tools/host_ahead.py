"""Host enqueue time per config-2 step vs device time per step (diagnostic tool)."""
import os, sys, time, json
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import torch
sys.path.insert(0, "/root/repo")
import paper_2309_14509_b200 as U
n, h, hd = 8192, 16, 128
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(2024)
mk = lambda: torch.randn((n, 1, h, hd), generator=g, device=dev).to(torch.bfloat16)
q, k, v, do = mk(), mk(), mk(), mk()
layer = U.DistributedAttention(U.FlashAttention("causal"), U.SequenceGroup.single(0))
flush = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
def step():
    qq, kk, vv = (x.detach().requires_grad_(True) for x in (q, k, v))
    o = layer(qq, kk, vv)
    torch.autograd.backward([o], [do])
for _ in range(5): step()
torch.cuda.synchronize()
res = {}
for flushing in (True, False):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    t0 = time.perf_counter(); hs = []
    for i in range(20):
        if flushing: flush.view(torch.int64).sum()
        h0 = time.perf_counter()
        ev[i][0].record(); step(); ev[i][1].record()
        hs.append(time.perf_counter() - h0)
    t1 = time.perf_counter()
    torch.cuda.synchronize(); t2 = time.perf_counter()
    res[f"flush={flushing}"] = {"host_ms_per_step_enqueue": round(1e3 * sum(hs) / 20, 3), "host_total_ms": round(1e3 * (t1 - t0), 2),
                                "wait_after_enqueue_ms": round(1e3 * (t2 - t1), 2),
                                "gpu_ms_per_step": round(sum(a.elapsed_time(b) for a, b in ev) / 20, 4)}
print(json.dumps(res))
