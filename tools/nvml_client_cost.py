"""Config-2 step time with another process holding an NVML client open (diagnostic tool)."""
import os, sys, time, json, subprocess
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
CHILD = {
 "none": None,
 "sleeper": "import time\nprint('ready',flush=True)\ntime.sleep(5)",
 "nvml_idle": "import time, pynvml\npynvml.nvmlInit()\nprint('ready',flush=True)\ntime.sleep(5)",
 "nvml_idle_shutdown": "import time, pynvml\npynvml.nvmlInit()\npynvml.nvmlShutdown()\nprint('ready',flush=True)\ntime.sleep(5)",
}
def timed():
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    for i in range(20):
        flush.view(torch.int64).sum()
        ev[i][0].record(); step(); ev[i][1].record()
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in ev) / 20
res = {}
for rep in range(3):
    for name, code in CHILD.items():
        p = None
        if code:
            p = subprocess.Popen([sys.executable, "-c", code], stdout=subprocess.PIPE, text=True)
            p.stdout.readline()
        t = timed()
        if p: p.kill(); p.wait()
        res.setdefault(name, []).append(round(t, 4))
print(json.dumps(res))
