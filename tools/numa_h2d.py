"""H2D bandwidth from pinned host memory allocated (first-touched) on each
NUMA node, with the copying thread bound to that node: is the e2e leg's
PCIe rate NUMA-dependent on this host?  (diagnostic tool, not product)"""
import json
import os
import subprocess

import torch

out = {}
try:
    out["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout[-1500:]
except Exception as e:
    out["topo"] = str(e)
nodes = {}
base = "/sys/devices/system/node"
for d in sorted(os.listdir(base)) if os.path.isdir(base) else []:
    if d.startswith("node"):
        with open(os.path.join(base, d, "cpulist")) as f:
            nodes[d] = f.read().strip()
out["nodes"] = nodes
try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    out["gpu_numa_affinity_words"] = [hex(x) for x in pynvml.nvmlDeviceGetCpuAffinity(h, 4)]
except Exception as e:
    out["nvml"] = str(e)


def parse(cl):
    cpus = set()
    for part in cl.split(","):
        if "-" in part:
            a, b = part.split("-")
            cpus.update(range(int(a), int(b) + 1))
        elif part:
            cpus.add(int(part))
    return cpus


dev = torch.device("cuda", 0)
N = 128 << 20
d = torch.empty(N, dtype=torch.uint8, device=dev)
all_cpus = os.sched_getaffinity(0)
res = {}
for name, cl in list(nodes.items()) + [("unbound", None)]:
    cpus = parse(cl) & all_cpus if cl else all_cpus
    if not cpus:
        continue
    os.sched_setaffinity(0, cpus)
    h = torch.empty(N, dtype=torch.uint8).pin_memory()
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        d.copy_(h, non_blocking=True)
    e.record()
    torch.cuda.synchronize()
    res[name] = round(10 * N / (s.elapsed_time(e) / 1e3) / 1e9, 1)
    del h
os.sched_setaffinity(0, all_cpus)
out["h2d_gbs"] = res
print(json.dumps(out, indent=1))
