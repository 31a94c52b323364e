"""How much GPU time does one NVML query cost while kernels run?  (diagnostic
tool): 40 back-to-back 8192^2 bf16 GEMMs timed with CUDA events, with 0 / 1 / 2
/ 8 queries of the SM clock or of the clock-event reasons issued from another
process while they run."""
import json
import subprocess
import sys
import time

import torch

Q = r"""
import sys, time, pynvml
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
kind, n = sys.argv[1], int(sys.argv[2])
print("ready", flush=True); sys.stdin.readline()
time.sleep(0.01)
for _ in range(n):
    if kind == "clock": pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    else: pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
    time.sleep(0.004)
print("done", flush=True)
"""
a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
b = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
for _ in range(5):
    a @ b
torch.cuda.synchronize()
out = {}
for kind in ("clock", "reasons"):
    for n in (0, 1, 2, 8):
        ts = []
        for rep in range(3):
            p = subprocess.Popen([sys.executable, "-c", Q, kind, str(n)], stdin=subprocess.PIPE, stdout=subprocess.PIPE, text=True)
            p.stdout.readline()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(60):
                a @ b
            e.record()
            p.stdin.write("go\n"); p.stdin.flush()
            torch.cuda.synchronize()
            p.stdout.readline(); p.wait()
            ts.append(s.elapsed_time(e))
        out[f"{kind}_{n}"] = round(min(ts), 3)
print(json.dumps(out))
