"""A/B of the forward kernel instantiations (UL_FWD_VARIANT, read once per
process): each variant in a subprocess times the config-2 forward (L2 flushed
by reading a 1 GiB buffer before every launch) and checks its output
against the two-tile kernel (variant 0)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, math, statistics, sys, torch
sys.path.insert(0, sys.argv[1])
import paper_2309_14509_b200 as U
n, h, hd = int(sys.argv[2]), int(sys.argv[3]), 128
hkv = int(sys.argv[4])
g = torch.Generator(device="cuda"); g.manual_seed(1)
q = torch.randn((n, 1, h, hd), generator=g, device="cuda").to(torch.bfloat16)
k = torch.randn((n, 1, hkv, hd), generator=g, device="cuda").to(torch.bfloat16)
v = torch.randn((n, 1, hkv, hd), generator=g, device="cuda").to(torch.bfloat16)
attn = U.FlashAttention("causal")
flush = torch.empty(1 << 28, dtype=torch.float32, device="cuda")
ts = []
for it in range(13):
    flush.sum()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); o, lse = attn.forward_with_lse(q, k, v); e.record()
    if it >= 3: ts.append((a, e))
torch.cuda.synchronize()
ms = statistics.mean(a.elapsed_time(e) for a, e in ts)
torch.save((o.cpu(), lse.cpu()), sys.argv[5])
print(json.dumps({"ms": round(ms, 4), "tflops": round(4 * h * n * n * hd * 0.5 / ms / 1e9, 1)}))
"""


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    h = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    hkv = int(sys.argv[3]) if len(sys.argv) > 3 else h
    variants = [int(x) for x in (sys.argv[4].split(",") if len(sys.argv) > 4 else "0,1,2,3,4".split(","))]
    import torch
    out = {}
    ref = None
    for var in variants:
        path = f"/tmp/fwd_ab_{var}.pt"
        env = dict(os.environ, UL_FWD_VARIANT=str(var))
        r = subprocess.run([sys.executable, "-c", CHILD, ROOT, str(n), str(h), str(hkv), path], env=env,
                           capture_output=True, text=True, timeout=600)
        if r.returncode != 0:
            out[var] = {"error": r.stderr[-800:]}
            continue
        rec = json.loads(r.stdout.strip().splitlines()[-1])
        o, lse = torch.load(path)
        if ref is None:
            ref = (o, lse)
        else:
            rec["max_abs_o_vs_first"] = float((o.float() - ref[0].float()).abs().max())
            rec["max_abs_lse_vs_first"] = float((lse - ref[1]).abs().max())
        out[var] = rec
    print(json.dumps({"n": n, "h": h, "hkv": hkv, "variants": out}))


if __name__ == "__main__":
    main()
