"""Library anchor (never on the product path): FlashAttention-4 (the CuTe-DSL
sm100 kernels vendored in vllm, JIT-compiled) at config 2 -- 16 heads x 128,
N = 8192, bf16, causal -- forward and forward+backward, CUDA events, L2
flushed by a read before each timed call.
    python tools/anchor_fa4.py [--ncu]   (--ncu: a few forward calls only)"""
import json
import statistics
import sys
import types

import torch

BASE = "/opt/prime-rl/.venv/lib/python3.12/site-packages/vllm/vllm_flash_attn"
import vllm  # noqa: E402,F401
_m = types.ModuleType("vllm.vllm_flash_attn")
_m.__path__ = [BASE]          # skip the package __init__ (it needs vllm's FA2/FA3 extensions)
sys.modules["vllm.vllm_flash_attn"] = _m
from vllm.vllm_flash_attn.cute.interface import flash_attn_func  # noqa: E402

n, h, hd = 8192, 16, 128
g = torch.Generator(device="cuda")
g.manual_seed(2024)
q, k, v, do = (torch.randn((1, n, h, hd), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
if "--ncu" in sys.argv:
    for _ in range(4):
        flash_attn_func(q, k, v, causal=True)
    torch.cuda.synchronize()
    sys.exit(0)
flush = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")


def timed(fn, reps=10, warm=3):
    ts = []
    for it in range(warm + reps):
        flush.view(torch.int64).sum()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        e.record()
        if it >= warm:
            ts.append((a, e))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(e) for a, e in ts)


def fb():
    qq, kk, vv = (x.detach().requires_grad_(True) for x in (q, k, v))
    o = flash_attn_func(qq, kk, vv, causal=True)
    o = o[0] if isinstance(o, tuple) else o
    o.backward(do)


ms_f = timed(lambda: flash_attn_func(q, k, v, causal=True))
ms_fb = timed(fb)
ff = 4.0 * h * n * n * hd * 0.5
print(json.dumps({"fa4_fwd_ms": round(ms_f, 4), "fa4_fwd_tflops": round(ff / ms_f / 1e9, 1),
                  "fa4_fwd_bwd_ms": round(ms_fb, 4), "fa4_bwd_ms_derived": round(ms_fb - ms_f, 4),
                  "fa4_bwd_tflops_derived": round(2 * ff / (ms_fb - ms_f) / 1e9, 1)}))
