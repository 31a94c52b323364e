"""Same-box library anchors for config 2 (16 heads x 128, N = 8192, bf16,
causal): cuDNN SDPA (torch, fwd and fwd+bwd) and flashinfer's sm100 FMHA
(forward only) beside this repo's kernels.  Never on the product path;
bench.py imports `library_anchors` for its `anchors` field."""

from __future__ import annotations

import json
import math
import statistics
import sys


def _time(fn, warmup=3, reps=10, flush=None):
    import torch
    ts = []
    for it in range(warmup + reps):
        if flush is not None:
            flush.sum()    # L2 flush by reading (no dirty lines left behind)
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        e.record()
        if it >= warmup:
            ts.append((a, e))
    torch.cuda.synchronize()
    return statistics.mean(a.elapsed_time(e) for a, e in ts)


def library_anchors(n=8192, h=16, hd=128, warmup=3, reps=10, flush=None):
    import torch
    import torch.nn.functional as F
    from torch.nn.attention import SDPBackend, sdpa_kernel
    dev = torch.device("cuda")
    g = torch.Generator(device=dev)
    g.manual_seed(2024)
    mk = lambda: torch.randn((1, h, n, hd), generator=g, device=dev).to(torch.bfloat16)
    q, k, v, do = mk(), mk(), mk(), mk()
    f_fwd = 4.0 * h * n * n * hd * 0.5
    f_bwd = 2.0 * f_fwd
    out = {"shape": f"b=1, h={h}, n={n}, hd={hd}, bf16, causal"}
    try:
        with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
            ms_f = _time(lambda: F.scaled_dot_product_attention(q, k, v, is_causal=True), warmup, reps, flush)
            qq, kk, vv = (t.detach().requires_grad_(True) for t in (q, k, v))

            def fb():
                o = F.scaled_dot_product_attention(qq, kk, vv, is_causal=True)
                o.backward(do)
            ms_fb = _time(fb, warmup, reps, flush)
        out["cudnn_sdpa"] = {"fwd_ms": round(ms_f, 4), "fwd_tflops": round(f_fwd / ms_f / 1e9, 1),
                             "fwd_bwd_ms": round(ms_fb, 4),
                             "bwd_ms_derived": round(ms_fb - ms_f, 4),
                             "bwd_tflops_derived": round(f_bwd / (ms_fb - ms_f) / 1e9, 1),
                             "fwd_bwd_tflops": round((f_fwd + f_bwd) / ms_fb / 1e9, 1)}
    except Exception as exc:
        out["cudnn_sdpa"] = {"error": repr(exc)[:300]}
    try:
        with sdpa_kernel([SDPBackend.FLASH_ATTENTION]):
            ms_f = _time(lambda: F.scaled_dot_product_attention(q, k, v, is_causal=True), warmup, reps, flush)
            qq, kk, vv = (t.detach().requires_grad_(True) for t in (q, k, v))

            def fb2():
                o = F.scaled_dot_product_attention(qq, kk, vv, is_causal=True)
                o.backward(do)
            ms_fb = _time(fb2, warmup, reps, flush)
        out["torch_flash_sdpa"] = {"fwd_ms": round(ms_f, 4), "fwd_tflops": round(f_fwd / ms_f / 1e9, 1),
                                   "fwd_bwd_ms": round(ms_fb, 4),
                                   "fwd_bwd_tflops": round((f_fwd + f_bwd) / ms_fb / 1e9, 1)}
    except Exception as exc:
        out["torch_flash_sdpa"] = {"error": repr(exc)[:300]}
    try:
        import flashinfer
        qn, kn, vn = (t[0].transpose(0, 1).contiguous() for t in (q, k, v))   # [n, h, hd] (NHD)
        for backend in ("cutlass", "fa2"):
            try:
                fn = lambda: flashinfer.single_prefill_with_kv_cache(qn, kn, vn, causal=True, backend=backend,
                                                                     sm_scale=1.0 / math.sqrt(hd))
                fn()
                torch.cuda.synchronize()
                ms = _time(fn, warmup, reps, flush)
                out[f"flashinfer_{backend}"] = {"fwd_ms": round(ms, 4), "fwd_tflops": round(f_fwd / ms / 1e9, 1)}
            except Exception as exc:
                out[f"flashinfer_{backend}"] = {"error": repr(exc)[:300]}
    except Exception as exc:
        out["flashinfer"] = {"error": repr(exc)[:300]}
    return out


if __name__ == "__main__":
    import torch
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    flush = torch.empty(1 << 28, dtype=torch.float32, device="cuda")
    print(json.dumps(library_anchors(n=n, flush=flush)))
