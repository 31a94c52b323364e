"""Shared test helpers (GPU-side runners for in-process sequence groups)."""

from __future__ import annotations

import numpy as np
import torch


def to_dev(x, dtype=torch.float32, device="cuda"):
    return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64).to(dtype).to(device).contiguous()


def to_np(t):
    return t.detach().to(torch.float64).cpu().numpy()


_WARMED = set()


def _warm_stream(s):
    """Reserve caching-allocator memory on a rank's stream once: a cudaMalloc
    issued while an earlier rank's flag wait spins can serialize the device
    behind it (implicit synchronization) -- a deadlock for in-process groups,
    whose peers are issued by the same host thread afterwards."""
    if s is None or s.stream_id in _WARMED:
        return
    _WARMED.add(s.stream_id)
    with torch.cuda.stream(s):
        small = [torch.empty(n, dtype=torch.uint8, device="cuda") for n in (512, 1 << 16, 1 << 19)]
        big = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        del small, big


def run_ranks(groups, fn):
    """Issue fn(rank) for every rank of an in-process group, each on its own
    stream (ranks of a local group must not share a stream: their device
    waits would serialise), then synchronise and surface desync errors."""
    torch.cuda.synchronize()
    for g in groups:
        _warm_stream(g.stream)
        ch = getattr(g, "_channel", None)
        if ch is not None:
            _warm_stream(ch.stream)
    torch.cuda.synchronize()
    out = []
    for g in groups:
        s = g.stream if g.stream is not None else torch.cuda.current_stream()
        with torch.cuda.stream(s):
            out.append(fn(g.rank))
    torch.cuda.synchronize()
    for g in groups:
        g.check()
    return out


def warm_streams(groups, dtypes=(torch.float32, torch.bfloat16), mb=256):
    """Create every rank stream's cuBLAS handle/workspace and reserve
    allocator memory on it before an in-process group runs library ops:
    first-use setup can block the host thread while an earlier rank's stream
    spins in a flag wait that only a later rank (same thread) can satisfy."""
    torch.cuda.synchronize()
    for g in groups:
        s = g.stream if g.stream is not None else torch.cuda.current_stream()
        with torch.cuda.stream(s):
            for dt in dtypes:
                a = torch.ones((256, 256), dtype=dt, device="cuda")
                (a @ a).sum().item()
                t = torch.nn.functional.layer_norm(a, (256,))
                torch.nn.functional.gelu(t).sum()
                # the ring merge's elementwise kernels (ring_attention_core)
                f = a.float().reshape(256, 1, 256, 1)
                m = torch.logaddexp(f, f)
                ((f * torch.exp(f - m) + f * torch.exp(m - f)).to(dt)).sum()
                f.permute(2, 0, 1, 3).unsqueeze(-1).contiguous()
            del a
            torch.empty(mb << 20, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()


def rel_max_err(a, ref):
    a = np.asarray(a, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.abs(a - ref).max() / max(np.abs(ref).max(), 1e-30))


# fp32-mode tolerance (north star: rtol 1e-5), with an absolute floor of
# 1e-6 * max(1, max|o|) for entries that are near zero by cancellation (the
# reference's own FD checks use the same max(1, ...) floor, test_kernels.py:131).
FP32_RTOL = 1e-5
FP32_ATOL_REL = 1e-6
# bf16-mode tolerance (north star): max|a - o| <= 2e-2 * max|o|, o in f64.
BF16_MAXREL = 2e-2


def assert_rtol(a, ref, rtol=FP32_RTOL, atol_rel=FP32_ATOL_REL):
    """fp32-mode contract: |a - o| <= rtol*|o| + atol_rel*max(1, max|o|)."""
    a = np.asarray(a, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    tol = rtol * np.abs(ref) + atol_rel * max(np.abs(ref).max(), 1.0)
    bad = np.abs(a - ref) > tol
    assert not bad.any(), f"{bad.sum()} elements out of tolerance; max err {np.abs(a - ref).max():.3e}"
