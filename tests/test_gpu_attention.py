"""K3/K4 local attention on the GPU vs the f64 oracle.

bf16 mode (tcgen05/TMEM/TMA): max|a - o| <= 2e-2 * max|o| (north star),
o = oracle in float64 on the same bf16-rounded inputs.
fp32 mode (SIMT): |a - o| <= 1e-5 |o| + 1e-6 max|o|.
Mirrors test_kernels.py (n=1, causal row 0, FD-checked backward) and
test_oracle.py (causality probe) at GPU sizes.
"""

import math

import numpy as np
import pytest
import torch

from helpers import BF16_MAXREL, assert_rtol, rel_max_err, to_dev, to_np
from oracle import ulysses_oracle as O

pytestmark = pytest.mark.gpu


def U():
    import paper_2309_14509_b200 as mod
    return mod


def inputs(n, b, hq, hkv, hd, dtype, seed=0):
    dt = "bfloat16" if dtype == torch.bfloat16 else "float32"
    q = O.make_tensor((n, b, hq, hd), seed, 1, dt)
    k = O.make_tensor((n, b, hkv, hd), seed, 2, dt)
    v = O.make_tensor((n, b, hkv, hd), seed, 3, dt)
    do = O.make_tensor((n, b, hq, hd), seed, 4, dt)
    return q, k, v, do


FWD_CASES = [
    # n, b, hq, hkv, hd, mask
    (1, 1, 1, 1, 64, "none"),
    (5, 1, 2, 2, 64, "causal"),
    (128, 1, 2, 2, 128, "causal"),
    (200, 2, 4, 2, 128, "causal"),
    (256, 1, 2, 1, 64, "none"),
    (384, 1, 4, 4, 128, "none"),
    (1000, 1, 2, 2, 128, "causal"),
    (1024, 1, 8, 8, 64, "causal"),
]


@pytest.mark.parametrize("n,b,hq,hkv,hd,mask", FWD_CASES)
def test_fwd_bf16_vs_oracle(n, b, hq, hkv, hd, mask):
    q, k, v, _ = inputs(n, b, hq, hkv, hd, torch.bfloat16, seed=n + hd)
    kind = "causal" if mask == "causal" else "none"
    ref, ref_lse = O.local_attention(q, k, v, kind, exact=False)
    attn = U().FlashAttention(mask)
    o, lse = attn.forward_with_lse(*(to_dev(x, torch.bfloat16) for x in (q, k, v)))
    torch.cuda.synchronize()
    assert rel_max_err(to_np(o), ref) <= BF16_MAXREL
    assert np.abs(to_np(lse) - ref_lse).max() <= 2e-2


BWD_CASES = [
    # n, b, hq, hkv, hd, mask
    (1, 1, 1, 1, 64, "causal"),
    (64, 1, 2, 2, 128, "causal"),
    (130, 1, 2, 1, 128, "none"),
    (256, 2, 4, 2, 64, "causal"),
    (512, 1, 4, 4, 128, "causal"),
    (640, 1, 4, 1, 128, "none"),
    (1000, 1, 2, 2, 128, "causal"),
    (384, 2, 4, 2, 128, "causal"),      # batch 2 + GQA through the fused kernel
    (200, 3, 2, 1, 128, "none"),
]


@pytest.mark.parametrize("deterministic", [False, True], ids=["fused", "deterministic"])
@pytest.mark.parametrize("n,b,hq,hkv,hd,mask", BWD_CASES)
def test_bwd_bf16_vs_oracle(n, b, hq, hkv, hd, mask, deterministic):
    q, k, v, do = inputs(n, b, hq, hkv, hd, torch.bfloat16, seed=100 + n + hd)
    kind = "causal" if mask == "causal" else "none"
    dq_r, dk_r, dv_r = O.local_attention_backward(q, k, v, do, kind, exact=False)
    attn = U().FlashAttention(mask, deterministic=deterministic)
    tq, tk, tv, tdo = (to_dev(x, torch.bfloat16) for x in (q, k, v, do))
    o, lse = attn.forward_with_lse(tq, tk, tv)
    dq, dk, dv = attn.backward(tq, tk, tv, o, lse, tdo)
    torch.cuda.synchronize()
    for name, got, ref in (("dq", dq, dq_r), ("dk", dk, dk_r), ("dv", dv, dv_r)):
        err = rel_max_err(to_np(got), ref)
        assert err <= BF16_MAXREL, f"{name}: max-abs / max|ref| = {err:.3e}"
    # dK/dV never use atomics: a second backward is bitwise identical; dQ too
    # in deterministic mode (the fused mode's fp32 atomic order may vary)
    dq2, dk2, dv2 = attn.backward(tq, tk, tv, o, lse, tdo)
    assert torch.equal(dk, dk2) and torch.equal(dv, dv2)
    if deterministic or hd != 128:
        assert torch.equal(dq, dq2)
    else:
        assert rel_max_err(to_np(dq2), to_np(dq)) <= 1e-2


@pytest.mark.parametrize("n,b,hq,hkv,hd,mask", [(1, 1, 1, 1, 8, "none"), (7, 2, 4, 2, 3, "causal"),
                                                (64, 1, 4, 4, 16, "none"), (300, 1, 4, 1, 64, "causal"),
                                                (129, 2, 2, 2, 128, "causal")])
def test_fwd_bwd_fp32_vs_oracle(n, b, hq, hkv, hd, mask):
    q, k, v, do = inputs(n, b, hq, hkv, hd, torch.float32, seed=7 + n)
    kind = "causal" if mask == "causal" else "none"
    ref, ref_lse = O.local_attention(q, k, v, kind, exact=False)
    dq_r, dk_r, dv_r = O.local_attention_backward(q, k, v, do, kind, exact=False)
    attn = U().FlashAttention(mask)
    tq, tk, tv, tdo = (to_dev(x) for x in (q, k, v, do))
    o, lse = attn.forward_with_lse(tq, tk, tv)
    dq, dk, dv = attn.backward(tq, tk, tv, o, lse, tdo)
    torch.cuda.synchronize()
    assert_rtol(to_np(o), ref)
    assert np.abs(to_np(lse) - ref_lse).max() <= 1e-5
    assert_rtol(to_np(dq), dq_r)
    assert_rtol(to_np(dk), dk_r)
    assert_rtol(to_np(dv), dv_r)


def test_single_token_context_is_v():
    # test_kernels.py:32-35
    for dt in (torch.float32, torch.bfloat16):
        q, k, v, _ = inputs(1, 2, 2, 2, 64, dt, seed=3)
        o, _ = U().FlashAttention("none").forward_with_lse(*(to_dev(x, dt) for x in (q, k, v)))
        assert np.array_equal(to_np(o), v)


def test_causal_first_row_is_v0():
    # test_kernels.py:37-40
    for dt in (torch.float32, torch.bfloat16):
        q, k, v, _ = inputs(300, 1, 2, 2, 128 if dt == torch.bfloat16 else 32, dt, seed=4)
        o, _ = U().FlashAttention("causal").forward_with_lse(*(to_dev(x, dt) for x in (q, k, v)))
        assert np.array_equal(to_np(o)[0], v[0])


def test_causality_probe_bf16():
    # test_oracle.py:83-93: perturbing key/value row j must not change rows < j
    n, hd = 512, 128
    q, k, v, _ = inputs(n, 1, 2, 2, hd, torch.bfloat16, seed=5)
    attn = U().FlashAttention("causal")
    base, _ = attn.forward_with_lse(*(to_dev(x, torch.bfloat16) for x in (q, k, v)))
    k2, v2 = k.copy(), v.copy()
    k2[300] += 4.0
    v2[300] += 4.0
    bumped, _ = attn.forward_with_lse(*(to_dev(x, torch.bfloat16) for x in (q, k2, v2)))
    assert torch.equal(base[:300], bumped[:300])
    assert (base[300:] - bumped[300:]).abs().max().item() > 1e-3


def test_deterministic_and_longest_first_order_independent():
    q, k, v, _ = inputs(1024, 1, 4, 4, 128, torch.bfloat16, seed=6)
    attn = U().FlashAttention("causal")
    tq, tk, tv = (to_dev(x, torch.bfloat16) for x in (q, k, v))
    a, la = attn.forward_with_lse(tq, tk, tv)
    b, lb = attn.forward_with_lse(tq, tk, tv)
    assert torch.equal(a, b) and torch.equal(la, lb)


def test_kernel_errors():
    attn = U().FlashAttention("causal")
    x = torch.zeros(4, 1, 2, 96, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(U().KernelError):
        attn.forward_with_lse(x, x, x)
    with pytest.raises(U().KernelError):
        U().get_kernel("blocked")
    y = torch.zeros(4, 1, 4, 64, device="cuda", dtype=torch.bfloat16)
    z = torch.zeros(4, 1, 3, 64, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(U().DivisibilityError):
        attn.forward_with_lse(y, z, z)
    with pytest.raises(U().ForwardStateError):
        attn.backward(y, y, y, y, None, y)


def test_bwd_bf16_large_gqa_full():
    # N = 4096, GQA 4q/1kv: every gradient element against the f64 oracle
    n, hq, hkv, hd = 4096, 4, 1, 128
    q, k, v, do = inputs(n, 1, hq, hkv, hd, torch.bfloat16, seed=77)
    dq_r, dk_r, dv_r = O.local_attention_backward(q, k, v, do, "causal", exact=False)
    attn = U().FlashAttention("causal")
    tq, tk, tv, tdo = (to_dev(x, torch.bfloat16) for x in (q, k, v, do))
    o, lse = attn.forward_with_lse(tq, tk, tv)
    dq, dk, dv = attn.backward(tq, tk, tv, o, lse, tdo)
    torch.cuda.synchronize()
    for name, got, ref in (("dq", dq, dq_r), ("dk", dk, dk_r), ("dv", dv, dv_r)):
        err = rel_max_err(to_np(got), ref)
        assert err <= BF16_MAXREL, f"{name}: {err:.3e}"


def test_p_invariance_of_head_sharded_kernels():
    # a rank's heads give bitwise the same result as the same heads inside a
    # larger launch (what Ulysses P-invariance needs from the local kernel)
    n, hd = 1024, 128
    q, k, v, do = inputs(n, 1, 8, 8, hd, torch.bfloat16, seed=12)
    attn = U().FlashAttention("causal", deterministic=True)
    tq, tk, tv, tdo = (to_dev(x, torch.bfloat16) for x in (q, k, v, do))
    o, lse = attn.forward_with_lse(tq, tk, tv)
    g = attn.backward(tq, tk, tv, o, lse, tdo)
    sl = slice(2, 4)
    parts = [t[:, :, sl].contiguous() for t in (tq, tk, tv, tdo)]
    o2, lse2 = attn.forward_with_lse(*parts[:3])
    g2 = attn.backward(*parts[:3], o2, lse2, parts[3])
    assert torch.equal(o2, o[:, :, sl]) and torch.equal(lse2, lse[:, sl])
    for a, b in zip(g2, g):
        assert torch.equal(a, b[:, :, sl])


@pytest.mark.parametrize("n,hq", [(8192, 4), (40960, 2)])
def test_fwd_bf16_large_sampled_rows(n, hq):
    # full-size config-2 shape (persistent grid, pair-major order) and a
    # sequence with >= 148 query-tile pairs per head (one-shot grid,
    # head-major order); oracle on sampled query-row blocks (row_offset)
    hd = 128
    q, k, v, _ = inputs(n, 1, hq, hq, hd, torch.bfloat16, seed=9)
    o, lse = U().FlashAttention("causal").forward_with_lse(*(to_dev(x, torch.bfloat16) for x in (q, k, v)))
    o = to_np(o)
    lse = to_np(lse)
    for r0 in (0, 4000, n // 2 + 64, n - 128):
        ref, ref_lse = O.local_attention(q, k, v, "causal", exact=False, rows=(r0, r0 + 128))
        assert rel_max_err(o[r0:r0 + 128], ref) <= BF16_MAXREL
        assert np.abs(lse[:, :, r0:r0 + 128] - ref_lse).max() <= 2e-2


@pytest.mark.parametrize("n,hq,hkv", [(8192, 12, 12), (8192, 24, 12), (4096, 20, 10), (20480, 2, 2)])
def test_fused_bwd_head_groups_match_deterministic(n, hq, hkv):
    # long sequences with many heads take the head-grouped CTA order (a
    # partial last group exits early), >= 148 kv tiles per head the
    # head-major order: gradients must equal the
    # deterministic two-kernel path's within bf16 rounding
    hd = 128
    g = torch.Generator(device="cuda")
    g.manual_seed(n + hq)
    mk = lambda h: (torch.randn((n, 1, h, hd), generator=g, device="cuda")).to(torch.bfloat16)
    q, k, v, do = mk(hq), mk(hkv), mk(hkv), mk(hq)
    fused, det = U().FlashAttention("causal"), U().FlashAttention("causal", deterministic=True)
    o, lse = fused.forward_with_lse(q, k, v)
    a = fused.backward(q, k, v, o, lse, do)
    b = det.backward(q, k, v, o, lse, do)
    for name, x, y in zip(("dq", "dk", "dv"), a, b):
        err = float((x.float() - y.float()).abs().max() / y.float().abs().max())
        assert err <= 1e-2, f"{name}: {err:.3e}"


@pytest.mark.parametrize("n,hq", [(2048, 4), (38912, 1)])
def test_fwd_under_cuda_graph_capture(n, hq):
    # the persistent forward takes its items from a per-stream counter; under
    # capture it must not (a graph can be replayed on several streams): it
    # falls back to static waves (pair-major order) or the one-shot grid
    # (head-major, >= 148 pairs per head).  Replays equal the eager result.
    hd = 128
    g = torch.Generator(device="cuda")
    g.manual_seed(n)
    q, k, v = ((torch.randn((n, 1, hq, hd), generator=g, device="cuda")).to(torch.bfloat16) for _ in range(3))
    attn = U().FlashAttention("causal")
    o_ref, lse_ref = attn.forward_with_lse(q, k, v)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        attn.forward_with_lse(q, k, v)           # warm-up on the capture stream's side
    torch.cuda.current_stream().wait_stream(side)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        o_g, lse_g = attn.forward_with_lse(q, k, v)
    for _ in range(2):
        graph.replay()
    torch.cuda.synchronize()
    if n == 2048:      # same kernel, other schedule: per-item math is identical
        assert torch.equal(o_g, o_ref) and torch.equal(lse_g, lse_ref)
    else:
        assert rel_max_err(to_np(o_g), to_np(o_ref)) <= 1e-2
        assert float((lse_g - lse_ref).abs().max()) <= 1e-2


def test_layer_fwd_bwd_under_cuda_graph_capture():
    # the whole DistributedAttention step (forward + autograd backward, P = 1)
    # captured in one CUDA graph (tools/graph_step.py): replays equal the
    # eager step -- O and dK / dV exactly (same kernels, per-tile math), dQ
    # within the fused kernel's atomic-order rounding
    n, h, hd = 2048, 4, 128
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    mk = lambda: torch.randn((n, 1, h, hd), generator=g, device="cuda").to(torch.bfloat16)
    q, k, v, do = mk(), mk(), mk(), mk()
    layer = U().DistributedAttention(U().FlashAttention("causal"), U().SequenceGroup.single())
    eq, ek, ev = (x.detach().clone().requires_grad_(True) for x in (q, k, v))
    o_ref = layer(eq, ek, ev)
    torch.autograd.backward([o_ref], [do])
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        # fresh leaves: their AccumulateGrad nodes belong to the capture stream
        cq, ck, cv = (x.detach().clone().requires_grad_(True) for x in (q, k, v))
        o_w = layer(cq, ck, cv)
        torch.autograd.backward([o_w], [do])
        del o_w
        torch.cuda.synchronize()
        for t in (cq, ck, cv):
            t.grad = None
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            o_g = layer(cq, ck, cv)
            torch.autograd.backward([o_g], [do])
    torch.cuda.current_stream().wait_stream(side)
    for _ in range(2):
        graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(o_g, o_ref)
    assert torch.equal(ck.grad, ek.grad) and torch.equal(cv.grad, ev.grad)
    assert rel_max_err(to_np(cq.grad), to_np(eq.grad)) <= 1e-2
