"""The fused Q/K/V projection + seq->head exchange (ul_qkv_proj_exchange,
csrc/proj_sm100.cu) against project() + _to_head of the
oracle (layers.py:118-122, ulysses.py:140-146, 161-164): float64 GEMM of the
same bf16 operands, routed by the oracle's all_to_all, rounded to bf16."""

import numpy as np
import pytest
import torch

from helpers import run_ranks, to_dev, to_np, warm_streams
from oracle import ulysses_oracle as O

pytestmark = pytest.mark.gpu


def U():
    import paper_2309_14509_b200 as mod
    return mod


@pytest.mark.parametrize("p,nl,b,hq,hkv", [
    (1, 256, 1, 2, 2),
    (1, 200, 1, 3, 3),      # rows not a multiple of 128, columns not a multiple of 256
    (2, 128, 2, 4, 2),      # batch 2, GQA
    (4, 64, 1, 8, 4),
])
def test_qkv_projection_exchange(p, nl, b, hq, hkv):
    hd = 128
    d, dkv = hq * hd, hkv * hd
    n = nl * p
    x = O.bf16_round(O.make_tensor((n, b, d), 41, 1))
    w = O.bf16_round(O.make_tensor((d, d + 2 * dkv), 41, 2) / np.sqrt(d))
    groups = U().SequenceGroup.local_group(p, slot_bytes=32 << 20) if p > 1 else [U().SequenceGroup.single()]
    warm_streams(groups)
    wd = run_ranks(groups, lambda r: to_dev(w, torch.bfloat16))
    xs = run_ranks(groups, lambda r: to_dev(x[r * nl:(r + 1) * nl].reshape(nl * b, d), torch.bfloat16))
    outs = run_ranks(groups, lambda r: groups[r].qkv_projection(xs[r], wd[r], b, hq, hkv))
    # oracle: per-rank projections, then the seq->head all_to_all (split 2, concat 0)
    y = [O.matmul(x[r * nl:(r + 1) * nl].reshape(nl * b, d), w, exact=False) for r in range(p)]
    for t, (c0, c1, h) in enumerate(((0, d, hq), (d, d + dkv, hkv), (d + dkv, d + 2 * dkv, hkv))):
        seq = [yy[:, c0:c1].reshape(nl, b, h, hd) for yy in y]
        heads = O.all_to_all(seq, 2, 0)
        for r in range(p):
            got = to_np(outs[r][t])
            ref = heads[r]
            assert got.shape == ref.shape
            err = np.abs(got - ref).max() / np.abs(ref).max()
            assert err <= 1e-2, f"tensor {t} rank {r}: {err:.3e}"
            # bf16 rounding of an fp32-accumulated dot: within 2 ulp of the f64 value
            assert np.all(np.abs(got - ref) <= 2 * 2.0 ** -8 * np.abs(ref) + 1e-3 * np.abs(ref).max())
    if p > 1:
        led = groups[0].records
        assert [r.step_label for r in led[-3:]] == ["attn.q.seq2head", "attn.k.seq2head", "attn.v.seq2head"]


def test_layer_fused_path_is_taken_and_matches_unfused():
    # the bf16 hd-128 layer runs the fused projection; the generic route
    # (cuBLAS projections + stand-alone exchanges) gives the same result
    n, b, d, h, seed = 256, 1, 256, 2, 3
    w = {k: O.bf16_round(v) for k, v in O.make_weights(d, seed).items()}
    x = to_dev(O.bf16_round(O.make_input(n, b, d, seed)), torch.bfloat16)
    fused = U().UlyssesAttention(d, h, None, "causal", weights=w)
    generic = U().UlyssesAttention(d, h, None, "causal", weights=w)
    generic._fused_ok = lambda _x: False
    lib = U()._lib
    c0 = lib.total_launch_count()
    a = fused(x)
    torch.cuda.synchronize()
    assert lib.total_launch_count() > c0
    bb = generic(x)
    err = float((a.float() - bb.float()).abs().max() / bb.float().abs().max())
    assert err <= 2e-2


@pytest.mark.parametrize("p,nl,b,h", [(1, 200, 1, 3), (2, 128, 2, 4), (4, 64, 1, 8)])
def test_transposed_projection_exchange_dc(p, nl, b, h):
    # the backward's dc = g Wo^T (ulysses.py:207) with the dctx seq->head flip
    # (ulysses.py:213) in the GEMM epilogue: W read K-major from its [N, d_in] rows
    hd = 128
    d = h * hd
    n = nl * p
    g = O.bf16_round(O.make_tensor((n, b, d), 43, 1))
    wo = O.bf16_round(O.make_tensor((d, d), 43, 2) / np.sqrt(d))
    groups = U().SequenceGroup.local_group(p, slot_bytes=1 << 20) if p > 1 else [U().SequenceGroup.single()]
    warm_streams(groups)
    wd = run_ranks(groups, lambda r: to_dev(wo, torch.bfloat16))
    gs = run_ranks(groups, lambda r: to_dev(g[r * nl:(r + 1) * nl].reshape(nl * b, d), torch.bfloat16))
    outs = run_ranks(groups, lambda r: groups[r].proj_exchange(gs[r], wd[r], (h,), b, transposed=True)[0])
    seq = [O.matmul(g[r * nl:(r + 1) * nl].reshape(nl * b, d), wo.T, exact=False).reshape(nl, b, h, hd)
           for r in range(p)]
    heads = O.all_to_all(seq, 2, 0)
    for r in range(p):
        got, ref = to_np(outs[r]), heads[r]
        assert got.shape == ref.shape
        assert np.all(np.abs(got - ref) <= 2 * 2.0 ** -8 * np.abs(ref) + 1e-3 * np.abs(ref).max())
