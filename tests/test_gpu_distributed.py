"""DistributedAttention end to end on the GPU vs the reference goldens.

P ranks run as an in-process SequenceGroup on one B200 (own stream per
rank).  Mirrors test_ulysses.py TestForward / TestBackward: oracle
equivalence, P-invariance, ledger law (8 logical all_to_all of n*b*d per
fwd+bwd), config 1 (P=2, N=1024, 8x64, fp32) against the reference's own
outputs.
"""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from helpers import BF16_MAXREL, assert_rtol, rel_max_err, run_ranks, to_dev, to_np
from oracle import ulysses_oracle as O

pytestmark = pytest.mark.gpu


def U():
    import paper_2309_14509_b200 as mod
    return mod


def run_layer(p, q, k, v, do, mask, dtype, backward=True, slot_bytes=16 << 20):
    """Forward (+backward) of DistributedAttention over P local ranks.
    q/k/v/do are full [n, b, h, hd] float64 arrays; returns full arrays."""
    n = q.shape[0]
    nl = n // p
    groups = U().SequenceGroup.local_group(p, slot_bytes=slot_bytes) if p > 1 else [U().SequenceGroup.single()]
    attn = U().FlashAttention(mask)
    layers = [U().DistributedAttention(attn, g) for g in groups]
    sh = lambda x, r: to_dev(x[r * nl:(r + 1) * nl], dtype).requires_grad_(backward)
    # every rank's tensors (leaves and incoming grads) live on that rank's
    # stream, so autograd never couples two ranks' streams (a rank's device
    # wait would then block its peer's push on a shared stream)
    ins = run_ranks(groups, lambda r: [sh(x, r) for x in (q, k, v)])
    dos = run_ranks(groups, lambda r: to_dev(do[r * nl:(r + 1) * nl], dtype))

    def fwd(r):
        return layers[r](*ins[r])

    outs = run_ranks(groups, fwd)
    o = np.concatenate([to_np(x) for x in outs], 0)
    grads = None
    if backward:
        def bwd(r):
            torch.autograd.backward([outs[r]], [dos[r]])
            return [t.grad for t in ins[r]]
        gr = run_ranks(groups, bwd)
        grads = [np.concatenate([to_np(gr[r][i]) for r in range(p)], 0) for i in range(3)]
    return o, grads, groups


@pytest.mark.parametrize("ci", range(4))
def test_golden_small_fp32(ci):
    g = np.load(os.path.join(GOLDEN, "attn_small.npz"))
    p, n, b, h, hd, causal, seed = (int(x) for x in g[f"case{ci}_meta"])
    mask = "causal" if causal else "none"
    q, k, v, do = (g[f"case{ci}_{t}"].astype(np.float64) for t in ("q", "k", "v", "do"))
    o, (dq, dk, dv), groups = run_layer(p, q, k, v, do, mask, torch.float32)
    assert_rtol(o, g[f"case{ci}_o"])
    assert_rtol(dq, g[f"case{ci}_dq"])
    assert_rtol(dk, g[f"case{ci}_dk"])
    assert_rtol(dv, g[f"case{ci}_dv"])
    if p > 1:
        # ledger law: 8 logical all_to_all of aggregate n*b*d (test_ulysses.py:220-222)
        recs = groups[0].records
        assert len(recs) == 8
        assert all(r.aggregate_elements == n * b * h * hd for r in recs)
        assert groups[0].total_egress() == 8 * (n // p * b * h * hd) // p * (p - 1)


def test_config1_fp32_against_reference_outputs():
    g = np.load(os.path.join(GOLDEN, "config1.npz"))
    p, n, b, h, hd, seed = (int(x) for x in g["meta"])
    rows = g["rows"]
    q, k, v, do = (O.make_tensor((n, b, h, hd), seed, s) for s in (1, 2, 3, 4))
    for mask in ("none", "causal"):
        o, grads, _ = run_layer(p, q, k, v, do, mask, torch.float32, backward=(mask == "causal"))
        assert_rtol(o[rows], g[f"{mask}_o_rows"])
        if grads is not None:
            for name, gr in zip(("dq", "dk", "dv"), grads):
                assert_rtol(gr[rows], g[f"causal_{name}_rows"])


@pytest.mark.parametrize("p", [1, 2, 4, 8])
def test_bf16_forward_vs_oracle_and_p_invariance(p):
    n, b, hq, hkv, hd = 1024, 1, 8, 8, 128
    q, k, v, do = (O.make_tensor((n, b, hh, hd), 31, s, "bfloat16") for s, hh in
                   ((1, hq), (2, hkv), (3, hkv), (4, hq)))
    ref, _ = O.local_attention(q, k, v, "causal", exact=False)
    o, _, _ = run_layer(p, q, k, v, do, "causal", torch.bfloat16, backward=False)
    assert rel_max_err(o, ref) <= BF16_MAXREL
    o1, _, _ = run_layer(1, q, k, v, do, "causal", torch.bfloat16, backward=False)
    # per-head kernel is deterministic and independent of P -> bitwise P-invariance
    assert np.array_equal(o, o1)


@pytest.mark.parametrize("p,hq,hkv", [(2, 8, 8), (4, 8, 4), (8, 16, 8)])
def test_bf16_forward_backward_vs_oracle(p, hq, hkv):
    n, b, hd = 1024, 1, 128
    q, k, v, do = (O.make_tensor((n, b, hh, hd), 51 + p, s, "bfloat16") for s, hh in
                   ((1, hq), (2, hkv), (3, hkv), (4, hq)))
    ref, _ = O.local_attention(q, k, v, "causal", exact=False)
    gref = O.local_attention_backward(q, k, v, do, "causal", exact=False)
    o, grads, groups = run_layer(p, q, k, v, do, "causal", torch.bfloat16, backward=True)
    assert rel_max_err(o, ref) <= BF16_MAXREL
    for name, got, r in zip(("dq", "dk", "dv"), grads, gref):
        err = rel_max_err(got, r)
        assert err <= BF16_MAXREL, f"{name}: {err:.3e}"
    # 4 native exchange calls per fwd+bwd (QKV fused, O, dO, dQdKdV fused)
    assert groups[0].native_ledger()["calls"] == 4


@pytest.mark.parametrize("p,hq,hkv,n", [(2, 4, 4, 640), (4, 8, 4, 1024), (8, 8, 8, 1024)])
def test_fused_epilogue_exchange_equals_unfused(p, hq, hkv, n):
    # K2 fused into the attention epilogues must move exactly the bytes the
    # stand-alone head->seq all-to-all moves (bitwise)
    hd = 128
    attn = U().FlashAttention("causal", deterministic=True)
    groups = U().SequenceGroup.local_group(p, slot_bytes=3 * n * hq * hd * 2 // p + (1 << 20))
    mk = lambda h, s, r: to_dev(O.make_tensor((n, 1, h // p, hd), 60 + r, s, "bfloat16"), torch.bfloat16)
    ins = run_ranks(groups, lambda r: [mk(hq, 1, r), mk(hkv, 2, r), mk(hkv, 3, r), mk(hq, 4, r)])

    def fused(r):
        q, k, v, do = ins[r]
        o, lse, o_seq = attn.forward_exchange(q, k, v, groups[r])
        return o, lse, o_seq, attn.backward_exchange(q, k, v, o, lse, do, groups[r])

    def unfused(r):
        q, k, v, do = ins[r]
        o, lse = attn.forward_with_lse(q, k, v)
        (o_seq,) = groups[r].all_to_all([o], 0, 2)
        dq, dk, dv = attn.backward(q, k, v, o, lse, do)
        return o, lse, o_seq, groups[r].all_to_all([dq, dk, dv], 0, 2)

    a = run_ranks(groups, fused)
    b = run_ranks(groups, unfused)
    for r in range(p):
        assert torch.equal(a[r][0], b[r][0]) and torch.equal(a[r][1], b[r][1])
        assert torch.equal(a[r][2], b[r][2]), f"rank {r}: fused O exchange differs"
        for x, y in zip(a[r][3], b[r][3]):
            assert torch.equal(x, y), f"rank {r}: fused dQ/dK/dV exchange differs"


@pytest.mark.parametrize("p,hq,hkv,n", [(2, 4, 2, 640), (4, 8, 4, 1024)])
def test_fused_backward_exchange_moves_its_own_gradients(p, hq, hkv, n):
    # default (atomic-dQ) backward: the sequence-layout gradients a rank
    # receives are bitwise the stand-alone head->seq exchange of the
    # head-layout gradients the same calls produced, and match the oracle
    hd = 128
    attn = U().FlashAttention("causal")
    groups = U().SequenceGroup.local_group(p, slot_bytes=3 * n * hq * hd * 2 // p + (1 << 20))
    mk = lambda h, s, r: to_dev(O.make_tensor((n, 1, h // p, hd), 70 + r, s, "bfloat16"), torch.bfloat16)
    ins = run_ranks(groups, lambda r: [mk(hq, 1, r), mk(hkv, 2, r), mk(hkv, 3, r), mk(hq, 4, r)])

    def fused(r):
        q, k, v, do = ins[r]
        o, lse, _ = attn.forward_exchange(q, k, v, groups[r])
        return attn.backward_exchange(q, k, v, o, lse, do, groups[r], return_head=True)

    a = run_ranks(groups, fused)
    heads = run_ranks(groups, lambda r: groups[r].all_to_all(list(a[r][1]), 0, 2))
    for r in range(p):
        for x, y in zip(a[r][0], heads[r]):
            assert torch.equal(x, y), f"rank {r}: fused-backward exchange differs from its own head layout"
        q, k, v, do = (to_np(t).astype(np.float64) for t in ins[r])
        ref = O.local_attention_backward(q, k, v, do, "causal", exact=False)
        for name, got, want in zip(("dq", "dk", "dv"), a[r][1], ref):
            err = rel_max_err(to_np(got), want)
            assert err <= BF16_MAXREL, f"rank {r} {name}: {err:.3e}"


def test_bf16_gqa_forward_p4():
    n, b, hq, hkv, hd = 512, 1, 8, 4, 128
    q, k, v, do = (O.make_tensor((n, b, hh, hd), 41, s, "bfloat16") for s, hh in
                   ((1, hq), (2, hkv), (3, hkv), (4, hq)))
    ref, _ = O.local_attention(q, k, v, "causal", exact=False)
    o, _, _ = run_layer(4, q, k, v, do, "causal", torch.bfloat16, backward=False)
    assert rel_max_err(o, ref) <= BF16_MAXREL


def test_generic_local_attn_plugin_route():
    # any callable local_attn(q, k, v) on head-sharded tensors plugs in
    # (kernels.py plugin contract); the exchanges run through seq_all_to_all
    import torch.nn.functional as F

    def torch_attn(q, k, v):   # [n, b, h, d] -> [n, b, h, d], causal
        to = lambda x: x.permute(1, 2, 0, 3)
        return F.scaled_dot_product_attention(to(q), to(k), to(v), is_causal=True).permute(2, 0, 1, 3)

    p, n, h, hd = 4, 256, 8, 64
    q, k, v, do = (O.make_tensor((n, 1, h, hd), 91, s) for s in (1, 2, 3, 4))
    # in-process groups: every kernel on the path must be loaded before a
    # rank's flag wait spins (CUDA lazy loading blocks the issuing thread) --
    # warm the plugin's own kernels once, forward and backward
    w = [torch.zeros((n, 1, h // p, hd), device="cuda", requires_grad=True) for _ in range(3)]
    torch_attn(*w).sum().backward()
    torch.cuda.synchronize()
    groups = U().SequenceGroup.local_group(p, slot_bytes=1 << 20)
    layers = [U().DistributedAttention(torch_attn, g) for g in groups]
    nl = n // p
    ins = run_ranks(groups, lambda r: [to_dev(x[r * nl:(r + 1) * nl]).requires_grad_(True) for x in (q, k, v)])
    outs = run_ranks(groups, lambda r: layers[r](*ins[r]))
    ref, _ = O.local_attention(q, k, v, "causal", exact=False)
    got = np.concatenate([to_np(o) for o in outs], 0)
    assert rel_max_err(got, ref) <= 1e-4
    dos = run_ranks(groups, lambda r: to_dev(do[r * nl:(r + 1) * nl]))
    run_ranks(groups, lambda r: torch.autograd.backward([outs[r]], [dos[r]]))
    gref = O.local_attention_backward(q, k, v, do, "causal", exact=False)
    for i in range(3):
        g = np.concatenate([to_np(ins[r][i].grad) for r in range(p)], 0)
        assert rel_max_err(g, gref[i]) <= 1e-4
    # 4 separate seq_all_to_all per direction: 8 logical records, 8 native calls
    assert len(groups[0].records) == 8 and groups[0].native_ledger()["calls"] == 8


def test_divisibility_errors():
    groups = U().SequenceGroup.local_group(4, slot_bytes=1 << 20)
    layer = U().DistributedAttention(U().FlashAttention("causal"), groups[0])
    x = torch.zeros(8, 1, 6, 64, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(U().DivisibilityError, match="head count 6"):
        layer(x, x, x)
