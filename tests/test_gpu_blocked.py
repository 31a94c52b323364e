"""Blocked-sparse local attention on the B200 against
the reference goldens (tests/golden/blocked.npz: the Ulysses core with the
reference's blocked_kernel, kernels.py:55-86) and the blocked oracle."""

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


def ulysses_fwd(p, attn, q, k, v, dtype):
    """DistributedAttention forward over P in-process ranks; full arrays in/out."""
    n = q.shape[0]
    nl = n // p
    groups = U().SequenceGroup.local_group(p, slot_bytes=16 << 20) if p > 1 else [U().SequenceGroup.single()]
    layers = [U().DistributedAttention(attn, g) for g in groups]
    ins = run_ranks(groups, lambda r: [to_dev(x[r * nl:(r + 1) * nl], dtype) for x in (q, k, v)])
    outs = run_ranks(groups, lambda r: layers[r](*ins[r]))
    return np.concatenate([to_np(x) for x in outs], 0)


@pytest.mark.parametrize("ci", range(4))
def test_blocked_golden_fp32(ci):
    g = np.load(os.path.join(GOLDEN, "blocked.npz"))
    p, n, b, h, hd, bs, seed = (int(x) for x in g[f"case{ci}_meta"])
    pattern = [tuple(int(v) for v in row) for row in g[f"case{ci}_pattern"]]
    q, k, v = (g[f"case{ci}_{t}"].astype(np.float64) for t in ("q", "k", "v"))
    attn = U().get_kernel("blocked", block_size=bs, pattern=pattern)
    o = ulysses_fwd(p, attn, q, k, v, torch.float32)
    assert_rtol(o, g[f"case{ci}_o"])


@pytest.mark.parametrize("ci", [2, 3])   # hd 64 / 128: the tcgen05 kernel
def test_blocked_golden_bf16(ci):
    g = np.load(os.path.join(GOLDEN, "blocked.npz"))
    p, n, b, h, hd, bs, seed = (int(x) for x in g[f"case{ci}_meta"])
    pattern = [tuple(int(v) for v in row) for row in g[f"case{ci}_pattern"]]
    q, k, v = (O.bf16_round(g[f"case{ci}_{t}"]) for t in ("q", "k", "v"))
    attn = U().get_kernel("blocked", block_size=bs, pattern=pattern)
    o = ulysses_fwd(p, attn, q, k, v, torch.bfloat16)
    ref, _ = O.local_attention_blocked(q, k, v, bs, pattern, exact=False)
    assert rel_max_err(o, ref) <= BF16_MAXREL


def _irregular(nb, seed, density=0.2):
    rng = np.random.default_rng(seed)
    return {(qb, qb) for qb in range(nb)} | {(qb, kb) for qb in range(nb) for kb in range(nb)
                                            if rng.random() < density}


@pytest.mark.parametrize("n,hq,hkv,hd,bs,kind", [
    (1024, 4, 4, 128, 128, "causal"),     # one block per tile, tile skipping
    (1024, 4, 2, 128, 64, "banded"),      # two blocks per tile, GQA
    (768, 2, 2, 64, 256, "irregular"),    # blocks spanning tiles, hd 64
    (512, 2, 1, 128, 16, "irregular"),    # many small blocks per tile
    (1000, 2, 2, 128, 8, "banded"),       # n not a multiple of the tile
])
def test_blocked_bf16_vs_oracle(n, hq, hkv, hd, bs, kind):
    nb = n // bs
    pattern = {"causal": O.causal_block_pattern(n, bs), "banded": O.banded_block_pattern(n, bs, 2),
               "irregular": _irregular(nb, n + bs)}[kind]
    q, k, v = (O.bf16_round(O.make_tensor((n, 1, h, hd), 31, s)) for s, h in ((1, hq), (2, hkv), (3, hkv)))
    attn = U().FlashAttention("blocked", block_size=bs, pattern=pattern)
    o, lse = attn.forward_with_lse(*(to_dev(x, torch.bfloat16) for x in (q, k, v)))
    ref, ref_lse = O.local_attention_blocked(q, k, v, bs, pattern, exact=False)
    assert rel_max_err(to_np(o), ref) <= BF16_MAXREL
    assert np.abs(to_np(lse) - ref_lse).max() <= 2e-2 * max(1.0, np.abs(ref_lse).max())


def test_blocked_full_pattern_equals_dense_kernel():
    n, h, hd, bs = 512, 2, 128, 64
    q, k, v = (to_dev(O.bf16_round(O.make_tensor((n, 1, h, hd), 5, s)), torch.bfloat16) for s in (1, 2, 3))
    o_b, _ = U().FlashAttention("blocked", block_size=bs, pattern=O.full_block_pattern(n, bs)).forward_with_lse(q, k, v)
    o_d, _ = U().FlashAttention("none").forward_with_lse(q, k, v)
    assert rel_max_err(to_np(o_b), to_np(o_d)) <= 1e-2


def test_blocked_errors():
    E = U()
    x = torch.zeros((64, 1, 2, 128), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(E.DivisibilityError):
        E.FlashAttention("blocked", block_size=24, pattern={(0, 0)}).forward_with_lse(x, x, x)
    with pytest.raises(ValueError, match="out of range"):
        E.FlashAttention("blocked", block_size=32, pattern={(0, 0), (1, 2)}).forward_with_lse(x, x, x)
    with pytest.raises(E.DegenerateRowError):
        E.FlashAttention("blocked", block_size=32, pattern={(0, 0)}).forward_with_lse(x, x, x)
    with pytest.raises(E.KernelError):
        E.get_kernel("blocked")
    # forward only, like the reference (masked_attention_backward: dense/causal)
    attn = E.FlashAttention("blocked", block_size=32, pattern={(0, 0), (1, 1)})
    q = x.clone().requires_grad_(True)
    out = attn(q, x, x)
    with pytest.raises(E.KernelError):
        out.backward(torch.ones_like(out))
