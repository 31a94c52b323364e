"""Pin the blocked-sparse restatement (oracle/ulysses_oracle.py L2b) to the
reference: the Ulysses core run with the reference's own ``blocked_kernel``
(kernels.py:55-86) on ``Mask.blocked`` patterns (tensor.py:147-206) --
tests/golden/blocked.npz, made by oracle/gen_golden.py -- and to the
reference's blocked known answers (test_kernels.py:42-59: the blocked kernel
with the full / block-causal pattern equals the dense / block-causal masked
kernel)."""

import math
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import ulysses_oracle as O


def load(name):
    return np.load(os.path.join(GOLDEN, name))


@pytest.mark.parametrize("ci", range(4))
def test_blocked_golden_bitwise(ci):
    g = load("blocked.npz")
    p, n, b, h, hd, bs, seed = (int(x) for x in g[f"case{ci}_meta"])
    pattern = frozenset(tuple(int(v) for v in row) for row in g[f"case{ci}_pattern"])
    q, k, v = (g[f"case{ci}_{t}"].astype(np.float64) for t in ("q", "k", "v"))
    assert np.array_equal(q, O.make_tensor((n, b, h, hd), seed, 1))
    # the seq->head / head->seq exchanges are exact moves, so the Ulysses
    # result equals the per-head kernel on the full sequence, bitwise
    ctx, _ = O.local_attention_blocked(q, k, v, bs, pattern)
    assert np.array_equal(ctx, g[f"case{ci}_o"])


def test_full_pattern_equals_dense_and_block_causal():
    n, b, hd, bs = 32, 1, 8, 8
    q, k, v = (O.make_tensor((n, b, hd), 9, s) for s in (1, 2, 3))
    scale = 1 / math.sqrt(hd)
    dense, _ = O.attention_head(q, k, v, "none", scale)
    full, _ = O.blocked_attention_head(q, k, v, bs, O.full_block_pattern(n, bs), scale)
    assert np.allclose(full, dense, rtol=0, atol=1e-12)
    # block-causal = dense with the blocked visibility mask
    vis = O.blocked_visibility(bs, O.causal_block_pattern(n, bs), n, n)
    s = O.matmul(q[:, 0], k[:, 0].T) * scale
    pr = np.where(vis, np.exp(s - np.where(vis, s, -np.inf).max(1, keepdims=True)), 0)
    ref = (pr / pr.sum(1, keepdims=True)) @ v[:, 0]
    bc, lse = O.blocked_attention_head(q, k, v, bs, O.causal_block_pattern(n, bs), scale)
    assert np.allclose(bc[:, 0], ref, rtol=0, atol=1e-12)
    # LSE restatement: log of the row normaliser over the visible scores
    m = np.where(vis, s, -np.inf).max(1)
    assert np.allclose(lse[0], m + np.log(np.where(vis, np.exp(s - m[:, None]), 0).sum(1)), atol=1e-12)


def test_pattern_helpers():
    assert O.causal_block_pattern(8, 4) == {(0, 0), (1, 0), (1, 1)}
    assert O.banded_block_pattern(12, 4, 1) == {(0, 0), (1, 0), (1, 1), (2, 1), (2, 2)}
    assert len(O.full_block_pattern(8, 2)) == 16
    bits = O.pattern_bits(64 * 40, 64, {(0, 0), (1, 33), (39, 39)})
    assert bits.shape == (40, 2) and bits[0, 0] == 1 and bits[1, 1] == 2 and bits[39, 1] == 1 << 7


def test_blocked_errors_in_reference_order():
    q = O.make_tensor((16, 1, 4), 1, 1)
    with pytest.raises(O.DivisibilityError):
        O.blocked_attention_head(q, q, q, 5, {(0, 0)}, 0.5)          # kernels.py:69-70
    with pytest.raises(ValueError, match="out of range"):
        O.blocked_attention_head(q, q, q, 4, {(0, 4)}, 0.5)          # kernels.py:72-74
    with pytest.raises(O.DegenerateRowError):
        O.blocked_attention_head(q, q, q, 4, {(0, 0), (1, 1), (3, 3)}, 0.5)   # kernels.py:83-85
