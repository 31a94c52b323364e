"""The sampled-block backward oracles (used at BASELINE shapes on the GPU)
equal the same rows / columns of the full per-head backward
(kernels.py:89-111), which is itself pinned bitwise to the reference
goldens (test_oracle_golden.py)."""

import numpy as np
import pytest

from oracle import ulysses_oracle as O


@pytest.mark.parametrize("kind", ["causal", "none"])
def test_row_and_column_blocks_equal_full_backward(kind):
    n, hd, scale = 300, 16, 0.25
    q, k, v, d = (np.random.default_rng([9, i]).standard_normal((n, hd)) for i in range(4))
    dq, dk, dv = O.attention_head_backward(q[:, None], k[:, None], v[:, None], d[:, None], kind, scale)
    a = O.attention_head_backward_rows(q, k, v, d, kind, scale, (100, 170))
    assert np.abs(a - dq[100:170, 0]).max() <= 1e-12
    ctx, lse = O.attention_head(q[:, None], k[:, None], v[:, None], kind, scale)
    dot = (ctx[:, 0] * d).sum(axis=1)
    for extra in ({}, {"lse": lse[0], "dot": dot}):
        b, c = O.attention_head_backward_cols(q, k, v, d, kind, scale, (37, 101), chunk=64, **extra)
        assert np.abs(b - dk[37:101, 0]).max() <= 1e-12
        assert np.abs(c - dv[37:101, 0]).max() <= 1e-12
