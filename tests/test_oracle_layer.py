"""Pin the layer / block restatements (oracle/ulysses_oracle.py L4) bitwise
to the reference's run_ulysses_attention_backward and run_ulysses_blocks
(ulysses.py:264-307) -- tests/golden/layer.npz, made by oracle/gen_golden.py."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import ulysses_oracle as O


@pytest.mark.parametrize("ci", range(3))
def test_layer_forward_backward_bitwise(ci):
    g = np.load(os.path.join(GOLDEN, "layer.npz"))
    p, n, b, d, h, causal, seed = (int(x) for x in g[f"case{ci}_meta"])
    kind = "causal" if causal else "none"
    w = O.make_weights(d, seed)
    x, go = O.make_input(n, b, d, seed), O.make_input(n, b, d, seed + 1000)
    nl = n // p
    sh = lambda t: [t[r * nl:(r + 1) * nl] for r in range(p)]
    out, st = O.ulysses_attention_layer(sh(x), w, h, kind)
    gx, gw = O.ulysses_attention_layer_backward(sh(go), st, w, kind)
    assert np.array_equal(np.concatenate(out), g[f"case{ci}_out"])
    assert np.array_equal(np.concatenate(gx), g[f"case{ci}_gx"])
    for key in ("wq", "wk", "wv", "wo"):
        assert np.array_equal(gw[key], g[f"case{ci}_g{key}"])


def test_block_stack_bitwise():
    g = np.load(os.path.join(GOLDEN, "layer.npz"))
    p, n, b, d, h, layers, seed = (int(x) for x in g["blocks_meta"])
    x = O.make_input(n, b, d, seed)
    nl = n // p
    cur = [x[r * nl:(r + 1) * nl] for r in range(p)]
    for i in range(layers):
        cur = O.ulysses_block(cur, O.make_weights(d, seed, i), h, "causal")
    assert np.array_equal(np.concatenate(cur), g["blocks_out"])


def test_package_weights_match_reference_draws():
    # the torch-side make_weights draws the same numbers (layers.py:83-99)
    from paper_2309_14509_b200.layer import make_weights
    a, b = make_weights(32, 5, 1), O.make_weights(32, 5, 1)
    assert all(np.array_equal(a[k], b[k]) for k in b)


@pytest.mark.parametrize("ci", range(3))
def test_ring_attention_bitwise(ci):
    # the reference's ring baseline (baselines.py:68-121, run_ring_attention)
    g = np.load(os.path.join(GOLDEN, "layer.npz"))
    p, n, b, d, h, causal, seed = (int(x) for x in g[f"ring{ci}_meta"])
    x, w = O.make_input(n, b, d, seed), O.make_weights(d, seed)
    nl = n // p
    out = O.ring_attention_layer([x[r * nl:(r + 1) * nl] for r in range(p)], w, h, "causal" if causal else "none")
    assert np.array_equal(np.concatenate(out), g[f"ring{ci}_out"])
    # its ledger: 2 (P-1) ring shifts of the local (n/P, b, d) tensor, metered (P*local, local)
    led = g[f"ring{ci}_ledger"]
    assert len(led) == 2 * (p - 1)
    assert all(int(a) == p * nl * b * d and int(e) == nl * b * d for a, e in led)
