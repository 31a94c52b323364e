"""UlyssesAttention (projections + the Ulysses core) and UlyssesBlock on the
B200 against the reference (tests/golden/layer.npz: run_ulysses_attention_
backward / run_ulysses_blocks, ulysses.py:264-307) and the float64 oracle.
Tolerance of the whole layer in fp32 mode: |a - o| <= 1e-4 |o| + 1e-6 max(1, |o|)
(the projections are fp32 cuBLAS GEMMs around the 1e-5 attention core)."""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from helpers import BF16_MAXREL, assert_rtol, rel_max_err, run_ranks, to_dev, to_np, warm_streams
from oracle import ulysses_oracle as O

pytestmark = pytest.mark.gpu
LAYER_RTOL = 1e-4


def U():
    import paper_2309_14509_b200 as mod
    return mod


def run_layer(p, d, h, kind, x, go, w, dtype):
    n = x.shape[0]
    nl = n // p
    groups = U().SequenceGroup.local_group(p, slot_bytes=16 << 20) if p > 1 else [U().SequenceGroup.single()]
    warm_streams(groups)
    if p > 1:   # load every library kernel of these shapes first (lazy loading can block the host)
        run_layer(1, d, h, kind, x[:nl], go[:nl], w, dtype)
    mods = run_ranks(groups, lambda r: U().UlyssesAttention(d, h, groups[r], kind, weights=w, dtype=dtype))
    xs = run_ranks(groups, lambda r: to_dev(x[r * nl:(r + 1) * nl], dtype).requires_grad_(True))
    gs = run_ranks(groups, lambda r: to_dev(go[r * nl:(r + 1) * nl], dtype))
    outs = run_ranks(groups, lambda r: mods[r](xs[r]))
    run_ranks(groups, lambda r: torch.autograd.backward([outs[r]], [gs[r]]))
    out = np.concatenate([to_np(o) for o in outs], 0)
    gx = np.concatenate([to_np(t.grad) for t in xs], 0)
    gw = {k: sum(to_np(getattr(m, k).grad) for m in mods) for k in ("wq", "wk", "wv", "wo")}
    return out, gx, gw


@pytest.mark.parametrize("ci", range(3))
def test_layer_fp32_vs_reference(ci):
    g = np.load(os.path.join(GOLDEN, "layer.npz"))
    p, n, b, d, h, causal, seed = (int(x) for x in g[f"case{ci}_meta"])
    kind = "causal" if causal else "none"
    w = O.make_weights(d, seed)
    x, go = O.make_input(n, b, d, seed), O.make_input(n, b, d, seed + 1000)
    out, gx, gw = run_layer(p, d, h, kind, x, go, w, torch.float32)
    assert_rtol(out, g[f"case{ci}_out"], rtol=LAYER_RTOL)
    assert_rtol(gx, g[f"case{ci}_gx"], rtol=LAYER_RTOL)
    for key in ("wq", "wk", "wv", "wo"):
        assert_rtol(gw[key], g[f"case{ci}_g{key}"], rtol=LAYER_RTOL)


@pytest.mark.parametrize("p", [1, 2])
def test_layer_bf16_vs_oracle(p):
    n, b, d, h, seed = 512, 1, 256, 2, 31   # hd 128: the tcgen05 kernels
    w = {k: O.bf16_round(v) for k, v in O.make_weights(d, seed).items()}
    x, go = O.bf16_round(O.make_input(n, b, d, seed)), O.bf16_round(O.make_input(n, b, d, seed + 1))
    out, gx, gw = run_layer(p, d, h, "causal", x, go, w, torch.bfloat16)
    nl = n // p
    sh = lambda t: [t[r * nl:(r + 1) * nl] for r in range(p)]
    ro, st = O.ulysses_attention_layer(sh(x), w, h, "causal", exact=False)
    rgx, rgw = O.ulysses_attention_layer_backward(sh(go), st, w, "causal", exact=False)
    assert rel_max_err(out, np.concatenate(ro)) <= BF16_MAXREL
    assert rel_max_err(gx, np.concatenate(rgx)) <= BF16_MAXREL
    for key in ("wq", "wk", "wv", "wo"):
        assert rel_max_err(gw[key], rgw[key]) <= BF16_MAXREL, key


def test_block_stack_fp32_vs_reference():
    g = np.load(os.path.join(GOLDEN, "layer.npz"))
    p, n, b, d, h, layers, seed = (int(x) for x in g["blocks_meta"])
    x = O.make_input(n, b, d, seed)
    nl = n // p
    groups = U().SequenceGroup.local_group(p, slot_bytes=16 << 20)
    warm_streams(groups)
    warm = [U().UlyssesBlock(d, h, None, "causal", dtype=torch.float32, seed=seed, layer=i) for i in range(layers)]
    t = to_dev(x[:nl])
    for blk in warm:   # load every library kernel of these shapes first (lazy loading can block the host)
        t = blk(t)
    torch.cuda.synchronize()
    blocks = run_ranks(groups, lambda r: [U().UlyssesBlock(d, h, groups[r], "causal", dtype=torch.float32,
                                                            seed=seed, layer=i) for i in range(layers)])
    cur = run_ranks(groups, lambda r: to_dev(x[r * nl:(r + 1) * nl]))
    for i in range(layers):
        cur = run_ranks(groups, lambda r: blocks[r][i](cur[r]))
    assert_rtol(np.concatenate([to_np(c) for c in cur], 0), g["blocks_out"], rtol=LAYER_RTOL)


def test_layer_ledger_law_and_device_bytes():
    # verify.check_ledger's zero-tolerance law on the fused bf16 layer (P = 2,
    # fwd + bwd), and the device-side byte ledger agrees with the logical one
    p, n, b, d, h, seed = 2, 256, 1, 256, 2, 9
    w = {k: O.bf16_round(v) for k, v in O.make_weights(d, seed).items()}
    x, go = O.bf16_round(O.make_input(n, b, d, seed)), O.bf16_round(O.make_input(n, b, d, seed + 1))
    nl = n // p
    groups = U().SequenceGroup.local_group(p, slot_bytes=16 << 20)
    warm_streams(groups)
    run_layer(1, d, h, "causal", x[:nl], go[:nl], w, torch.bfloat16)
    mods = run_ranks(groups, lambda r: U().UlyssesAttention(d, h, groups[r], "causal", weights=w))
    xs = run_ranks(groups, lambda r: to_dev(x[r * nl:(r + 1) * nl], torch.bfloat16).requires_grad_(True))
    gs = run_ranks(groups, lambda r: to_dev(go[r * nl:(r + 1) * nl], torch.bfloat16))
    outs = run_ranks(groups, lambda r: mods[r](xs[r]))
    run_ranks(groups, lambda r: torch.autograd.backward([outs[r]], [gs[r]]))
    for g in groups:
        ok, measured, predicted = U().check_ledger(g.ledger, n, b, d, p, layers=1, backward=True)
        assert ok, (measured, predicted, g.ledger.rows())
        nat = g.native_ledger()
        assert nat["egress_bytes"] == 2 * g.ledger.total_egress()     # bf16
        assert nat["aggregate_bytes"] == 2 * g.ledger.total_aggregate()
        # counted on the device by each call's signalling CTA: the same bytes
        assert g.device_ledger() == nat
