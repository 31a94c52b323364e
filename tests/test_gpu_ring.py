"""Ring attention (the ring half of a hybrid) and the
ring_shift collective on the B200, against the reference's ring baseline
(tests/golden/layer.npz: run_ring_attention, baselines.py:68-155) and the
oracle (simgroup.py:374-388 for ring_shift)."""

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


@pytest.mark.parametrize("p,steps", [(2, 1), (3, 1), (3, 2), (4, 0), (4, 5)])
def test_ring_shift_bitwise(p, steps):
    groups = U().SequenceGroup.local_group(p, slot_bytes=4 << 20)
    xs = [O.make_tensor((37, 3, 8), 90 + r, 1) for r in range(p)]
    ys = [O.make_tensor((129,), 90 + r, 2) for r in range(p)]
    ins = run_ranks(groups, lambda r: [to_dev(xs[r]), to_dev(ys[r], torch.bfloat16)])
    outs = run_ranks(groups, lambda r: groups[r].ring_shift(ins[r], steps, label="t"))
    ex, ey = O.ring_shift(xs, steps), O.ring_shift([O.bf16_round(y) for y in ys], steps)
    for r in range(p):
        assert np.array_equal(to_np(outs[r][0]), ex[r]) and np.array_equal(to_np(outs[r][1]), ey[r])
        rec = groups[r].ledger.select("ring_shift")
        assert rec[0].aggregate_elements == p * 37 * 3 * 8 and rec[0].per_rank_egress_elements == 37 * 3 * 8 * steps


class _LoopbackRing:
    """world-2 stand-in whose ring_shift returns its input: drives
    ring_attention_core through the merge path on one stream, so every
    kernel it launches is loaded before an in-process group runs (lazy
    module loading can block the host thread that still has to issue the
    peers' pushes)."""
    world, rank = 2, 1

    def ring_shift(self, tensors, steps=1, label="", labels=None):
        return [t.clone() for t in tensors]


def warm_ring_merge(n, b, h, hd, dtype):
    mk = lambda: torch.randn((n, b, h, hd), device="cuda").to(dtype)
    U().ring_attention_core(mk(), mk(), mk(), _LoopbackRing(), "causal")


def warm_ring_backward(n, b, h, hd, dtype):
    mk = lambda: torch.randn((n, b, h, hd), device="cuda").to(dtype).requires_grad_(True)
    q, k, v = mk(), mk(), mk()
    o = U().ring_attention_core(q, k, v, _LoopbackRing(), "causal")
    o.backward(torch.ones_like(o))


def run_ring(p, d, h, kind, x, w, dtype):
    n = x.shape[0]
    nl = n // p
    groups = U().SequenceGroup.local_group(p, slot_bytes=16 << 20) if p > 1 else [U().SequenceGroup.single()]
    warm_streams(groups)
    t = to_dev(x[:nl], dtype)   # load every library kernel of these shapes first
    U().RingAttention(d, h, None, kind, weights=w, dtype=dtype)(t)
    torch.cuda.synchronize()
    mods = run_ranks(groups, lambda r: U().RingAttention(d, h, groups[r], kind, weights=w, dtype=dtype))
    xs = run_ranks(groups, lambda r: to_dev(x[r * nl:(r + 1) * nl], dtype))
    outs = run_ranks(groups, lambda r: mods[r](xs[r]))
    return np.concatenate([to_np(o) for o in outs], 0), groups


@pytest.mark.parametrize("ci", range(3))
def test_ring_fp32_vs_reference(ci):
    g = np.load(os.path.join(GOLDEN, "layer.npz"))
    p, n, b, d, h, causal, seed = (int(x) for x in g[f"ring{ci}_meta"])
    out, groups = run_ring(p, d, h, "causal" if causal else "none", O.make_input(n, b, d, seed),
                           O.make_weights(d, seed), torch.float32)
    assert_rtol(out, g[f"ring{ci}_out"], rtol=LAYER_RTOL)
    nl = n // p
    for grp in groups:   # 2 (P-1) ring shifts of n/P*b*d elements, the reference's metering
        led = grp.ledger.select("ring_shift")
        assert len(led) == 2 * (p - 1)
        assert all(r.aggregate_elements == p * nl * b * d and r.per_rank_egress_elements == nl * b * d for r in led)


@pytest.mark.parametrize("p", [2, 4])
def test_ring_bf16_vs_oracle_and_ulysses(p):
    # hd 128 on the tcgen05 kernels; ring and Ulysses compute the same layer
    n, b, d, h, seed = 512, 1, 512, 4, 5
    w = {k: O.bf16_round(v) for k, v in O.make_weights(d, seed).items()}
    x = O.bf16_round(O.make_input(n, b, d, seed))
    out, _ = run_ring(p, d, h, "causal", x, w, torch.bfloat16)
    nl = n // p
    ref = np.concatenate(O.ring_attention_layer([x[r * nl:(r + 1) * nl] for r in range(p)], w, h, "causal",
                                                exact=False))
    assert rel_max_err(out, ref) <= BF16_MAXREL


def test_hybrid_ulysses_ring():
    # P = pu * pr ranks, ring-major, two sub-groups per rank; forward and
    # backward equal the plain attention layer's (oracle at P = 1).  Runs in
    # a child process with eager CUDA module loading: the ranks of an
    # in-process group are issued by one host thread, and a lazily loaded
    # kernel (first launch) can block that thread while an earlier rank's
    # stream spins in a flag wait.  Configs: 2x2 fp32, 2x2 bf16, 4x2 bf16.
    import json
    import subprocess
    import sys
    from conftest import ROOT
    env = dict(os.environ, CUDA_MODULE_LOADING="EAGER")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "hybrid_worker.py"), "2,2,float32",
                        "2,2,bfloat16", "4,2,bfloat16"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["ok"], res


@pytest.mark.parametrize("p,dtype", [(2, torch.float32), (3, torch.float32), (2, torch.bfloat16), (4, torch.bfloat16)])
def test_ring_backward_vs_oracle(p, dtype):
    # the ring layer's gradients equal the attention layer's (same function):
    # oracle = ulysses_attention_layer(_backward) at P = 1
    hd = 128 if dtype == torch.bfloat16 else 16
    h = 4
    d, b, seed = h * hd, 1, 8
    n = 96 * p
    nl = n // p
    w = {k: O.bf16_round(v) for k, v in O.make_weights(d, seed).items()}
    x, go = O.bf16_round(O.make_input(n, b, d, seed)), O.bf16_round(O.make_input(n, b, d, seed + 1))
    groups = U().SequenceGroup.local_group(p, slot_bytes=16 << 20)
    warm_streams(groups)
    t = to_dev(x[:nl], dtype).requires_grad_(True)   # single-rank pass: load every kernel first
    mod1 = U().RingAttention(d, h, None, "causal", weights=w, dtype=dtype)
    torch.autograd.backward([mod1(t)], [to_dev(go[:nl], dtype)])
    warm_ring_merge(nl, b, h, hd, dtype)
    warm_ring_backward(nl, b, h, hd, dtype)
    torch.cuda.synchronize()
    mods = run_ranks(groups, lambda r: U().RingAttention(d, h, groups[r], "causal", weights=w, dtype=dtype))
    xs = run_ranks(groups, lambda r: to_dev(x[r * nl:(r + 1) * nl], dtype).requires_grad_(True))
    gs = run_ranks(groups, lambda r: to_dev(go[r * nl:(r + 1) * nl], dtype))
    outs = run_ranks(groups, lambda r: mods[r](xs[r]))
    run_ranks(groups, lambda r: torch.autograd.backward([outs[r]], [gs[r]]))
    gx = np.concatenate([to_np(t.grad) for t in xs], 0)
    gw = {k: sum(to_np(getattr(m, k).grad) for m in mods) for k in ("wq", "wk", "wv", "wo")}
    ro, st = O.ulysses_attention_layer([x], w, h, "causal", exact=False)
    rgx, rgw = O.ulysses_attention_layer_backward([go], st, w, "causal", exact=False)
    if dtype == torch.float32:
        assert_rtol(gx, rgx[0], rtol=LAYER_RTOL)
        for key in gw:
            assert_rtol(gw[key], rgw[key], rtol=LAYER_RTOL)
    else:
        assert rel_max_err(gx, rgx[0]) <= BF16_MAXREL
        for key in gw:
            assert rel_max_err(gw[key], rgw[key]) <= BF16_MAXREL, key


def test_ring_shift_desync_is_error_not_hang():
    # mismatched payload sizes across ranks: the signature check fires (simgroup.py:265-276)
    groups = U().SequenceGroup.local_group(2, slot_bytes=1 << 20)
    for g in groups:
        g.set_timeout_ms(3000)
    ins = run_ranks(groups, lambda r: [torch.zeros(64 + 16 * r, device="cuda")])
    with pytest.raises(U().GroupDesyncError):
        run_ranks(groups, lambda r: groups[r].ring_shift(ins[r], 1))
