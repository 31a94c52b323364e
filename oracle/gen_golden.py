"""Generate golden vectors from the UNMODIFIED reference (``seqlab``).

TEST INFRASTRUCTURE.  Runs only in the build container where
``/root/reference`` exists; the outputs are committed under
``tests/golden/`` so the GPU box (which has no reference tree) can use
them.  Every vector is produced by the reference's own functions:

  * ``RankGroup`` / ``RankContext.all_to_all``      simgroup.py:198-468
  * ``seq_to_head`` / ``head_to_seq``               ulysses.py:104-124
  * ``get_kernel`` (dense/causal)                   kernels.py:43-52,124-128
  * ``masked_attention_backward``                   kernels.py:89-111
  * ``blocked_kernel`` + ``Mask.blocked`` patterns   kernels.py:55-86, tensor.py:147-206

with the loop structure of ``ulysses_attention_forward_with_state``
(ulysses.py:144-154) and ``ulysses_attention_backward`` (ulysses.py:
213-226) but taking q/k/v as inputs instead of projecting x (the
DistributedAttention boundary).

Usage:  python oracle/gen_golden.py [--config1]
"""

from __future__ import annotations

import argparse
import hashlib
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)

from oracle.ulysses_oracle import make_tensor  # noqa: E402


def _ref():
    sys.path.insert(0, REF_SRC)
    import seqlab.kernels as K
    import seqlab.layers as L
    import seqlab.simgroup as G
    import seqlab.tensor as T
    import seqlab.ulysses as U
    return K, L, G, T, U


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]


def ref_a2a(p, locals_, split, concat, mode="lockstep"):
    _, _, G, _, _ = _ref()
    results, ledger = G.run_group(
        p, lambda ctx: ctx.all_to_all(locals_[ctx.rank], split, concat, label="golden"),
        mode=mode)
    rec = ledger.records[0]
    return results, rec.aggregate_elements, rec.per_rank_egress_elements


def gen_a2a():
    """Routing goldens at several P / axis pairs (float32 payloads)."""
    out = {}
    # the reference's own 2x2 block-transpose known answer (test_simgroup.py:143-151)
    res, _, _ = ref_a2a(2, [np.array([0.0, 1.0]), np.array([10.0, 11.0])], 0, 0)
    out["transpose2_r0"], out["transpose2_r1"] = res[0], res[1]
    cases = [
        # (p, per-rank shape, split, concat)
        (2, (4, 1, 4, 8), 2, 0),
        (4, (4, 2, 8, 4), 2, 0),
        (8, (2, 1, 8, 16), 2, 0),
        (2, (8, 1, 2, 8), 0, 2),
        (4, (16, 2, 2, 4), 0, 2),
        (8, (16, 1, 1, 16), 0, 2),
        (4, (8, 2, 8), 0, 1),        # generic 3-D case (test_simgroup.py:153-164 shape)
        (2, (4, 6, 4, 2), 1, 3),     # batch-first style axes
    ]
    for ci, (p, shape, split, concat) in enumerate(cases):
        locals_ = [make_tensor(shape, 900 + ci, r, "float32") for r in range(p)]
        res, agg, egress = ref_a2a(p, locals_, split, concat)
        out[f"case{ci}_meta"] = np.array([p, split, concat, agg, egress] + list(shape))
        for r in range(p):
            out[f"case{ci}_in{r}"] = locals_[r].astype(np.float32)
            out[f"case{ci}_out{r}"] = res[r].astype(np.float32)
            assert np.array_equal(res[r].astype(np.float32).astype(np.float64), res[r])
    np.savez_compressed(os.path.join(GOLDEN, "a2a.npz"), **out)
    print("a2a.npz", len(out), "arrays")


def ref_ulysses(p, n, b, h, hd, kind, seed, dtype="float32", with_backward=True):
    """Reference forward+backward of the DistributedAttention core."""
    K, L, G, T, U = _ref()
    d = h * hd
    mask = T.Mask.none() if kind == "none" else T.Mask.causal()
    spec = L.AttentionSpec(n=n, b=b, d=d, h_heads=h, mask=mask)
    kernel = K.get_kernel("dense" if kind == "none" else "causal")
    q = make_tensor((n, b, h, hd), seed, 1, dtype)
    k = make_tensor((n, b, h, hd), seed, 2, dtype)
    v = make_tensor((n, b, h, hd), seed, 3, dtype)
    do = make_tensor((n, b, h, hd), seed, 4, dtype)
    nl = n // p

    def shard(x, r):
        return U.ShardedTensor(rank=r, layout=U.SEQUENCE,
                               data=T.Tensor3(x[r * nl:(r + 1) * nl].reshape(nl, b, d)))

    def program(ctx):
        r = ctx.rank
        q4 = U.seq_to_head(shard(q, r), spec, ctx, "attn.q.seq2head").data.data
        k4 = U.seq_to_head(shard(k, r), spec, ctx, "attn.k.seq2head").data.data
        v4 = U.seq_to_head(shard(v, r), spec, ctx, "attn.v.seq2head").data.data
        ctx4 = np.empty_like(q4)
        for hh in range(q4.shape[2]):                              # ulysses.py:149-152
            ctx4[:, :, hh, :] = kernel(q4[:, :, hh, :], k4[:, :, hh, :], v4[:, :, hh, :],
                                       spec.mask, spec.scale)
        o = U.head_to_seq(U.ShardedTensor(rank=r, layout=U.HEAD, data=T.Tensor4(ctx4)),
                          spec, ctx, "attn.ctx.head2seq").data.data
        if not with_backward:
            return o, None, None, None
        dctx4 = U.seq_to_head(shard(do, r), spec, ctx, "bwd.ctx.seq2head").data.data
        dq4, dk4, dv4 = (np.empty_like(dctx4) for _ in range(3))
        for hh in range(dctx4.shape[2]):                           # ulysses.py:218-222
            dq4[:, :, hh, :], dk4[:, :, hh, :], dv4[:, :, hh, :] = K.masked_attention_backward(
                q4[:, :, hh, :], k4[:, :, hh, :], v4[:, :, hh, :], dctx4[:, :, hh, :],
                spec.mask, spec.scale)
        dq = ctx.all_to_all(dq4, 0, 2, "bwd.q.head2seq")           # ulysses.py:224-226
        dk = ctx.all_to_all(dk4, 0, 2, "bwd.k.head2seq")
        dv = ctx.all_to_all(dv4, 0, 2, "bwd.v.head2seq")
        return o, dq, dk, dv

    results, ledger = G.run_group(p, program, mode="concurrent")
    cat = lambda i: np.concatenate([np.asarray(r[i]).reshape(nl, b, h, hd) for r in results], 0)
    o = cat(0)
    grads = (cat(1), cat(2), cat(3)) if with_backward else None
    return (q, k, v, do), o, grads, ledger


def gen_attn_small():
    out = {}
    for ci, (p, n, b, h, hd, kind) in enumerate([
        (2, 64, 1, 4, 16, "none"),
        (2, 64, 1, 4, 16, "causal"),
        (4, 32, 2, 4, 8, "causal"),
        (1, 48, 1, 2, 32, "causal"),
    ]):
        seed = 4000 + ci
        (q, k, v, do), o, (dq, dk, dv), ledger = ref_ulysses(p, n, b, h, hd, kind, seed)
        out[f"case{ci}_meta"] = np.array([p, n, b, h, hd, 0 if kind == "none" else 1, seed])
        out[f"case{ci}_ledger"] = np.array(
            [[r.aggregate_elements, r.per_rank_egress_elements] for r in ledger.records])
        for name, arr in (("q", q), ("k", k), ("v", v), ("do", do)):
            out[f"case{ci}_{name}"] = arr.astype(np.float32)
        for name, arr in (("o", o), ("dq", dq), ("dk", dk), ("dv", dv)):
            out[f"case{ci}_{name}"] = arr                          # float64 reference output
    np.savez_compressed(os.path.join(GOLDEN, "attn_small.npz"), **out)
    print("attn_small.npz", len(out), "arrays")


def gen_config1():
    """BASELINE config 1: P=2, N=1024, 8 heads x 64, fp32 -- dense and causal
    forward, causal backward.  Inputs are regenerated from the seed (their
    digest is stored); outputs are stored for every 16th sequence row."""
    out = {}
    p, n, b, h, hd, seed = 2, 1024, 1, 8, 64, 2024
    rows = np.arange(0, n, 16)
    for kind in ("none", "causal"):
        (q, k, v, do), o, grads, ledger = ref_ulysses(
            p, n, b, h, hd, kind, seed, with_backward=(kind == "causal"))
        out["inputs_digest"] = np.frombuffer(digest(q, k, v, do).encode(), dtype=np.uint8)
        out[f"{kind}_o_rows"] = o[rows]
        if grads is not None:
            for name, g in zip(("dq", "dk", "dv"), grads):
                out[f"{kind}_{name}_rows"] = g[rows]
        out[f"{kind}_ledger"] = np.array(
            [[r.aggregate_elements, r.per_rank_egress_elements] for r in ledger.records])
    out["rows"] = rows
    out["meta"] = np.array([p, n, b, h, hd, seed])
    np.savez_compressed(os.path.join(GOLDEN, "config1.npz"), **out)
    print("config1.npz", len(out), "arrays")


def gen_blocked():
    """Blocked-sparse forward through the Ulysses core with the reference's
    ``blocked_kernel`` (kernels.py:55-86) and ``Mask.blocked`` patterns from
    tensor.py:183-206 (plus one irregular pattern)."""
    K, L, G, T, U = _ref()
    out = {}
    rng = np.random.default_rng([2024, 7])
    cases = [
        (2, 64, 1, 4, 16, 8, "causal"),
        (1, 48, 2, 2, 32, 16, "banded"),
        (2, 128, 1, 2, 64, 32, "irregular"),
        (1, 256, 1, 2, 128, 64, "full"),
    ]
    for ci, (p, n, b, h, hd, bs, kind) in enumerate(cases):
        nb = n // bs
        if kind == "causal":
            pattern = T.causal_block_pattern(n, bs)
        elif kind == "banded":
            pattern = T.banded_block_pattern(n, bs, bandwidth=1)
        elif kind == "full":
            pattern = T.full_block_pattern(n, bs)
        else:   # every query block sees itself plus a random subset
            pattern = frozenset({(qb, qb) for qb in range(nb)} |
                                {(qb, kb) for qb in range(nb) for kb in range(nb) if rng.random() < 0.3})
        seed = 5000 + ci
        d = h * hd
        mask = T.Mask.blocked(bs, pattern)
        spec = L.AttentionSpec(n=n, b=b, d=d, h_heads=h, mask=mask)
        kernel = K.get_kernel("blocked")
        q = make_tensor((n, b, h, hd), seed, 1)
        k = make_tensor((n, b, h, hd), seed, 2)
        v = make_tensor((n, b, h, hd), seed, 3)
        nl = n // p

        def shard(x, r):
            return U.ShardedTensor(rank=r, layout=U.SEQUENCE,
                                   data=T.Tensor3(x[r * nl:(r + 1) * nl].reshape(nl, b, d)))

        def program(ctx):
            r = ctx.rank
            q4 = U.seq_to_head(shard(q, r), spec, ctx, "attn.q.seq2head").data.data
            k4 = U.seq_to_head(shard(k, r), spec, ctx, "attn.k.seq2head").data.data
            v4 = U.seq_to_head(shard(v, r), spec, ctx, "attn.v.seq2head").data.data
            ctx4 = np.empty_like(q4)
            for hh in range(q4.shape[2]):                              # ulysses.py:149-152
                ctx4[:, :, hh, :] = kernel(q4[:, :, hh, :], k4[:, :, hh, :], v4[:, :, hh, :],
                                           spec.mask, spec.scale)
            return U.head_to_seq(U.ShardedTensor(rank=r, layout=U.HEAD, data=T.Tensor4(ctx4)),
                                 spec, ctx, "attn.ctx.head2seq").data.data

        results, _ = G.run_group(p, program, mode="concurrent")
        o = np.concatenate([np.asarray(x).reshape(nl, b, h, hd) for x in results], 0)
        out[f"case{ci}_meta"] = np.array([p, n, b, h, hd, bs, seed])
        out[f"case{ci}_pattern"] = np.array(sorted(pattern), dtype=np.int64)
        for name, arr in (("q", q), ("k", k), ("v", v)):
            out[f"case{ci}_{name}"] = arr.astype(np.float32)
        out[f"case{ci}_o"] = o
    np.savez_compressed(os.path.join(GOLDEN, "blocked.npz"), **out)
    print("blocked.npz", len(out), "arrays")


def gen_layer():
    """The full attention layer with projections (run_ulysses_attention_backward,
    ulysses.py:281-307) and a 2-block stack (run_ulysses_blocks, ulysses.py:
    264-278) from the reference, fp64, seeded inputs and weights."""
    K, L, G, T, U = _ref()
    out = {}
    for ci, (p, n, b, d, h, kind, seed) in enumerate([
        (2, 32, 1, 64, 4, "causal", 11),
        (1, 24, 2, 48, 3, "none", 12),
        (4, 32, 1, 64, 4, "causal", 13),
    ]):
        mask = T.Mask.causal() if kind == "causal" else T.Mask.none()
        spec = L.AttentionSpec(n=n, b=b, d=d, h_heads=h, mask=mask)
        kname = "causal" if kind == "causal" else "dense"
        w = L.make_weights(d, seed)
        x = L.make_input(n, b, d, seed)
        gout = L.make_input(n, b, d, seed + 1000)
        o, gx, gw, _ = U.run_ulysses_attention_backward(x, gout, w, spec, kname, p)
        out[f"case{ci}_meta"] = np.array([p, n, b, d, h, 1 if kind == "causal" else 0, seed])
        out[f"case{ci}_out"] = np.asarray(o.data)
        out[f"case{ci}_gx"] = np.asarray(gx.data)
        for key in ("wq", "wk", "wv", "wo"):
            out[f"case{ci}_g{key}"] = gw[key]
    # two blocks, P = 2
    p, n, b, d, h, seed = 2, 32, 1, 64, 4, 21
    spec = L.AttentionSpec(n=n, b=b, d=d, h_heads=h, mask=T.Mask.causal())
    ws = [L.make_weights(d, seed, layer=i) for i in range(2)]
    x = L.make_input(n, b, d, seed)
    y, _ = U.run_ulysses_blocks(x, ws, spec, "causal", p)
    out["blocks_meta"] = np.array([p, n, b, d, h, 2, seed])
    out["blocks_out"] = np.asarray(y.data)
    # the reference's ring baseline (baselines.py:68-121, run_ring_attention :142-155)
    import seqlab.baselines as B
    for ci, (p, n, b, d, h, kind, seed) in enumerate([(2, 32, 1, 64, 4, "causal", 31),
                                                       (4, 32, 1, 64, 4, "causal", 32),
                                                       (2, 24, 2, 48, 4, "none", 33)]):
        mask = T.Mask.causal() if kind == "causal" else T.Mask.none()
        spec = L.AttentionSpec(n=n, b=b, d=d, h_heads=h, mask=mask)
        y, led = B.run_ring_attention(L.make_input(n, b, d, seed), [L.make_weights(d, seed)], spec, p)
        out[f"ring{ci}_meta"] = np.array([p, n, b, d, h, 1 if kind == "causal" else 0, seed])
        out[f"ring{ci}_out"] = np.asarray(y.data)
        out[f"ring{ci}_ledger"] = np.array([[r.aggregate_elements, r.per_rank_egress_elements]
                                            for r in led.records])
    np.savez_compressed(os.path.join(GOLDEN, "layer.npz"), **out)
    print("layer.npz", len(out), "arrays")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config1", action="store_true")
    args = ap.parse_args()
    os.makedirs(GOLDEN, exist_ok=True)
    gen_a2a()
    gen_attn_small()
    gen_blocked()
    gen_layer()
    if args.config1:
        gen_config1()
