"""Float64 NumPy restatement of the reference's Ulysses attention path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Every function cites
the reference line range it restates; paths are relative to
``/root/reference/pkg/src/seqlab``.  Layout is the reference's
sequence-major ``[s, b, h, hd]`` (ulysses.py:47-48).

Two arithmetic modes:
  * ``exact=True`` (default) uses the reference's fixed left-to-right
    ``matmul`` (tensor.py:209-224) so results are bitwise equal to the
    reference.  Cost is the reference's: O(N^2*hd) numpy passes.
  * ``exact=False`` uses BLAS ``np.matmul`` in float64 for the larger
    parity cases; tests pin it to the exact mode at <=1e-12.
"""

from __future__ import annotations

import math
from fractions import Fraction

import numpy as np


class ShardError(ValueError):
    """simgroup.py:62-63."""


class DivisibilityError(ValueError):
    """tensor.py:27-28."""


class DegenerateRowError(ValueError):
    """tensor.py:31-32."""


class KernelError(ValueError):
    """kernels.py:22-23."""


# ---------------------------------------------------------------------------
# L1: the collective
# ---------------------------------------------------------------------------

def all_to_all(locals_, split_axis: int, concat_axis: int):
    """Rank-ordered all-to-all of ``locals_`` (one array per rank).

    Restates ``RankGroup._all_to_all`` (simgroup.py:313-335): every rank's
    operand is split into ``p`` equal chunks along ``split_axis``; rank ``i``
    receives chunk ``i`` of every rank, concatenated in source-rank order
    along ``concat_axis`` (``combine``, simgroup.py:322-327).  Divisibility
    failure raises ShardError (simgroup.py:315-319).  Dtype is preserved
    (the reference upcasts to f64, simgroup.py:308-311, which is exact for
    f32/bf16 payloads, so routing is bitwise either way).
    """
    p = len(locals_)
    arrs = [np.asarray(a) for a in locals_]
    shape = arrs[0].shape
    if shape[split_axis] % p != 0:
        raise ShardError(
            f"all_to_all split axis {split_axis} (length {shape[split_axis]}) "
            f"not divisible by p={p}")
    chunks = [np.split(a, p, axis=split_axis) for a in arrs]
    return [np.concatenate([chunks[j][i] for j in range(p)], axis=concat_axis)
            for i in range(p)]


def all_to_all_metering(local_elements: int, p: int) -> tuple[int, int]:
    """(aggregate, per-rank egress) elements, simgroup.py:329-332."""
    chunk = local_elements // p
    return p * local_elements, chunk * (p - 1)


def ulysses_volume(n: int, b: int, h: int, p: int, convention: str = "exact") -> Fraction:
    """Per-link a2a volume of one layer's forward, costmodel.py:82-87.

    ``h`` here is the hidden size d (the reference's CostInputs.h)."""
    m = Fraction(4 * n * b * h)
    if convention == "paper_asymptotic":
        return m / p
    return m * (p - 1) / (p * p)


def seq_to_head(seq_locals, h: int):
    """(n/P, b, h, hd) sequence shards -> (n, b, h/P, hd) head shards.

    ulysses.py:104-111 and ``_to_head`` ulysses.py:161-164:
    ``all_to_all(split_axis=2, concat_axis=0)``.  Accepts 3-D (n/P, b, d)
    shards (reshaped like ulysses.py:109) or 4-D shards.
    """
    four = []
    for x in seq_locals:
        x = np.asarray(x)
        if x.ndim == 3:
            x = x.reshape(x.shape[0], x.shape[1], h, x.shape[2] // h)
        four.append(x)
    p = len(four)
    if h % p != 0:
        raise DivisibilityError(f"p={p} does not divide head count {h}")
    return all_to_all(four, split_axis=2, concat_axis=0)


def head_to_seq(head_locals):
    """Exact inverse: ``all_to_all(split_axis=0, concat_axis=2)``.

    ulysses.py:114-124 / ``_to_seq`` ulysses.py:167-169 (returns 4-D; the
    reference then reshapes to (n/P, b, d))."""
    return all_to_all(head_locals, split_axis=0, concat_axis=2)


# ---------------------------------------------------------------------------
# L0: numeric core
# ---------------------------------------------------------------------------

def matmul(a, bm, exact: bool = True) -> np.ndarray:
    """tensor.py:209-224: fixed left-to-right accumulation over k."""
    a = np.asarray(a, dtype=np.float64)
    bm = np.asarray(bm, dtype=np.float64)
    if a.ndim != 2 or bm.ndim != 2 or a.shape[1] != bm.shape[0]:
        raise ValueError(f"matmul shapes {a.shape} x {bm.shape}")
    if not exact:
        return a @ bm
    out = np.zeros((a.shape[0], bm.shape[1]), dtype=np.float64)
    for k in range(a.shape[1]):
        out += a[:, k, None] * bm[None, k, :]
    return out


def visibility(kind: str, rows: int, cols: int, row_offset: int = 0) -> np.ndarray:
    """Mask.visibility for 'none'/'causal' (tensor.py:151-162)."""
    if kind == "none":
        return np.ones((rows, cols), dtype=bool)
    if kind != "causal":
        raise KernelError(f"mask kind {kind!r} not on this path")
    qidx = np.arange(row_offset, row_offset + rows)
    kidx = np.arange(cols)
    return kidx[None, :] <= qidx[:, None]


def row_softmax(scores, kind: str, row_offset: int = 0) -> np.ndarray:
    """tensor.py:227-249: masked, row-max stabilised softmax; masked -> 0."""
    scores = np.asarray(scores, dtype=np.float64)
    vis = visibility(kind, scores.shape[0], scores.shape[1], row_offset)
    counts = vis.sum(axis=1)
    if np.any(counts == 0):
        row = int(np.argmax(counts == 0))
        raise DegenerateRowError(
            f"row {row_offset + row} has zero unmasked entries (mask kind {kind!r})")
    shifted = np.where(vis, scores, -np.inf)
    rowmax = shifted.max(axis=1, keepdims=True)
    expd = np.where(vis, np.exp(np.where(vis, scores - rowmax, 0.0)), 0.0)
    return expd / expd.sum(axis=1, keepdims=True)


def row_lse(scores, kind: str, row_offset: int = 0) -> np.ndarray:
    """RESTATEMENT (no reference counterpart): natural-log LSE of the rows
    ``row_softmax`` normalises, i.e. ``rowmax + log(sum(exp(s - rowmax)))``
    over visible entries (same terms as tensor.py:245-249)."""
    scores = np.asarray(scores, dtype=np.float64)
    vis = visibility(kind, scores.shape[0], scores.shape[1], row_offset)
    shifted = np.where(vis, scores, -np.inf)
    rowmax = shifted.max(axis=1)
    expd = np.where(vis, np.exp(np.where(vis, scores - rowmax[:, None], 0.0)), 0.0)
    return rowmax + np.log(expd.sum(axis=1))


# ---------------------------------------------------------------------------
# L2: the local-attention plugin (per head)
# ---------------------------------------------------------------------------

def _check_kind(kind: str):
    if kind not in ("none", "causal"):
        raise KernelError(f"kernel supports dense/causal masks only, got {kind!r}")


def attention_head(q, k, v, kind: str, scale: float, exact: bool = True,
                   rows: tuple[int, int] | None = None):
    """Per-head context and LSE for (n, b, hd) views.

    ``_masked_attention`` kernels.py:31-40 (dense_kernel :43-46,
    causal_kernel :49-52): scores = matmul(q, k^T) * scale; row_softmax;
    ctx = matmul(probs, v).  ``rows=(r0, r1)`` evaluates only query rows
    [r0, r1) with ``row_offset=r0`` (the reference's chunked-causal
    convention, tensor.py:151-156, used by baselines.py:104).
    Returns (ctx (r, b, hd), lse (b, r)).
    """
    _check_kind(kind)
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    n, b, hd = q.shape
    r0, r1 = (0, n) if rows is None else rows
    ctx = np.empty((r1 - r0, b, hd))
    lse = np.empty((b, r1 - r0))
    for bi in range(b):
        scores = matmul(q[r0:r1, bi, :], k[:, bi, :].T, exact) * scale
        probs = row_softmax(scores, kind, row_offset=r0)
        ctx[:, bi, :] = matmul(probs, v[:, bi, :], exact)
        lse[bi] = row_lse(scores, kind, row_offset=r0)
    return ctx, lse


def attention_head_backward(q, k, v, dctx, kind: str, scale: float, exact: bool = True):
    """kernels.py:89-111 ``masked_attention_backward``: recompute probs,
    dprobs = dctx v^T, dot = rowsum(dprobs*probs), dscores =
    probs*(dprobs-dot)*scale, dq = dscores k, dk = dscores^T q,
    dv = probs^T dctx."""
    _check_kind(kind)
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    dctx = np.asarray(dctx, dtype=np.float64)
    n, b, hd = q.shape
    dq = np.empty_like(q)
    dk = np.empty_like(k)
    dv = np.empty_like(v)
    for bi in range(b):
        q2, k2, v2, d2 = q[:, bi, :], k[:, bi, :], v[:, bi, :], dctx[:, bi, :]
        probs = row_softmax(matmul(q2, k2.T, exact) * scale, kind, row_offset=0)
        dprobs = matmul(d2, v2.T, exact)
        dot = (dprobs * probs).sum(axis=1, keepdims=True)
        dscores = probs * (dprobs - dot) * scale
        dq[:, bi, :] = matmul(dscores, k2, exact)
        dk[:, bi, :] = matmul(dscores.T, q2, exact)
        dv[:, bi, :] = matmul(probs.T, d2, exact)
    return dq, dk, dv


def attention_head_backward_rows(q, k, v, dctx, kind: str, scale: float, rows: tuple[int, int]):
    """dq of query rows [r0, r1) only: kernels.py:89-111 restricted to those
    rows with the reference's row_offset convention (tensor.py:151-156,
    227-249) -- each row's probabilities, dprobs, dot and dscores depend on
    that row alone, so the block equals the same rows of the full result.
    q, k, v, dctx: (n, hd) of ONE batch entry.  BLAS float64."""
    _check_kind(kind)
    r0, r1 = rows
    q = np.asarray(q[r0:r1], dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    d2 = np.asarray(dctx[r0:r1], dtype=np.float64)
    probs = row_softmax((q @ k.T) * scale, kind, row_offset=r0)
    dprobs = d2 @ v.T
    dot = (dprobs * probs).sum(axis=1, keepdims=True)
    dscores = probs * (dprobs - dot) * scale
    return dscores @ k


def attention_head_backward_cols(q, k, v, dctx, kind: str, scale: float, cols: tuple[int, int],
                                 lse=None, dot=None, chunk: int = 2048):
    """dk, dv of key rows [c0, c1) only (kernels.py:89-111: dk = dscores^T q,
    dv = probs^T dctx, restricted to those columns of probs / dscores).

    Every query row that sees a key in the block contributes (causal: rows
    i >= c0).  A row's probabilities need its full-row normaliser and its
    dot = rowsum(dprobs * probs); both are computed here from the row's full
    scores (exact, costs O(rows * n * hd)) unless given as ``lse`` /
    ``dot`` arrays over all n rows (natural-log LSE; dot == rowsum(dctx *
    ctx)), in which case only the block's columns are evaluated.  Query rows
    are processed in chunks.  q, k, v, dctx: (n, hd) of ONE batch entry."""
    _check_kind(kind)
    c0, c1 = cols
    n = q.shape[0]
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    kb, vb = k[c0:c1], v[c0:c1]
    dk = np.zeros((c1 - c0, q.shape[1]))
    dv = np.zeros((c1 - c0, v.shape[1]))
    start = c0 if kind == "causal" else 0
    for i0 in range(start, n, chunk):
        i1 = min(n, i0 + chunk)
        qi = np.asarray(q[i0:i1], dtype=np.float64)
        di = np.asarray(dctx[i0:i1], dtype=np.float64)
        if lse is None or dot is None:
            s_full = (qi @ k.T) * scale
            vis = visibility(kind, i1 - i0, n, row_offset=i0)
            shifted = np.where(vis, s_full, -np.inf)
            mx = shifted.max(axis=1, keepdims=True)
            e = np.where(vis, np.exp(np.where(vis, s_full - mx, 0.0)), 0.0)
            probs_full = e / e.sum(axis=1, keepdims=True)
            dprobs_full = di @ v.T
            row_dot = (dprobs_full * probs_full).sum(axis=1, keepdims=True)
            pb = probs_full[:, c0:c1]
            dpb = dprobs_full[:, c0:c1]
        else:
            sb = (qi @ kb.T) * scale
            vis = visibility(kind, i1 - i0, n, row_offset=i0)[:, c0:c1]
            pb = np.where(vis, np.exp(np.where(vis, sb - np.asarray(lse[i0:i1])[:, None], 0.0)), 0.0)
            dpb = di @ vb.T
            row_dot = np.asarray(dot[i0:i1])[:, None]
        dsb = pb * (dpb - row_dot) * scale
        dk += dsb.T @ qi
        dv += pb.T @ di
    return dk, dv


def kv_head_for(h: int, hq: int, hkv: int) -> int:
    """GQA RESTATEMENT: query head h reads kv head h // (hq/hkv)."""
    if hq % hkv != 0:
        raise DivisibilityError(f"kv heads {hkv} do not divide query heads {hq}")
    return h // (hq // hkv)


def local_attention(q4, k4, v4, kind: str, scale: float | None = None,
                    exact: bool = True, rows=None):
    """Head loop of ulysses.py:148-152 over (n, b, Hq, hd) q4 and
    (n, b, Hkv, hd) k4/v4 (GQA restatement; Hkv == Hq is the reference).
    Returns (ctx4 (r, b, Hq, hd), lse (b, Hq, r))."""
    q4 = np.asarray(q4)
    n, b, hq, hd = q4.shape
    hkv = np.asarray(k4).shape[2]
    if scale is None:
        scale = 1.0 / math.sqrt(hd)      # layers.py:51
    r0, r1 = (0, n) if rows is None else rows
    ctx4 = np.empty((r1 - r0, b, hq, hd))
    lse = np.empty((b, hq, r1 - r0))
    for hh in range(hq):
        g = kv_head_for(hh, hq, hkv)
        c, l = attention_head(q4[:, :, hh, :], k4[:, :, g, :], v4[:, :, g, :],
                              kind, scale, exact, rows)
        ctx4[:, :, hh, :] = c
        lse[:, hh, :] = l
    return ctx4, lse


def local_attention_backward(q4, k4, v4, dctx4, kind: str, scale: float | None = None,
                             exact: bool = True):
    """Head loop of ulysses.py:218-222; GQA dK/dV summed over each kv
    head's query group in ascending head order (restatement)."""
    q4 = np.asarray(q4)
    n, b, hq, hd = q4.shape
    hkv = np.asarray(k4).shape[2]
    if scale is None:
        scale = 1.0 / math.sqrt(hd)
    dq4 = np.empty((n, b, hq, hd))
    dk4 = np.zeros((n, b, hkv, hd))
    dv4 = np.zeros((n, b, hkv, hd))
    for hh in range(hq):
        g = kv_head_for(hh, hq, hkv)
        dq, dk, dv = attention_head_backward(q4[:, :, hh, :], k4[:, :, g, :], v4[:, :, g, :],
                                             dctx4[:, :, hh, :], kind, scale, exact)
        dq4[:, :, hh, :] = dq
        dk4[:, :, g, :] += dk
        dv4[:, :, g, :] += dv
    return dq4, dk4, dv4


def local_lse(q4, k4, kind, scale=None, exact=False):
    """LSE only (b, Hq, n) -- convenience for the backward parity tests."""
    q4 = np.asarray(q4, dtype=np.float64)
    n, b, hq, hd = q4.shape
    hkv = np.asarray(k4).shape[2]
    if scale is None:
        scale = 1.0 / math.sqrt(hd)
    out = np.empty((b, hq, n))
    for hh in range(hq):
        g = kv_head_for(hh, hq, hkv)
        for bi in range(b):
            s = matmul(q4[:, bi, hh, :], np.asarray(k4, np.float64)[:, bi, g, :].T, exact) * scale
            out[bi, hh] = row_lse(s, kind)
    return out


# ---------------------------------------------------------------------------
# L2b: blocked-sparse local attention
# ---------------------------------------------------------------------------

def causal_block_pattern(n: int, block_size: int) -> frozenset:
    """tensor.py:183-189: (qb, kb) for all kb <= qb."""
    if n % block_size != 0:
        raise DivisibilityError(f"block_size {block_size} does not divide n={n}")
    nb = n // block_size
    return frozenset((q, k) for q in range(nb) for k in range(q + 1))


def full_block_pattern(n: int, block_size: int) -> frozenset:
    """tensor.py:192-197: every (qb, kb) pair."""
    if n % block_size != 0:
        raise DivisibilityError(f"block_size {block_size} does not divide n={n}")
    nb = n // block_size
    return frozenset((q, k) for q in range(nb) for k in range(nb))


def banded_block_pattern(n: int, block_size: int, bandwidth: int = 1) -> frozenset:
    """tensor.py:200-206: causal local window, kb in [qb - bandwidth, qb]."""
    if n % block_size != 0:
        raise DivisibilityError(f"block_size {block_size} does not divide n={n}")
    nb = n // block_size
    return frozenset((q, k) for q in range(nb) for k in range(max(0, q - bandwidth), q + 1))


def blocked_visibility(block_size: int, pattern, rows: int, cols: int, row_offset: int = 0) -> np.ndarray:
    """Mask.visibility for kind 'blocked' (tensor.py:163-180)."""
    bs = block_size
    if cols % bs != 0:
        raise DivisibilityError(f"block_size {bs} does not divide key length {cols}")
    if rows % bs != 0 or row_offset % bs != 0:
        raise DivisibilityError(f"block_size {bs} does not align with {rows} rows at offset {row_offset}")
    nkb = cols // bs
    bad = sorted(kb for _, kb in pattern if kb >= nkb)
    if bad:
        raise ValueError(f"pattern key blocks {bad[:4]} out of range for {nkb} key blocks")
    qblk = np.arange(row_offset, row_offset + rows) // bs
    kblk = np.arange(cols) // bs
    vis = np.zeros((rows, cols), dtype=bool)
    for qb, kb in pattern:
        vis |= (qblk[:, None] == qb) & (kblk[None, :] == kb)
    return vis


def check_block_pattern(n: int, block_size: int, pattern) -> dict:
    """The argument checks of blocked_kernel (kernels.py:63-80), in its
    order; returns {qb: sorted visible kb}."""
    if n % block_size != 0:
        raise DivisibilityError(f"block_size {block_size} does not divide sequence length {n}")
    nblocks = n // block_size
    bad = sorted((qb, kb) for qb, kb in pattern if qb >= nblocks or kb >= nblocks)
    if bad:
        raise ValueError(f"pattern blocks {bad[:4]} out of range for {nblocks} blocks")
    visible = {qb: sorted(kb for qb2, kb in pattern if qb2 == qb) for qb in range(nblocks)}
    for qb in range(nblocks):
        if not visible[qb]:
            raise DegenerateRowError(f"query block {qb} has no visible key blocks (invalid sparse pattern)")
    return visible


def blocked_attention_head(q, k, v, block_size: int, pattern, scale: float, exact: bool = True):
    """blocked_kernel (kernels.py:55-86) on (n, b, hd) views: per query
    block, scores against the concatenated visible key blocks (ascending
    kb), unmasked row_softmax, ctx = probs v.  Also returns the row LSE over
    the same scores (RESTATEMENT, no reference counterpart).
    Returns (ctx (n, b, hd), lse (b, n))."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    n, b, hd = q.shape
    bs = block_size
    visible = check_block_pattern(n, bs, pattern)
    ctx = np.empty((n, b, hd))
    lse = np.empty((b, n))
    for bi in range(b):
        for qb, kbs in visible.items():
            rows = slice(qb * bs, (qb + 1) * bs)
            kcat = np.concatenate([k[kb * bs:(kb + 1) * bs, bi, :] for kb in kbs], axis=0)
            vcat = np.concatenate([v[kb * bs:(kb + 1) * bs, bi, :] for kb in kbs], axis=0)
            scores = matmul(q[rows, bi, :], kcat.T, exact) * scale
            ctx[rows, bi, :] = matmul(row_softmax(scores, "none"), vcat, exact)
            lse[bi, rows] = row_lse(scores, "none")
    return ctx, lse


def local_attention_blocked(q4, k4, v4, block_size: int, pattern, scale: float | None = None,
                            exact: bool = True):
    """Head loop of ulysses.py:148-152 with the blocked kernel (GQA
    restatement as in local_attention).  Returns (ctx4, lse (b, Hq, n))."""
    q4 = np.asarray(q4)
    n, b, hq, hd = q4.shape
    hkv = np.asarray(k4).shape[2]
    if scale is None:
        scale = 1.0 / math.sqrt(hd)
    ctx4 = np.empty((n, b, hq, hd))
    lse = np.empty((b, hq, n))
    for hh in range(hq):
        g = kv_head_for(hh, hq, hkv)
        c, l = blocked_attention_head(q4[:, :, hh, :], k4[:, :, g, :], v4[:, :, g, :], block_size, pattern,
                                      scale, exact)
        ctx4[:, :, hh, :] = c
        lse[:, hh, :] = l
    return ctx4, lse


def pattern_bits(n: int, block_size: int, pattern) -> np.ndarray:
    """Device encoding of a block pattern (include/ulysses_b200.h,
    ul_attn_fwd_blocked): uint32 rows of ceil(nb/32) words, bit kb % 32 of
    word kb / 32 in row qb set iff (qb, kb) is in the pattern."""
    nb = n // block_size
    words = (nb + 31) // 32
    bits = np.zeros((nb, words), dtype=np.uint32)
    for qb, kb in pattern:
        bits[qb, kb // 32] |= np.uint32(1 << (kb % 32))
    return bits


# ---------------------------------------------------------------------------
# L3: the DistributedAttention core across P simulated ranks
# ---------------------------------------------------------------------------

def check_group(n: int, h: int, p: int):
    """layers.py:53-57 (P | n and P | H)."""
    if n % p != 0:
        raise DivisibilityError(f"p={p} does not divide sequence length n={n}")
    if h % p != 0:
        raise DivisibilityError(f"p={p} does not divide head count {h}")


def ulysses_forward(q_loc, k_loc, v_loc, kind: str, scale: float | None = None,
                    exact: bool = True):
    """Forward core ulysses.py:144-154 with q/k/v given per rank as
    (n/P, b, H, hd) sequence shards: 3x seq->head, per-head kernel, 1x
    head->seq.  Returns (out_loc list, state) where state carries the
    head-sharded q4/k4/v4 and the per-rank LSE."""
    p = len(q_loc)
    nl, b, hq, hd = np.asarray(q_loc[0]).shape
    hkv = np.asarray(k_loc[0]).shape[2]
    check_group(nl * p, hq, p)
    if hkv % p != 0:
        raise DivisibilityError(f"p={p} does not divide kv head count {hkv}")
    q4 = all_to_all(q_loc, 2, 0)
    k4 = all_to_all(k_loc, 2, 0)
    v4 = all_to_all(v_loc, 2, 0)
    ctx4, lse = [], []
    for r in range(p):
        c, l = local_attention(q4[r], k4[r], v4[r], kind, scale, exact)
        ctx4.append(c)
        lse.append(l)
    out = all_to_all(ctx4, 0, 2)
    return out, {"q4": q4, "k4": k4, "v4": v4, "ctx4": ctx4, "lse": lse}


def ulysses_backward(dout_loc, state, kind: str, scale: float | None = None,
                     exact: bool = True):
    """Backward core ulysses.py:213-226: dctx seq->head, per-head backward,
    3x head->seq (dq, dk, dv)."""
    p = len(dout_loc)
    dctx4 = all_to_all(dout_loc, 2, 0)
    dq4, dk4, dv4 = [], [], []
    for r in range(p):
        dq, dk, dv = local_attention_backward(state["q4"][r], state["k4"][r], state["v4"][r],
                                              dctx4[r], kind, scale, exact)
        dq4.append(dq)
        dk4.append(dk)
        dv4.append(dv)
    return all_to_all(dq4, 0, 2), all_to_all(dk4, 0, 2), all_to_all(dv4, 0, 2)


# ---------------------------------------------------------------------------
# L4: the attention layer with its projections, and the transformer block
# (ulysses.py:135-157, 172-184, 188-245)
# ---------------------------------------------------------------------------

LN_EPS = 1e-5           # layers.py:22
MLP_EXPANSION = 4       # layers.py:23


def make_weights(d: int, seed: int, layer: int = 0) -> dict:
    """layers.py:83-99: one layer's replicated weights from
    default_rng([seed, 101, layer]) in the reference's draw order."""
    rng = np.random.default_rng([int(seed), 101, int(layer)])
    inv = 1.0 / np.sqrt(d)
    w = {}
    w["wq"] = rng.standard_normal((d, d)) * inv
    w["wk"] = rng.standard_normal((d, d)) * inv
    w["wv"] = rng.standard_normal((d, d)) * inv
    w["wo"] = rng.standard_normal((d, d)) * inv
    w["w1"] = rng.standard_normal((d, MLP_EXPANSION * d)) * inv
    w["w2"] = rng.standard_normal((MLP_EXPANSION * d, d)) / np.sqrt(MLP_EXPANSION * d)
    w["ln1_gain"] = 1.0 + 0.1 * rng.standard_normal(d)
    w["ln1_bias"] = 0.1 * rng.standard_normal(d)
    w["ln2_gain"] = 1.0 + 0.1 * rng.standard_normal(d)
    w["ln2_bias"] = 0.1 * rng.standard_normal(d)
    return w


def make_input(n: int, b: int, d: int, seed: int) -> np.ndarray:
    """layers.py:102-105."""
    return np.random.default_rng([int(seed), 202]).standard_normal((n, b, d))


def project(x3, w, exact: bool = True) -> np.ndarray:
    """layers.py:118-122: (s, b, d_in) @ (d_in, d_out)."""
    s, b, din = x3.shape
    return matmul(np.asarray(x3).reshape(s * b, din), w, exact).reshape(s, b, w.shape[1])


def layernorm(x, gain, bias) -> np.ndarray:
    """layers.py:106-110."""
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + LN_EPS) * gain + bias


def gelu(x) -> np.ndarray:
    """layers.py:113-115 (exact, erf-based)."""
    from scipy.special import erf
    return 0.5 * x * (1.0 + erf(x / np.sqrt(2.0)))


def ulysses_attention_layer(x_loc, w: dict, h: int, kind: str, exact: bool = True):
    """ulysses_attention_forward_with_state (ulysses.py:135-157) on P
    sequence shards x_loc[r] (n/P, b, d): project, the core, project wo.
    Returns (out_loc list, state)."""
    p = len(x_loc)
    nl, b, d = np.asarray(x_loc[0]).shape
    hd = d // h
    four = lambda t: t.reshape(nl, b, h, hd)
    q = [four(project(x, w["wq"], exact)) for x in x_loc]
    k = [four(project(x, w["wk"], exact)) for x in x_loc]
    v = [four(project(x, w["wv"], exact)) for x in x_loc]
    c_loc, st = ulysses_forward(q, k, v, kind, exact=exact)
    c_seq = [c.reshape(nl, b, d) for c in c_loc]
    out = [project(c, w["wo"], exact) for c in c_seq]
    st = dict(st, x_loc=[np.asarray(x, np.float64) for x in x_loc], c_seq=c_seq, h=h)
    return out, st


def ulysses_attention_layer_backward(grad_loc, state, w: dict, kind: str, exact: bool = True):
    """ulysses_attention_backward (ulysses.py:188-245): returns (grad_x_loc,
    grad_w summed over ranks in rank order, like
    run_ulysses_attention_backward ulysses.py:296-302)."""
    p = len(grad_loc)
    nl, b, d = np.asarray(grad_loc[0]).shape
    h = state["h"]
    hd = d // h
    g2 = [np.asarray(g, np.float64).reshape(nl * b, d) for g in grad_loc]
    c2 = [c.reshape(nl * b, d) for c in state["c_seq"]]
    dwo = [matmul(c.T, g, exact) for c, g in zip(c2, g2)]
    dc = [matmul(g, w["wo"].T, exact).reshape(nl, b, h, hd) for g in g2]
    dq, dk, dv = ulysses_backward(dc, state, kind, exact=exact)
    x2 = [x.reshape(nl * b, d) for x in state["x_loc"]]
    flat = lambda t: np.asarray(t).reshape(nl * b, d)
    gw = {"wq": [matmul(x.T, flat(g), exact) for x, g in zip(x2, dq)],
          "wk": [matmul(x.T, flat(g), exact) for x, g in zip(x2, dk)],
          "wv": [matmul(x.T, flat(g), exact) for x, g in zip(x2, dv)],
          "wo": dwo}
    grad_w = {}
    for key, parts in gw.items():
        tot = parts[0]
        for t in parts[1:]:
            tot = tot + t
        grad_w[key] = tot
    gx = [(matmul(flat(a), w["wq"].T, exact) + matmul(flat(bq), w["wk"].T, exact)
           + matmul(flat(c), w["wv"].T, exact)).reshape(nl, b, d) for a, bq, c in zip(dq, dk, dv)]
    return gx, grad_w


def ulysses_block(x_loc, w: dict, h: int, kind: str, exact: bool = True):
    """ulysses_block_forward (ulysses.py:172-184): pre-LN attention with
    residual, then pre-LN GELU MLP with residual; only attention talks."""
    xs = [np.asarray(x, np.float64) for x in x_loc]
    t1 = [layernorm(x, w["ln1_gain"], w["ln1_bias"]) for x in xs]
    attn, _ = ulysses_attention_layer(t1, w, h, kind, exact)
    x1 = [x + a for x, a in zip(xs, attn)]
    t2 = [layernorm(x, w["ln2_gain"], w["ln2_bias"]) for x in x1]
    return [x + project(gelu(project(t, w["w1"], exact)), w["w2"], exact) for x, t in zip(x1, t2)]


def ring_shift(locals_, steps: int = 1):
    """RankContext.ring_shift combine (simgroup.py:380-381): rank i gets
    rank (i - steps) mod P's payload."""
    p = len(locals_)
    return [locals_[(i - steps) % p] for i in range(p)]


def ring_attention_layer(x_loc, w: dict, h: int, kind: str, exact: bool = True):
    """ring_attention_forward (baselines.py:68-121): per rank, full score
    rows assembled from the circulating K chunks (ascending global key
    order == chunk src), masked row_softmax with row_offset = rank*n/P, the
    context accumulated over the circulating V chunks in arrival order."""
    p = len(x_loc)
    nl, b, d = np.asarray(x_loc[0]).shape
    hd = d // h
    n = nl * p
    scale = 1.0 / np.sqrt(hd)
    q4 = [project(x, w["wq"], exact).reshape(nl, b, h, hd) for x in x_loc]
    ks = [project(x, w["wk"], exact) for x in x_loc]
    vs = [project(x, w["wv"], exact) for x in x_loc]
    scores = [np.empty((h, b, nl, n)) for _ in range(p)]
    cur = ks
    for step in range(p):
        for r in range(p):
            src = (r - step) % p
            k4 = cur[r].reshape(nl, b, h, hd)
            for hh in range(h):
                for bi in range(b):
                    scores[r][hh, bi, :, src * nl:(src + 1) * nl] = matmul(q4[r][:, bi, hh, :],
                                                                          k4[:, bi, hh, :].T, exact) * scale
        if step < p - 1:
            cur = ring_shift(cur, 1)
    probs = [np.empty_like(s_) for s_ in scores]
    for r in range(p):
        for hh in range(h):
            for bi in range(b):
                probs[r][hh, bi] = row_softmax(scores[r][hh, bi], kind, row_offset=r * nl)
    ctx4 = [np.zeros((nl, b, h, hd)) for _ in range(p)]
    cur = vs
    for step in range(p):
        for r in range(p):
            src = (r - step) % p
            v4 = cur[r].reshape(nl, b, h, hd)
            for hh in range(h):
                for bi in range(b):
                    ctx4[r][:, bi, hh, :] += matmul(probs[r][hh, bi, :, src * nl:(src + 1) * nl],
                                                    v4[:, bi, hh, :], exact)
        if step < p - 1:
            cur = ring_shift(cur, 1)
    return [project(c.reshape(nl, b, d), w["wo"], exact) for c in ctx4]


# ---------------------------------------------------------------------------
# seeded synthetic inputs
# ---------------------------------------------------------------------------

def make_tensor(shape, seed: int, stream: int, dtype: str = "float32") -> np.ndarray:
    """N(0,1) draws from ``default_rng([seed, stream])`` (the reference seeds
    the same way, layers.py:100-103), rounded to ``dtype`` and returned as
    float64 holding exactly-representable values.  ``dtype`` 'bfloat16'
    rounds to nearest-even bf16."""
    x = np.random.default_rng([int(seed), int(stream)]).standard_normal(shape).astype(np.float32)
    if dtype == "bfloat16":
        x = bf16_round(x)
    elif dtype != "float32":
        raise ValueError(dtype)
    return x.astype(np.float64)


def bf16_round(x) -> np.ndarray:
    """Round-to-nearest-even float32 -> bfloat16 -> float32 (bit-exact with
    the CUDA __float2bfloat16_rn conversion for finite inputs)."""
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounding = ((u >> 16) & 1) + 0x7FFF
    u = ((u + rounding) >> 16) << 16
    return u.astype(np.uint32).view(np.float32)
