"""The Ulysses attention layer with its projections, and the transformer
block around it.

Mirrors the reference's layer (paths relative to /root/reference/pkg/src/seqlab):

  * ``UlyssesAttention`` == ``ulysses_attention_forward_with_state``
    (ulysses.py:135-157): q/k/v = x @ wq/wk/wv (layers.py:118-122), the
    DistributedAttention core (3x seq->head, local attention, head->seq),
    out = c @ wo.  Its backward is ``ulysses_attention_backward``
    (ulysses.py:188-245): grad_x plus this rank's partial weight gradients
    (their sum over ranks is the single-rank gradient; reducing them is the
    data-parallel engine's job, not the attention path's -- ulysses.py:193-197).
  * ``UlyssesBlock`` == ``ulysses_block_forward`` (ulysses.py:172-184):
    pre-LN attention + residual, pre-LN GELU MLP (4x, exact erf) + residual;
    only attention communicates.
  * ``make_weights`` == layers.py:83-99 (same draws, same order).

The attention core runs on this package's kernels and exchanges.  In bf16
with hd = 128 the Q/K/V projection is this package's tcgen05 GEMM whose
epilogue performs the seq->head exchange (csrc/proj_sm100.cu), and the layer
is one autograd node; its backward's dc = g Wo^T is the same tcgen05 GEMM
with the dO seq->head exchange in its epilogue (W read K-major); the
remaining plain GEMMs (c Wo, dWo, dX, dW) are cuBLAS,
and the row-wise pieces are torch ops -- off the hot path.  Weights are (d_in, d_out) like
the reference's ``project``.
"""

from __future__ import annotations

import math

import numpy as np
import torch
import torch.nn.functional as F

from . import _lib
from .attention import _ATTN_DTYPES, DistributedAttention, FlashAttention
from .errors import DivisibilityError

LN_EPS = 1e-5          # layers.py:22
MLP_EXPANSION = 4      # layers.py:23


def make_weights(d: int, seed: int, layer: int = 0) -> dict:
    """layers.py:83-99 (float64 numpy; cast when loading into a module)."""
    rng = np.random.default_rng([int(seed), 101, int(layer)])
    inv = 1.0 / np.sqrt(d)
    w = {}
    for name in ("wq", "wk", "wv", "wo"):
        w[name] = rng.standard_normal((d, d)) * inv
    w["w1"] = rng.standard_normal((d, MLP_EXPANSION * d)) * inv
    w["w2"] = rng.standard_normal((MLP_EXPANSION * d, d)) / np.sqrt(MLP_EXPANSION * d)
    w["ln1_gain"] = 1.0 + 0.1 * rng.standard_normal(d)
    w["ln1_bias"] = 0.1 * rng.standard_normal(d)
    w["ln2_gain"] = 1.0 + 0.1 * rng.standard_normal(d)
    w["ln2_bias"] = 0.1 * rng.standard_normal(d)
    return w


def _param(x, dtype, device):
    return torch.nn.Parameter(torch.as_tensor(np.asarray(x), dtype=torch.float64).to(dtype).to(device))


class _UlyssesLayerFn(torch.autograd.Function):
    """The whole attention layer as one autograd node (bf16, hd = 128, the
    library's FlashAttention): fused QKV GEMM + seq->head exchange
    (ul_qkv_proj_exchange), attention with the O exchange in its epilogue,
    c @ wo; backward mirrors ulysses_attention_backward (ulysses.py:188-245)
    with the dQ/dK/dV exchange fused into the backward kernels and the
    remaining GEMMs on cuBLAS."""

    @staticmethod
    def forward(ctx, group, attn, h, hkv, x, wqkv, wo):
        nl, b, d = x.shape
        x2 = x.reshape(nl * b, d).contiguous()
        q4, k4, v4 = group.qkv_projection(x2, wqkv.contiguous(), b, h, hkv)
        if group.world > 1:
            o4, lse, c = attn.forward_exchange(q4, k4, v4, group, label="attn.ctx.head2seq")
        else:
            o4, lse = attn.forward_with_lse(q4, k4, v4)
            c = o4
        c2 = c.reshape(nl * b, d)
        ctx.group, ctx.attn, ctx.shape = group, attn, (nl, b, d, h, hkv)
        ctx.save_for_backward(x2, wqkv, wo, q4, k4, v4, o4, lse, c2)
        return (c2 @ wo).reshape(nl, b, d)

    @staticmethod
    def backward(ctx, gout):
        group, attn = ctx.group, ctx.attn
        nl, b, d, h, hkv = ctx.shape
        x2, wqkv, wo, q4, k4, v4, o4, lse, c2 = ctx.saved_tensors
        g2 = gout.reshape(nl * b, d).contiguous()
        dwo = c2.t() @ g2                                             # ulysses.py:206
        # dc = g Wo^T (ulysses.py:207) as the tcgen05 GEMM whose epilogue
        # stores each head block at its owner: the dctx seq->head flip
        # (ulysses.py:213) fused into it, no dc round trip through HBM
        (do4,) = group.proj_exchange(g2, wo.contiguous(), (h,), b, transposed=True, labels=("bwd.ctx.seq2head",),
                                     label="bwd.ctx.seq2head")
        if group.world > 1:
            dq, dk, dv = attn.backward_exchange(q4, k4, v4, o4, lse, do4, group, label="bwd.qkv.head2seq")
        else:
            dq, dk, dv = attn.backward(q4, k4, v4, o4, lse, do4)
        dqkv = torch.cat([t.reshape(nl * b, -1) for t in (dq, dk, dv)], dim=1)
        dx = (dqkv @ wqkv.t()).reshape(nl, b, d)                      # ulysses.py:240
        dwqkv = x2.t() @ dqkv                                         # ulysses.py:234-238
        return None, None, None, None, dx, dwqkv, dwo


class UlyssesAttention(torch.nn.Module):
    """``forward(x)``: this rank's sequence shard ``[n/P, b, d]`` -> ``[n/P, b, d]``."""

    def __init__(self, d_model: int, heads: int, sequence_process_group=None, mask: str = "causal",
                 weights: dict | None = None, dtype=torch.bfloat16, device=None, local_attention=None,
                 seed: int = 0):
        super().__init__()
        if d_model % heads != 0:   # AttentionSpec.__post_init__, layers.py:46-49
            raise DivisibilityError(f"head count {heads} does not divide hidden size {d_model}")
        self.d, self.h, self.hd = d_model, heads, d_model // heads
        device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        w = weights if weights is not None else make_weights(d_model, seed)
        self.wq, self.wk, self.wv, self.wo = (_param(w[k], dtype, device) for k in ("wq", "wk", "wv", "wo"))
        attn = local_attention if local_attention is not None else FlashAttention(mask)
        self.core = DistributedAttention(attn, sequence_process_group, scatter_idx=2, gather_idx=0)

    def _fused_ok(self, x):
        a = self.core.local_attn
        return (isinstance(a, FlashAttention) and a.mask != "blocked" and x.dtype == torch.bfloat16
                and self.hd == 128 and self.d % 64 == 0)

    def forward(self, x):
        nl, b, d = x.shape
        if self._fused_ok(x):   # one node: fused QKV GEMM + exchange, fused attention exchanges
            wqkv = torch.cat([self.wq, self.wk, self.wv], dim=1)
            return _UlyssesLayerFn.apply(self.core.spg, self.core.local_attn, self.h, self.h, x, wqkv, self.wo)
        x2 = x.reshape(nl * b, d)
        # one GEMM for q|k|v (ulysses.py:140-142), split into head views
        qkv = x2 @ torch.cat([self.wq, self.wk, self.wv], dim=1)
        q, k, v = (t.reshape(nl, b, self.h, self.hd) for t in qkv.split(d, dim=1))
        c = self.core(q.contiguous(), k.contiguous(), v.contiguous())     # ulysses.py:144-154
        return (c.reshape(nl * b, d) @ self.wo).reshape(nl, b, d)        # ulysses.py:155


# ---------------------------------------------------------------------------
# the block's row-wise kernels (csrc/block.cu): fused residual + layernorm,
# exact GELU -- forward and backward
# ---------------------------------------------------------------------------

_BLOCK_DTYPES = {torch.float32: _lib.DTYPE_F32, torch.bfloat16: _lib.DTYPE_BF16}


def _st(t):
    return torch.cuda.current_stream(t.device).cuda_stream


def _ln_forward(x, r, gain, bias, eps):
    d = x.shape[-1]
    rows = x.numel() // d
    s = torch.empty_like(x) if r is not None else None
    y = torch.empty_like(x)
    stats = torch.empty((rows, 2), dtype=torch.float32, device=x.device)
    _lib.check(_lib.lib().ul_add_layernorm(x.data_ptr(), r.data_ptr() if r is not None else None, gain.data_ptr(),
                                           bias.data_ptr(), s.data_ptr() if s is not None else None, y.data_ptr(),
                                           stats.data_ptr(), rows, d, eps, _BLOCK_DTYPES[x.dtype], _st(x)))
    return s, y, stats


def _ln_backward(dy, s, gain, stats):
    d = s.shape[-1]
    rows = s.numel() // d
    dy = dy.contiguous()
    dx = torch.empty_like(s)
    dgain, dbias = torch.empty_like(gain), torch.empty_like(gain)
    wsb = int(_lib.lib().ul_layernorm_bwd_workspace_bytes(rows, d))
    ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device=s.device)
    _lib.check(_lib.lib().ul_layernorm_bwd(dy.data_ptr(), s.data_ptr(), gain.data_ptr(), stats.data_ptr(),
                                           dx.data_ptr(), dgain.data_ptr(), dbias.data_ptr(), ws.data_ptr(),
                                           ws.numel(), rows, d, _BLOCK_DTYPES[s.dtype], _st(s)))
    return dx, dgain, dbias


class _LayerNormFn(torch.autograd.Function):
    """y = layernorm(x) * gain + bias (layers.py:106-110)."""

    @staticmethod
    def forward(ctx, x, gain, bias, eps):
        x = x.contiguous()
        _, y, stats = _ln_forward(x, None, gain, bias, eps)
        ctx.save_for_backward(x, gain, stats)
        return y

    @staticmethod
    def backward(ctx, dy):
        x, gain, stats = ctx.saved_tensors
        dx, dgain, dbias = _ln_backward(dy, x, gain, stats)
        return dx, dgain, dbias, None


class _AddLayerNormFn(torch.autograd.Function):
    """(s, y) = (x + r, layernorm(x + r) * gain + bias) in one pass: the
    residual of ulysses.py:179 fused into the layernorm after it."""

    @staticmethod
    def forward(ctx, x, r, gain, bias, eps):
        s, y, stats = _ln_forward(x.contiguous(), r.contiguous(), gain, bias, eps)
        ctx.save_for_backward(s, gain, stats)
        return s, y

    @staticmethod
    def backward(ctx, ds, dy):
        s, gain, stats = ctx.saved_tensors
        dx, dgain, dbias = _ln_backward(dy, s, gain, stats)
        if ds is not None:
            dx = dx + ds
        return dx, dx, dgain, dbias, None


class _GeluFn(torch.autograd.Function):
    """Exact erf GELU (layers.py:113-127) on the GPU, forward and backward."""

    @staticmethod
    def forward(ctx, x):
        x = x.contiguous()
        y = torch.empty_like(x)
        _lib.check(_lib.lib().ul_gelu(x.data_ptr(), None, y.data_ptr(), x.numel(), _BLOCK_DTYPES[x.dtype], _st(x)))
        ctx.save_for_backward(x)
        return y

    @staticmethod
    def backward(ctx, dy):
        (x,) = ctx.saved_tensors
        dy = dy.contiguous()
        dx = torch.empty_like(x)
        _lib.check(_lib.lib().ul_gelu(x.data_ptr(), dy.data_ptr(), dx.data_ptr(), x.numel(), _BLOCK_DTYPES[x.dtype],
                                      _st(x)))
        return dx


def layernorm(x, gain, bias, eps: float = LN_EPS):
    return _LayerNormFn.apply(x, gain, bias, eps)


def add_layernorm(x, r, gain, bias, eps: float = LN_EPS):
    """(x + r, layernorm(x + r))."""
    return _AddLayerNormFn.apply(x, r, gain, bias, eps)


def gelu(x):
    return _GeluFn.apply(x)


class UlyssesBlock(torch.nn.Module):
    """Pre-LN transformer block on sequence shards (ulysses.py:172-184)."""

    def __init__(self, d_model: int, heads: int, sequence_process_group=None, mask: str = "causal",
                 weights: dict | None = None, dtype=torch.bfloat16, device=None, seed: int = 0, layer: int = 0):
        super().__init__()
        device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        w = weights if weights is not None else make_weights(d_model, seed, layer)
        self.attn = UlyssesAttention(d_model, heads, sequence_process_group, mask, w, dtype, device)
        self.w1, self.w2 = _param(w["w1"], dtype, device), _param(w["w2"], dtype, device)
        self.ln1_gain, self.ln1_bias = _param(w["ln1_gain"], dtype, device), _param(w["ln1_bias"], dtype, device)
        self.ln2_gain, self.ln2_bias = _param(w["ln2_gain"], dtype, device), _param(w["ln2_bias"], dtype, device)

    def forward(self, x):
        # ulysses.py:172-184 on this package's kernels: LN (csrc/block.cu),
        # the attention layer, residual + LN fused, GELU MLP (cuBLAS GEMMs
        # around the GELU kernel), residual; only the attention communicates
        t1 = layernorm(x, self.ln1_gain, self.ln1_bias)                           # layers.py:106-110
        x1, t2 = add_layernorm(x, self.attn(t1), self.ln2_gain, self.ln2_bias)   # x1 = x + attn(t1)
        return x1 + gelu(t2 @ self.w1) @ self.w2                                  # layers.py:113-127


# ---------------------------------------------------------------------------
# ring attention (first step: the ring half of a hybrid)
# ---------------------------------------------------------------------------

def _ring_forward(q, k, v, group, mask, prefix):
    """Forward of the ring core: returns (o, lse [b, h, n/P]) with the
    partial contexts merged exactly in fp32."""
    p, r = group.world, group.rank
    o_acc = lse_acc = None
    cur_k, cur_v = k, v
    dense, causal = FlashAttention("none"), FlashAttention("causal")
    main = torch.cuda.current_stream(q.device)
    side = _side_stream(group, q.device) if p > 1 else None
    for step in range(p):
        src = (r - step) % p
        nxt = None
        if step < p - 1:
            # the next chunk travels on a second stream while this one is computed
            side.wait_stream(main)
            with torch.cuda.stream(side):
                nxt = group.ring_shift([cur_k, cur_v], 1, labels=[f"{prefix}.kring.{step}", f"{prefix}.vring.{step}"])
            for t in (cur_k, cur_v):
                t.record_stream(side)
        if mask == "none" or src <= r:
            attn = causal if (mask == "causal" and src == r) else dense
            o_s, lse_s = attn.forward_with_lse(q, cur_k, cur_v)        # lse [b, h, n/P]
            first = o_acc is None
            if first:
                o_acc = torch.empty(q.shape, dtype=torch.float32, device=q.device)
                lse_acc = torch.empty_like(lse_s)
            n_, b_, h_, hd_ = q.shape                                     # exact merge, one kernel
            _lib.check(_lib.lib().ul_lse_merge(o_acc.data_ptr(), lse_acc.data_ptr(), o_s.data_ptr(),
                                               lse_s.data_ptr(), n_, b_, h_, hd_, _ATTN_DTYPES[q.dtype],
                                               int(first), main.cuda_stream))
        if nxt is not None:
            main.wait_stream(side)
            for t in nxt:
                t.record_stream(main)
            cur_k, cur_v = nxt
    return o_acc.to(q.dtype), lse_acc


def _side_stream(group, device):
    """One extra stream per rank for the ring's transfers (cached on the group)."""
    s = getattr(group, "_ring_side_stream", None)
    if s is None:
        s = torch.cuda.Stream(device=device)
        try:
            group._ring_side_stream = s
        except AttributeError:
            pass
    return s


class _RingAttnFn(torch.autograd.Function):
    """Ring attention with its backward: K/V circulate again, each visible
    chunk runs the local backward kernels with the GLOBAL (merged) O and LSE
    -- P = exp(S - LSE) and D = rowsum(dO O) are then the full-row values, so
    the chunk gradients are exact partial sums -- dQ accumulates locally,
    dK/dV contributions travel with their chunk and a last shift brings
    them home (fp32 accumulators)."""

    @staticmethod
    def forward(ctx, group, mask, prefix, q, k, v):
        o, lse = _ring_forward(q, k, v, group, mask, prefix)
        ctx.group, ctx.mask, ctx.prefix = group, mask, prefix
        ctx.save_for_backward(q, k, v, o, lse)
        return o

    @staticmethod
    def backward(ctx, do):
        group, mask, prefix = ctx.group, ctx.mask, ctx.prefix
        q, k, v, o, lse = ctx.saved_tensors
        do = do.contiguous()
        p, r = group.world, group.rank
        dense, causal = FlashAttention("none"), FlashAttention("causal")
        dq = torch.zeros(q.shape, dtype=torch.float32, device=q.device)
        cur = [k, v, torch.zeros(k.shape, dtype=torch.float32, device=k.device),
               torch.zeros(v.shape, dtype=torch.float32, device=v.device)]
        main = torch.cuda.current_stream(q.device)
        side = _side_stream(group, q.device) if p > 1 else None
        for step in range(p):
            src = (r - step) % p
            nkv = None
            if step < p - 1:   # the next K/V chunk travels while this one is differentiated
                side.wait_stream(main)
                with torch.cuda.stream(side):
                    nkv = group.ring_shift(cur[:2], 1, labels=[f"{prefix}.bwd.kring.{step}",
                                                               f"{prefix}.bwd.vring.{step}"])
                for t in cur[:2]:
                    t.record_stream(side)
            if mask == "none" or src <= r:
                attn = causal if (mask == "causal" and src == r) else dense
                dq_c, dk_c, dv_c = attn.backward(q, cur[0], cur[1], o, lse, do)
                dq += dq_c.float()
                cur[2] += dk_c.float()
                cur[3] += dv_c.float()
            if nkv is not None:   # the chunk's dK/dV accumulators follow it once updated
                # (join the side stream first: consecutive calls of one group must
                # stay stream-ordered -- a rank reuses a receive slot every other call)
                main.wait_stream(side)
                for t in nkv:
                    t.record_stream(main)
                acc = group.ring_shift(cur[2:], 1, labels=[f"{prefix}.bwd.dkring.{step}",
                                                           f"{prefix}.bwd.dvring.{step}"])
                cur = list(nkv) + list(acc)
        dk, dv = cur[2], cur[3]
        if p > 1:   # the accumulators of chunk r are one hop away
            dk, dv = group.ring_shift([dk, dv], 1, labels=[f"{prefix}.bwd.dkring.home", f"{prefix}.bwd.dvring.home"])
        return None, None, None, dq.to(q.dtype), dk.to(k.dtype), dv.to(v.dtype)


def ring_attention_core(q, k, v, group, mask: str = "causal", prefix: str = "attn"):
    """Ring self-attention on sequence shards [n/P, b, h, hd] (baselines.py:
    68-121: Q local, K and V circulate P-1 steps; the reference fills full
    score rows, here every arriving chunk is one local-attention call that
    also returns its row LSE, and the partial contexts are merged exactly:
    o = sum_j exp(lse_j - lse) o_j with lse = logsumexp_j lse_j).  With
    contiguous shards, chunk src of rank r is dense (src < r), causal
    (src == r) or invisible (src > r) under the causal mask (tensor.py:161).
    Differentiable (the reference's ring baseline is forward only; the
    backward here is _RingAttnFn's).  Usable when P > H_kv, where Ulysses
    cannot split the kv heads."""
    if mask not in ("causal", "none"):
        from .errors import KernelError
        raise KernelError(f"ring attention supports dense/causal masks, got {mask!r}")
    return _RingAttnFn.apply(group, mask, prefix, q.contiguous(), k.contiguous(), v.contiguous())


class RingAttention(torch.nn.Module):
    """``ring_attention_forward`` (baselines.py:68-121): projections, the ring
    core above, output projection.  ``forward(x)``: [n/P, b, d] -> [n/P, b, d]."""

    def __init__(self, d_model: int, heads: int, sequence_process_group=None, mask: str = "causal",
                 weights: dict | None = None, dtype=torch.bfloat16, device=None, seed: int = 0):
        super().__init__()
        from .attention import _group
        if d_model % heads != 0:
            raise DivisibilityError(f"head count {heads} does not divide hidden size {d_model}")
        self.d, self.h, self.hd, self.mask = d_model, heads, d_model // heads, mask
        device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        w = weights if weights is not None else make_weights(d_model, seed)
        self.wq, self.wk, self.wv, self.wo = (_param(w[k], dtype, device) for k in ("wq", "wk", "wv", "wo"))
        self.group = _group(sequence_process_group)

    def forward(self, x, prefix: str = "L0.attn"):
        nl, b, d = x.shape
        x2 = x.reshape(nl * b, d)
        four = lambda t: t.reshape(nl, b, self.h, self.hd).contiguous()
        q, k, v = four(x2 @ self.wq), four(x2 @ self.wk), four(x2 @ self.wv)
        c = ring_attention_core(q, k, v, self.group, self.mask, prefix)
        return (c.reshape(nl * b, d) @ self.wo).reshape(nl, b, d)


class HybridAttention(torch.nn.Module):
    """Ulysses x ring: P = P_u * P_r ranks, rank index
    ring-major (rank = i * P_u + j).  Ulysses over the P_u ranks of a ring
    position (heads split P_u ways, sequence gathered to the n/P_r tokens of
    ring chunk i -- contiguous global positions), ring attention over the
    P_r ranks holding the same heads, Ulysses back.  For P beyond the head
    count (P_u <= H_kv) or across nodes (ring over the slow links).
    Differentiable (ring backward: _RingAttnFn)."""

    def __init__(self, d_model: int, heads: int, ulysses_group, ring_group, mask: str = "causal",
                 weights: dict | None = None, dtype=torch.bfloat16, device=None, seed: int = 0):
        super().__init__()
        from .attention import _group
        if d_model % heads != 0:
            raise DivisibilityError(f"head count {heads} does not divide hidden size {d_model}")
        self.ug, self.rg = _group(ulysses_group), _group(ring_group)
        if heads % self.ug.world:
            raise DivisibilityError(f"p_ulysses={self.ug.world} does not divide head count {heads}")
        self.d, self.h, self.hd, self.mask = d_model, heads, d_model // heads, mask
        device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        w = weights if weights is not None else make_weights(d_model, seed)
        self.wq, self.wk, self.wv, self.wo = (_param(w[k], dtype, device) for k in ("wq", "wk", "wv", "wo"))

    def forward(self, x):
        from .attention import seq_all_to_all
        nl, b, d = x.shape
        x2 = x.reshape(nl * b, d)
        four = lambda t: t.reshape(nl, b, self.h, self.hd).contiguous()
        q, k, v = four(x2 @ self.wq), four(x2 @ self.wk), four(x2 @ self.wv)
        if self.ug.world > 1:   # differentiable flips (backward swaps the axes)
            q, k, v = (seq_all_to_all(t, 2, 0, self.ug, f"attn.{n}.seq2head") for t, n in ((q, "q"), (k, "k"), (v, "v")))
        c = ring_attention_core(q, k, v, self.rg, self.mask, "attn")
        if self.ug.world > 1:
            c = seq_all_to_all(c, 0, 2, self.ug, "attn.ctx.head2seq")
        return (c.reshape(nl * b, d) @ self.wo).reshape(nl, b, d)
