"""DistributedAttention / seq_all_to_all and the local-attention plugins.

API surface (DeepSpeed-Ulysses, arXiv 2309.14509):

    seq_all_to_all(input, scatter_idx, gather_idx, group)
    DistributedAttention(local_attn, sequence_process_group, scatter_idx=2, gather_idx=0)

mapped onto the reference's semantics (paths relative to
/root/reference/pkg/src/seqlab):

  * ``seq_all_to_all`` == ``RankContext.all_to_all(local, split_axis=
    scatter_idx, concat_axis=gather_idx)`` (simgroup.py:453-456,
    313-335).  Its backward is the same call with the indices swapped --
    the reference's self-inverse law (test_simgroup.py:166-176).
  * ``DistributedAttention.forward(q, k, v)`` == the core of
    ``ulysses_attention_forward_with_state`` between the projections
    (ulysses.py:144-154): 3x seq->head, per-head ``kernel``, 1x head->seq.
    Its backward mirrors ``ulysses_attention_backward`` (ulysses.py:
    213-226): dctx seq->head, per-head backward, 3x head->seq.
  * ``local_attn`` is the kernel plugin ``kernel(q, k, v, mask, scale)``
    (kernels.py:31-52, registry kernels.py:114-128); ``FlashAttention``
    is this framework's implementation on full-sequence, head-sharded
    ``[n, b, h/P, hd]`` tensors (bf16: tcgen05/TMEM/TMA; fp32: SIMT).

Inputs are the reference's sequence-major ``[s/P, b, h, hd]`` shards
(ulysses.py:47-48).  When ``local_attn`` is a ``FlashAttention`` the whole
layer runs as one autograd node with fused launches: Q, K and V share one
seq->head exchange; dQ, dK and dV share one head->seq exchange.
"""

from __future__ import annotations

import math

import torch

from . import _lib
from .comm import SequenceGroup, slot_need
from .errors import DegenerateRowError, DivisibilityError, ForwardStateError, KernelError

_ATTN_DTYPES = {torch.float32: _lib.DTYPE_F32, torch.bfloat16: _lib.DTYPE_BF16}


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


_SCHED = {}


def _sched_counter(t: torch.Tensor):
    """Work counter of the persistent forward (UL_ATTN_SCHED_BYTES of zeroed
    device memory, one per (device, stream): launches sharing it must be
    stream-ordered).  None -- the static schedule -- under stream capture."""
    if torch.cuda.is_current_stream_capturing():
        return None
    s = torch.cuda.current_stream(t.device)
    key = (t.device.index, s.stream_id)
    c = _SCHED.get(key)
    if c is None:
        c = torch.zeros(_lib.ATTN_SCHED_BYTES // 4, dtype=torch.int32, device=t.device)
        _SCHED[key] = c
    return c.data_ptr()


_PG_GROUPS = {}


def _group(group) -> SequenceGroup:
    """sequence_process_group: a SequenceGroup, a torch.distributed
    ProcessGroup (wrapped once -- a collective over its ranks -- and cached),
    or None (P = 1)."""
    if group is None:
        return SequenceGroup.single()
    if isinstance(group, SequenceGroup):
        return group
    import torch.distributed as dist
    if isinstance(group, dist.ProcessGroup):
        key = id(group)
        hit = _PG_GROUPS.get(key)
        if hit is None or hit[0] is not group:
            hit = (group, SequenceGroup.from_process_group(group))
            _PG_GROUPS[key] = hit
        return hit[1]
    raise TypeError("sequence_process_group must be a SequenceGroup or a torch.distributed ProcessGroup, "
                    f"got {type(group).__name__}")


# ---------------------------------------------------------------------------
# seq_all_to_all
# ---------------------------------------------------------------------------

class _SeqAllToAll(torch.autograd.Function):
    @staticmethod
    def forward(ctx, group, x, scatter_idx, gather_idx, label):
        ctx.group, ctx.scatter_idx, ctx.gather_idx, ctx.label = group, scatter_idx, gather_idx, label
        return group.all_to_all([x], scatter_idx, gather_idx, label=label)[0]

    @staticmethod
    def backward(ctx, grad):
        g = _SeqAllToAll.apply(ctx.group, grad.contiguous(), ctx.gather_idx, ctx.scatter_idx,
                               ctx.label + ".bwd")
        return None, g, None, None, None


def seq_all_to_all(input: torch.Tensor, scatter_idx: int, gather_idx: int, group=None,
                   label: str = "all_to_all") -> torch.Tensor:
    """All-to-all over the sequence-parallel group: split ``input`` into P
    chunks along ``scatter_idx``, send chunk i to rank i, concatenate the
    received chunks in rank order along ``gather_idx`` (simgroup.py:322-327).
    Bit-exact routing; differentiable (backward swaps the indices)."""
    return _SeqAllToAll.apply(_group(group), input, scatter_idx, gather_idx, label)


# ---------------------------------------------------------------------------
# local attention plugin
# ---------------------------------------------------------------------------

class FlashAttention:
    """Local-attention plugin on head-sharded ``[n, b, h, hd]`` tensors.

    ``mask`` is "causal" (causal_kernel, kernels.py:49-52) or "none"
    (dense_kernel, kernels.py:43-46); ``scale`` defaults to 1/sqrt(hd)
    (AttentionSpec.scale, layers.py:51).  K/V may carry fewer heads than Q
    (GQA: query head h reads kv head h // (hq/hkv)).

    ``deterministic=False`` (default) runs the bf16 hd-128 backward as one
    fused kernel whose dQ is accumulated with fp32 atomics (last-bit run to
    run variation, within the stated tolerance); ``True`` selects the
    two-kernel backward (dQ kernel recomputes S and dP, no atomics) whose
    gradients are bitwise reproducible and bitwise P-invariant.
    """

    def __init__(self, mask: str = "causal", scale: float | None = None, deterministic: bool = False,
                 block_size: int | None = None, pattern=None):
        if mask not in ("causal", "none", "blocked"):
            raise KernelError(f"kernel supports dense/causal/blocked masks only, got {mask!r}")
        self.mask = mask
        self.scale = scale
        self.deterministic = bool(deterministic)
        if mask == "blocked":
            # Mask.blocked(block_size, pattern) (tensor.py:147-149) + blocked_kernel
            # (kernels.py:55-86): query block qb sees the key blocks kb with
            # (qb, kb) in pattern, every key inside a visible block
            if block_size is None or pattern is None:
                raise KernelError("blocked kernel needs block_size and pattern")
            self.block_size = int(block_size)
            self.pattern = frozenset((int(a), int(b)) for a, b in pattern)
            self._build_bits()
        elif block_size is not None or pattern is not None:
            raise KernelError(f"block_size/pattern apply to the blocked kernel, not {mask!r}")

    def _workspace(self, t, n, b, hq, hkv, hd, dt):
        """The backward workspace (L2/D rows and, for the fused hd-128
        kernel, its fp32 dQ accumulator), allocated on the calling stream."""
        need = max(int(_lib.lib().ul_attn_bwd_workspace_bytes(n, b, hq, hkv, hd, dt)), 16)
        return torch.empty(need, dtype=torch.uint8, device=t.device)

    @property
    def flags(self) -> int:
        """Per-call backward flags of the C-ABI (UL_ATTN_DETERMINISTIC)."""
        return _lib.ATTN_DETERMINISTIC if self.deterministic else 0

    @property
    def mask_code(self) -> int:
        return {"causal": _lib.MASK_CAUSAL, "none": _lib.MASK_NONE, "blocked": _lib.MASK_BLOCKED}[self.mask]

    def _pattern_bits(self, n: int, device) -> torch.Tensor:
        """Validate the pattern for sequence length n with blocked_kernel's
        rules and order (kernels.py:63-80) and return its device bitmap
        (uint32 rows of ceil(nb/32) words, include/ulysses_b200.h).

        A valid call has exactly nb = (largest block index + 1) blocks (every
        index < nb, every query block present), so the bitmap depends on the
        pattern alone: it is built at construction (``_device_bits``) and
        copied to a device at most once, outside any call when the device is
        current at construction.  No host allocation or copy happens while an
        in-process group's ranks are being issued (a pinned allocation there
        can serialize the device's streams behind a spinning flag wait)."""
        bs = self.block_size
        if bs < 1 or n % bs != 0:
            raise DivisibilityError(f"block_size {bs} does not divide sequence length {n}")
        nb = n // bs
        bad = sorted((qb, kb) for qb, kb in self.pattern if not (0 <= qb < nb and 0 <= kb < nb))
        if bad:
            raise ValueError(f"pattern blocks {bad[:4]} out of range for {nb} blocks")
        seen = {qb for qb, _ in self.pattern}
        empty = [qb for qb in range(nb) if qb not in seen]
        if empty:
            raise DegenerateRowError(f"query block {empty[0]} has no visible key blocks (invalid sparse pattern)")
        assert nb == self._nb
        return self._device_bits(device), self._words, self._host_bits

    def _build_bits(self):
        nb = 1 + max((max(a, b) for a, b in self.pattern), default=-1)
        words = max(1, (nb + 31) // 32)
        bits = [0] * (max(nb, 1) * words)
        for qb, kb in self.pattern:
            if qb >= 0 and kb >= 0:
                bits[qb * words + kb // 32] |= 1 << (kb % 32)
        self._nb, self._words = nb, words
        self._host_bits = torch.tensor(bits, dtype=torch.int64).to(torch.int32)   # (bit 31 wraps: same bits)
        self._bits = {}
        if torch.cuda.is_available():
            self._device_bits(torch.device("cuda", torch.cuda.current_device()))

    def _device_bits(self, device) -> torch.Tensor:
        device = torch.device(device)
        t = self._bits.get(device.index)
        if t is None:
            # (a blocking copy from pageable memory, on a private stream)
            side = torch.cuda.Stream(device=device)
            with torch.cuda.stream(side):
                t = self._host_bits.to(device)
            side.synchronize()
            self._bits[device.index] = t
        return t

    def _check(self, q, k, v):
        if q.dim() != 4 or k.dim() != 4 or v.dim() != 4:
            raise KernelError(f"kernel needs (n, b, h, hdim) tensors, got {tuple(q.shape)}, "
                              f"{tuple(k.shape)}, {tuple(v.shape)}")
        n, b, hq, hd = q.shape
        if k.shape != v.shape or k.shape[0] != n or k.shape[1] != b or k.shape[3] != hd:
            raise KernelError(f"kernel needs matching (n, b, hdim) views, got {tuple(q.shape)}, "
                              f"{tuple(k.shape)}, {tuple(v.shape)}")
        if q.dtype not in _ATTN_DTYPES or k.dtype != q.dtype or v.dtype != q.dtype:
            raise KernelError(f"attention computes in float32 or bfloat16, got {q.dtype}")
        if k.shape[2] < 1 or hq % k.shape[2] != 0:
            raise DivisibilityError(f"kv head count {k.shape[2]} does not divide query head count {hq}")
        if not (q.is_cuda and k.is_cuda and v.is_cuda):
            raise KernelError("FlashAttention runs on CUDA tensors only (no CPU path)")
        return n, b, hq, k.shape[2], hd

    def _scale(self, hd):
        return float(self.scale) if self.scale is not None else 1.0 / math.sqrt(hd)

    def forward_with_lse(self, q, k, v):
        n, b, hq, hkv, hd = self._check(q, k, v)
        q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
        o = torch.empty_like(q)
        lse = torch.empty((b, hq, n), dtype=torch.float32, device=q.device)
        if self.mask == "blocked":
            bits, words, _ = self._pattern_bits(n, q.device)
            _lib.check(_lib.lib().ul_attn_fwd_blocked(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                                                      lse.data_ptr(), n, b, hq, hkv, hd, _ATTN_DTYPES[q.dtype],
                                                      self.block_size, bits.data_ptr(), words, self._scale(hd),
                                                      _stream(q)))
            return o, lse
        _lib.check(_lib.lib().ul_attn_fwd(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                                          lse.data_ptr(), n, b, hq, hkv, hd, _ATTN_DTYPES[q.dtype],
                                          self.mask_code, self._scale(hd), _sched_counter(q), _stream(q)))
        return o, lse

    def _backward_mask_check(self):
        if self.mask == "blocked":   # kernels.py:95-96
            raise KernelError("backward supports dense/causal masks only, got 'blocked'")

    def backward(self, q, k, v, o, lse, do):
        self._backward_mask_check()
        if lse is None:
            raise ForwardStateError("backward needs the state saved by the forward pass")
        n, b, hq, hkv, hd = self._check(q, k, v)
        if o.shape != q.shape or do.shape != q.shape or tuple(lse.shape) != (b, hq, n):
            raise ForwardStateError(f"grad shape {tuple(do.shape)} does not match saved forward "
                                    f"shape {tuple(o.shape)}")
        q, k, v, o, do = (x.contiguous() for x in (q, k, v, o, do))
        dq = torch.empty_like(q)
        dk = torch.empty_like(k)
        dv = torch.empty_like(v)
        dt = _ATTN_DTYPES[q.dtype]
        ws = self._workspace(q, n, b, hq, hkv, hd, dt)
        _lib.check(_lib.lib().ul_attn_bwd(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                                          do.data_ptr(), lse.data_ptr(), dq.data_ptr(), dk.data_ptr(),
                                          dv.data_ptr(), ws.data_ptr(), ws.numel(), n, b, hq, hkv, hd,
                                          dt, self.mask_code, self._scale(hd), self.flags, _stream(q)))
        return dq, dk, dv

    # -- fused head->seq exchange (K2 in the kernels' epilogues) ------------
    def forward_exchange(self, q, k, v, group: SequenceGroup, label: str = "attn.ctx.head2seq",
                         ledger_elements: int | None = None):
        """Forward on head-sharded q/k/v [N, b, h, hd] plus the head->seq
        exchange of O fused into the kernel epilogue.  Returns (o_head, lse,
        o_seq) with o_seq = seq layout [N/P, b, P*h, hd] of this rank."""
        from .comm import label_hash
        if self.mask == "blocked":   # (no fused epilogue for the blocked kernel: two steps)
            o, lse = self.forward_with_lse(q, k, v)
            (o_seq,) = group.all_to_all([o], 0, 2, label=label)
            return o, lse, o_seq
        n, b, hq, hkv, hd = self._check(q, k, v)
        q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
        p = group.world
        o = torch.empty_like(q)
        lse = torch.empty((b, hq, n), dtype=torch.float32, device=q.device)
        o_seq = torch.empty((n // p, b, hq * p, hd), dtype=q.dtype, device=q.device)
        group.ensure_slot(slot_need([o_seq.numel() * o_seq.element_size()]))
        _lib.check(_lib.lib().ul_attn_fwd_exchange(group._handle, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                                   o.data_ptr(), lse.data_ptr(), o_seq.data_ptr(), n, b, hq, hkv,
                                                   hd, _ATTN_DTYPES[q.dtype], self.mask_code, self._scale(hd),
                                                   label_hash(label), _sched_counter(q), _stream(q)))
        if ledger_elements != 0:
            group._record(label, o.numel() if ledger_elements is None else ledger_elements)
        return o, lse, o_seq

    def backward_exchange(self, q, k, v, o, lse, do, group: SequenceGroup, label: str = "bwd.qkv.head2seq",
                          return_head: bool = False, ledger_scale: int = 1):
        """Backward with the head->seq exchange of dQ/dK/dV fused into the
        epilogues.  Returns sequence-layout (dq, dk, dv) of this rank (and
        the head-layout gradients the kernels also wrote, if return_head)."""
        from .comm import label_hash
        self._backward_mask_check()
        if lse is None:
            raise ForwardStateError("backward needs the state saved by the forward pass")
        n, b, hq, hkv, hd = self._check(q, k, v)
        q, k, v, o, do = (x.contiguous() for x in (q, k, v, o, do))
        p = group.world
        dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
        sq = torch.empty((n // p, b, hq * p, hd), dtype=q.dtype, device=q.device)
        sk = torch.empty((n // p, b, hkv * p, hd), dtype=q.dtype, device=q.device)
        sv = torch.empty_like(sk)
        dt = _ATTN_DTYPES[q.dtype]
        ws = self._workspace(q, n, b, hq, hkv, hd, dt)
        group.ensure_slot(slot_need(t.numel() * t.element_size() for t in (sq, sk, sv)))
        _lib.check(_lib.lib().ul_attn_bwd_exchange(group._handle, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                                   o.data_ptr(), do.data_ptr(), lse.data_ptr(), dq.data_ptr(),
                                                   dk.data_ptr(), dv.data_ptr(), ws.data_ptr(), ws.numel(),
                                                   sq.data_ptr(), sk.data_ptr(), sv.data_ptr(), n, b, hq, hkv, hd,
                                                   dt, self.mask_code, self._scale(hd), label_hash(label),
                                                   self.flags, _stream(q)))
        if ledger_scale:   # (a pipelined layer records its G group calls once, scaled by G)
            for name, t in (("bwd.q.head2seq", dq), ("bwd.k.head2seq", dk), ("bwd.v.head2seq", dv)):
                group._record(name, t.numel() * ledger_scale)
        if return_head:
            return (sq, sk, sv), (dq, dk, dv)
        return sq, sk, sv

    def __call__(self, q, k, v):
        return _LocalAttnFn.apply(self, q, k, v)


class _LocalAttnFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, attn, q, k, v):
        o, lse = attn.forward_with_lse(q, k, v)
        ctx.attn = attn
        ctx.save_for_backward(q, k, v, o, lse)
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, o, lse = ctx.saved_tensors
        dq, dk, dv = ctx.attn.backward(q, k, v, o, lse, do)
        return None, dq, dk, dv


def _blocked_kernel(block_size: int, pattern) -> FlashAttention:
    return FlashAttention("blocked", block_size=block_size, pattern=pattern)


# kernels.py:114-128.  The reference's kernels take the mask per call; here the
# mask is part of the plugin, so "blocked" maps to a factory taking
# (block_size, pattern) -- get_kernel("blocked", block_size=..., pattern=...).
KERNELS = {"dense": FlashAttention("none"), "causal": FlashAttention("causal"), "blocked": _blocked_kernel}


def get_kernel(name: str, **mask_args):
    """kernels.py:124-128."""
    try:
        k = KERNELS[name]
    except KeyError:
        raise KernelError(f"unknown kernel {name!r}, expected one of {sorted(KERNELS)}") from None
    if name == "blocked":
        if not mask_args:
            raise KernelError("the blocked kernel needs block_size and pattern: "
                              "get_kernel('blocked', block_size=bs, pattern=pairs)")
        return k(**mask_args)
    if mask_args:
        raise KernelError(f"kernel {name!r} takes no mask arguments")
    return k


# ---------------------------------------------------------------------------
# DistributedAttention
# ---------------------------------------------------------------------------

def _bytes(shape, dtype) -> int:
    n = 1
    for x in shape:
        n *= int(x)
    return n * torch.empty((), dtype=dtype).element_size()


def _presize(group: SequenceGroup, main_need: int, chan_need: int = 0):
    """Size the receive slots of every exchange a layer call will issue
    BEFORE issuing the first one: a regrowth then never happens while this
    rank already has flag waits queued (for an in-process group those waits
    can only be satisfied by peers the host has not issued yet, and the
    workspace allocation of a regrowth may serialize the device behind them)."""
    group.ensure_slot(main_need)
    if chan_need:
        group.channel.ensure_slot(chan_need)


class _UlyssesAttnFn(torch.autograd.Function):
    """Whole-layer node: fused QKV seq->head, local attention, O head->seq."""

    @staticmethod
    def forward(ctx, group, attn, scatter_idx, gather_idx, q, k, v):
        if group.world > 1 and (scatter_idx, gather_idx) == (2, 0):
            p = group.world
            nl, b, hq, hd = q.shape
            hkv = k.shape[2]
            _presize(group, max(slot_need([_bytes((nl * p, b, hq // p, hd), q.dtype)] +
                                          [_bytes((nl * p, b, hkv // p, hd), q.dtype)] * 2),
                                slot_need([_bytes(q.shape, q.dtype)])))
        if group.world > 1:
            q4, k4, v4 = group.all_to_all([q, k, v], scatter_idx, gather_idx, label="attn.qkv.seq2head",
                                          labels=["attn.q.seq2head", "attn.k.seq2head", "attn.v.seq2head"])
        else:
            q4, k4, v4 = q.contiguous(), k.contiguous(), v.contiguous()
        if group.world > 1:
            # head->seq of O fused into the attention epilogue (K2 in K3)
            o4, lse, o = attn.forward_exchange(q4, k4, v4, group, label="attn.ctx.head2seq")
        else:
            o4, lse = attn.forward_with_lse(q4, k4, v4)
            o = o4
        ctx.group, ctx.attn, ctx.idx = group, attn, (scatter_idx, gather_idx)
        ctx.save_for_backward(q4, k4, v4, o4, lse)
        return o

    @staticmethod
    def backward(ctx, do):
        group, attn = ctx.group, ctx.attn
        scatter_idx, gather_idx = ctx.idx
        q4, k4, v4, o4, lse = ctx.saved_tensors
        do = do.contiguous()
        if group.world > 1 and (scatter_idx, gather_idx) == (2, 0):
            _presize(group, max(slot_need([_bytes(q4.shape, q4.dtype)]),
                                slot_need([_bytes(q4.shape, q4.dtype)] + [_bytes(k4.shape, k4.dtype)] * 2)))
        if group.world > 1:
            (do4,) = group.all_to_all([do], scatter_idx, gather_idx, label="bwd.ctx.seq2head")
        else:
            do4 = do
        if group.world > 1:
            # head->seq of dQ, dK, dV fused into the backward kernels' epilogues
            dq, dk, dv = attn.backward_exchange(q4, k4, v4, o4, lse, do4, group, label="bwd.qkv.head2seq")
        else:
            dq, dk, dv = attn.backward(q4, k4, v4, o4, lse, do4)
        return None, None, None, None, dq, dk, dv


def _interleave(parts, p: int):
    """Per-head-group sequence outputs [nl, b, P*Hg, hd] (heads ordered
    (rank, h)) -> the layer's [nl, b, P*G*Hg, hd] with head r*Hl + g*Hg + h."""
    nl, b, ph, hd = parts[0].shape
    hg = ph // p
    return torch.stack([x.view(nl, b, p, hg, hd) for x in parts], dim=3).view(nl, b, p * len(parts) * hg, hd)


class _UlyssesAttnPipeFn(torch.autograd.Function):
    """The layer node with the exchanges pipelined over G head groups
    (north star item 3).  The seq->head exchange of group g+1 runs on the
    group's second channel and stream while group g is attended on the
    compute stream (its head->seq exchange fused into the attention
    epilogue, main channel); the backward does the same with dO.  Every
    group is the reference's layer on a subset of heads (attention is
    independent per head, ulysses.py:148-152), so the result is the one of
    _UlyssesAttnFn; the per-group sequence outputs are interleaved back into
    the [s/P, b, h, hd] layout."""

    @staticmethod
    def forward(ctx, group, attn, G, q, k, v):
        p = group.world
        chan = group.channel
        main = torch.cuda.current_stream(q.device)
        cs = chan.stream
        q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
        nl, b, hq, hd = q.shape
        hkv = k.shape[2]
        hg, hkg = hq // (p * G), hkv // (p * G)
        _presize(group, slot_need([_bytes((nl, b, p * hg, hd), q.dtype)]),
                 slot_need([_bytes((nl * p, b, hg, hd), q.dtype)] + [_bytes((nl * p, b, hkg, hd), q.dtype)] * 2))
        cs.wait_stream(main)
        heads, evs = [], []
        with torch.cuda.stream(cs):
            for t in (q, k, v):
                t.record_stream(cs)
            for gi in range(G):
                heads.append(chan.all_to_all_head_group(
                    [q, k, v], gi, G, label="attn.qkv.seq2head",
                    labels=["attn.q.seq2head", "attn.k.seq2head", "attn.v.seq2head"]))
                ev = torch.cuda.Event()
                ev.record(cs)
                evs.append(ev)
        outs, saved = [], []
        for gi in range(G):
            main.wait_event(evs[gi])
            q4, k4, v4 = heads[gi]
            for t in (q4, k4, v4):
                t.record_stream(main)
            o4, lse, o_seq = attn.forward_exchange(q4, k4, v4, group, label=f"attn.ctx.head2seq.{gi}/{G}",
                                                   ledger_elements=q.numel() if gi == 0 else 0)
            outs.append(o_seq)
            saved += [q4, k4, v4, o4, lse]
        ctx.group, ctx.attn, ctx.G = group, attn, G
        ctx.save_for_backward(*saved)
        return _interleave(outs, p)

    @staticmethod
    def backward(ctx, do):
        group, attn, G = ctx.group, ctx.attn, ctx.G
        p = group.world
        chan = group.channel
        main = torch.cuda.current_stream(do.device)
        cs = chan.stream
        saved = ctx.saved_tensors
        do = do.contiguous()
        nl, b, hq, hd = do.shape
        hkv = saved[1].shape[2] * p * G
        hg, hkg = hq // (p * G), hkv // (p * G)
        _presize(group, slot_need([_bytes((nl, b, p * hg, hd), do.dtype)] + [_bytes((nl, b, p * hkg, hd), do.dtype)] * 2),
                 slot_need([_bytes((nl * p, b, hg, hd), do.dtype)]))
        cs.wait_stream(main)
        dos, evs = [], []
        with torch.cuda.stream(cs):
            do.record_stream(cs)
            for gi in range(G):
                (do4,) = chan.all_to_all_head_group([do], gi, G, label="bwd.ctx.seq2head")
                ev = torch.cuda.Event()
                ev.record(cs)
                dos.append(do4)
                evs.append(ev)
        dq, dk, dv = [], [], []
        for gi in range(G):
            q4, k4, v4, o4, lse = saved[5 * gi:5 * gi + 5]
            main.wait_event(evs[gi])
            dos[gi].record_stream(main)
            a, b_, c = attn.backward_exchange(q4, k4, v4, o4, lse, dos[gi], group, label=f"bwd.qkv.head2seq.{gi}/{G}",
                                              ledger_scale=G if gi == 0 else 0)
            dq.append(a)
            dk.append(b_)
            dv.append(c)
        return None, None, None, _interleave(dq, p), _interleave(dk, p), _interleave(dv, p)


def pipeline_groups(heads_local: int, kv_heads_local: int, want: int = 2, n: int | None = None,
                    sms: int | None = None) -> int:
    """Head groups of the pipelined layer: the largest g <= want dividing
    both this rank's query and kv head counts (1 = no pipelining) -- and,
    when the full sequence length n is given, only if every group's
    attention still fills the GPU (>= 2 forward work items of two 128-row
    query tiles per SM): splitting a small problem costs more than the
    hidden exchange (r2, tools/inproc_layer.py: P = 4, 16 heads, N = 8K,
    2.49 -> 4.70 ms)."""
    for g in range(max(1, want), 0, -1):
        if heads_local % g == 0 and kv_heads_local % g == 0:
            if g > 1 and n is not None:
                items = ((n + 255) // 256) * (heads_local // g)
                if items < 2 * (sms or _sm_count()):
                    continue
            return g
    return 1


_SMS = {}


def _sm_count() -> int:
    d = torch.cuda.current_device()
    if d not in _SMS:
        _SMS[d] = torch.cuda.get_device_properties(d).multi_processor_count
    return _SMS[d]


class DistributedAttention(torch.nn.Module):
    """Ulysses sequence-parallel attention (arXiv 2309.14509 section 3.1).

    ``forward(query, key, value)`` takes this rank's sequence shards
    ``[s/P, b, h, hd]`` (key/value may have ``h_kv`` heads, GQA) and returns
    the context shard ``[s/P, b, h, hd]``.
    """

    def __init__(self, local_attention, sequence_process_group=None, scatter_idx: int = 2,
                 gather_idx: int = 0, pipeline: int = 2, adaptive_pipeline: bool = True):
        super().__init__()
        self.local_attn = local_attention
        self.spg = _group(sequence_process_group)
        self.scatter_idx = scatter_idx
        self.gather_idx = gather_idx
        # head groups over which the fused route pipelines its exchanges with
        # the attention (P > 1); 1 = one exchange of all heads, then attention
        self.pipeline = int(pipeline)
        # pipeline only problems whose head groups still fill the GPU (False:
        # always split into `pipeline` groups when the head counts allow)
        self.adaptive_pipeline = bool(adaptive_pipeline)

    def _check(self, q, k, v):
        p = self.spg.world
        if q.dim() != 4:
            raise KernelError(f"DistributedAttention needs [s/P, b, h, hd] shards, got {tuple(q.shape)}")
        h = q.shape[self.scatter_idx]
        n = q.shape[self.gather_idx] * p
        if n % p != 0:                                  # layers.py:53-57
            raise DivisibilityError(f"p={p} does not divide sequence length n={n}")
        if h % p != 0:
            raise DivisibilityError(f"p={p} does not divide head count {h}")
        hkv = k.shape[self.scatter_idx]
        if hkv % p != 0:
            raise DivisibilityError(f"p={p} does not divide kv head count {hkv}")

    def forward(self, query, key, value, *args, **kwargs):
        """``*args`` / ``**kwargs`` pass through to ``local_attn`` (the
        DeepSpeed signature); with extra arguments the generic route runs."""
        self._check(query, key, value)
        fused_layout = (self.scatter_idx, self.gather_idx) == (2, 0) or \
            ((self.scatter_idx, self.gather_idx) == (2, 1) and query.shape[0] == 1)
        if isinstance(self.local_attn, FlashAttention) and fused_layout and not args and not kwargs:
            if (self.scatter_idx, self.gather_idx) == (2, 1):      # [1, s, h, d] == [s, 1, h, d]
                q, k, v = (x.reshape(x.shape[1], 1, x.shape[2], x.shape[3]) for x in (query, key, value))
                o = _UlyssesAttnFn.apply(self.spg, self.local_attn, 2, 0, q, k, v)
                return o.reshape(1, o.shape[0], o.shape[2], o.shape[3])
            p = self.spg.world
            G = pipeline_groups(query.shape[2] // p, key.shape[2] // p, self.pipeline,
                                n=query.shape[0] * p if self.adaptive_pipeline else None) if p > 1 else 1
            if G > 1 and (self.scatter_idx, self.gather_idx) == (2, 0):
                return _UlyssesAttnPipeFn.apply(self.spg, self.local_attn, G, query, key, value)
            return _UlyssesAttnFn.apply(self.spg, self.local_attn, self.scatter_idx, self.gather_idx,
                                        query, key, value)
        # generic plugin: any callable local_attn(q, k, v) on head-sharded tensors
        q4 = seq_all_to_all(query, self.scatter_idx, self.gather_idx, self.spg, "attn.q.seq2head")
        k4 = seq_all_to_all(key, self.scatter_idx, self.gather_idx, self.spg, "attn.k.seq2head")
        v4 = seq_all_to_all(value, self.scatter_idx, self.gather_idx, self.spg, "attn.v.seq2head")
        ctx = self.local_attn(q4, k4, v4, *args, **kwargs)
        return seq_all_to_all(ctx, self.gather_idx, self.scatter_idx, self.spg, "attn.ctx.head2seq")
