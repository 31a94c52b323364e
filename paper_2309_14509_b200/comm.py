"""The sequence-parallel group: identity, peer-mapped workspace, all-to-all.

``SequenceGroup`` is this framework's ``sequence_process_group``.  It plays
the role of the reference's ``RankContext`` over a ``RankGroup``
(simgroup.py:198-224, 444-468), except that ranks are processes on
different GPUs (``from_process_group``) -- or, for single-GPU parity tests,
``world`` ranks driven from one process on one device, each on its own
CUDA stream (``local_group``).  Both run the same native kernels: fused
permute + NVLink peer stores + release/acquire flags (csrc/a2a.cu).

Plumbing only goes through torch.distributed (exchanging IPC handles at
setup); the data path never calls NCCL.
"""

from __future__ import annotations

import atexit
import ctypes
import struct
from dataclasses import dataclass

import torch

from . import _lib
from .errors import GroupDesyncError, ShardError

_DTYPES = {torch.float32: _lib.DTYPE_F32, torch.bfloat16: _lib.DTYPE_BF16}

DEFAULT_SLOT_BYTES = 64 << 20
CHANNEL_SLOT_BYTES = 1 << 20   # the prefetch channel starts small and grows on demand
SLOT_GRANULE = 16 << 20      # receive slots grow in multiples of this


def slot_need(byte_counts) -> int:
    """Receive-slot bytes a call with these per-tensor output sizes needs
    (each tensor image 256-byte aligned, csrc/a2a.cu plan_call)."""
    return sum((int(n) + 255) // 256 * 256 for n in byte_counts)

# layout of one rank's handle blob (csrc/a2a.cu HandleBlob): IPC handle,
# magic, slot bytes, rank, world -- padded to UL_IPC_HANDLE_BYTES
HANDLE_STRUCT = struct.Struct("<64sQQii")
HANDLE_MAGIC = 0x554C595353455332


def pack_handle(ipc_handle: bytes, slot_bytes: int, rank: int, world: int) -> bytes:
    blob = HANDLE_STRUCT.pack(ipc_handle.ljust(64, b"\0")[:64], HANDLE_MAGIC, slot_bytes, rank, world)
    return blob.ljust(_lib.IPC_HANDLE_BYTES, b"\0")


def gather_handles(blob: bytes, pg=None) -> bytes:
    """Rendezvous: every rank contributes its handle blob; returns all blobs
    concatenated in rank order (the only collective on the setup path)."""
    import torch.distributed as dist
    world = dist.get_world_size(pg)
    gathered = [None] * world
    dist.all_gather_object(gathered, bytes(blob), group=pg)
    return b"".join(gathered)


def validate_handles(all_blobs: bytes, world: int, rank: int, slot_bytes: int):
    """Raise GroupDesyncError if the gathered blobs disagree (rank order,
    group size, workspace geometry)."""
    buf = ctypes.create_string_buffer(bytes(all_blobs), len(all_blobs))
    _lib.check(_lib.lib().ul_comm_validate_handles(buf, world, rank, slot_bytes))


def label_hash(label: str) -> int:
    h = 1469598103934665603
    for ch in label.encode():
        h ^= ch
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def dtype_code(dtype: torch.dtype) -> int:
    try:
        return _DTYPES[dtype]
    except KeyError:
        from .errors import KernelError
        raise KernelError(f"all_to_all supports float32/bfloat16 payloads, got {dtype}") from None


def a2a_out_shape(shape, p: int, split_axis: int, concat_axis: int) -> tuple:
    """Output shape of simgroup.py:322-327's combine for one rank."""
    shape = list(shape)
    if shape[split_axis] % p != 0:
        raise ShardError(f"all_to_all split axis {split_axis} (length {shape[split_axis]}) "
                         f"not divisible by p={p}")
    shape[split_axis] //= p
    if split_axis != concat_axis:
        shape[concat_axis] *= p
    return tuple(shape)


@dataclass(frozen=True)
class CommRecord:
    """One logical all_to_all, as the reference ledger records it
    (CommRecord, simgroup.py:70-85), in elements."""
    collective: str
    step_label: str
    aggregate_elements: int
    per_rank_egress_elements: int


LEDGER_CSV_COLUMNS = ["step_label", "collective", "aggregate_elements", "per_rank_egress_elements"]  # simgroup.py:54-59


class CommLedger(list):
    """Append-only list of CommRecord with the reference ledger's queries and
    exports (CommLedger, simgroup.py:88-172; CSV/JSON in its schema)."""

    def select(self, collective=None, step_label=None):
        return tuple(r for r in self if (collective is None or r.collective == collective)
                     and (step_label is None or r.step_label == step_label))

    def count(self, collective=None, step_label=None) -> int:
        return len(self.select(collective, step_label))

    def total_egress(self, collective=None, step_label=None) -> int:
        return sum(r.per_rank_egress_elements for r in self.select(collective, step_label))

    def total_aggregate(self, collective=None, step_label=None) -> int:
        return sum(r.aggregate_elements for r in self.select(collective, step_label))

    def counts_by_collective(self) -> dict:
        out = {}
        for r in self:
            out[r.collective] = out.get(r.collective, 0) + 1
        return out

    def egress_by_collective(self) -> dict:
        out = {}
        for r in self:
            out[r.collective] = out.get(r.collective, 0) + r.per_rank_egress_elements
        return out

    def rows(self) -> list:
        return [[r.step_label, r.collective, r.aggregate_elements, r.per_rank_egress_elements] for r in self]

    def to_json_obj(self) -> list:
        return [dict(zip(LEDGER_CSV_COLUMNS, row)) for row in self.rows()]

    def to_csv_text(self) -> str:
        import csv
        import io
        buf = io.StringIO()
        w = csv.writer(buf, lineterminator="\n")
        w.writerow(LEDGER_CSV_COLUMNS)
        w.writerows(self.rows())
        return buf.getvalue()

    def write_csv(self, path: str) -> str:
        with open(path, "w") as f:
            f.write(self.to_csv_text())
        return path

    def write_json(self, path: str) -> str:
        import json
        with open(path, "w") as f:
            json.dump(self.to_json_obj(), f, indent=2)
        return path


def check_ledger(ledger, n: int, b: int, d: int, p: int, layers: int = 1, backward: bool = False):
    """verify.check_ledger (verify.py:146-169) for the Ulysses scheme, zero
    tolerance: total per-rank egress == the exact-convention volume
    (costmodel.py:82-87) x layers (x2 with the backward's mirrored
    exchanges), 4 all_to_all per layer per direction (LEDGER_SHAPE,
    verify.py:43-47), every record of aggregate n*b*d.  Returns
    (ok, measured, predicted)."""
    from fractions import Fraction
    flips = 2 if backward else 1
    predicted = Fraction(4 * n * b * d) * (p - 1) / (p * p) * layers * flips
    measured = ledger.total_egress()
    counts_ok = ledger.counts_by_collective() == ({"all_to_all": 4 * layers * flips} if len(ledger) or layers else {})
    records_ok = all(r.aggregate_elements == n * b * d for r in ledger)
    return bool(measured == predicted and counts_ok and records_ok), int(measured), int(predicted)


_GRAVEYARD = []   # workspaces of collected SequenceGroups, released at a safe point


def reap_workspaces():
    """Release the workspaces of garbage-collected groups (a device sync).
    Called when a group is created and at exit -- points where no rank of an
    in-process group is half issued."""
    while _GRAVEYARD:
        _lib.lib().ul_comm_destroy(_GRAVEYARD.pop())


atexit.register(reap_workspaces)


class SequenceGroup:
    """One rank of a P-way Ulysses sequence-parallel group."""

    def __init__(self, rank: int, world: int, device: int, handle, slot_bytes: int,
                 stream: torch.cuda.Stream | None = None, pg=None, local=None):
        self.rank = rank
        self.world = world
        self.p = world                      # reference spelling (RankContext.p)
        self.device = device
        self._handle = handle               # ul_comm* (None for world == 1)
        self.slot_bytes = slot_bytes
        self.stream = stream
        self._pg = pg
        # in-process group: weak references to every rank's SequenceGroup (no
        # reference cycle: a group must be freed by refcount, deterministically
        # -- a cyclic-GC collection that destroys a group (device sync) while
        # another group's ranks are being issued would deadlock them)
        self._local = local
        self._timeout_ms = None
        # second exchange channel of the same ranks (own workspace, epochs and
        # stream) for the pipelined layer's prefetch exchanges; see `channel`
        self._channel = None
        # in-process regrowth: workspaces this rank switched away from, and
        # new generations prepared by a peer that this rank has not reached
        self._retired, self._pending = [], []
        self.records: CommLedger = CommLedger()   # the logical ledger (elements, reference schema)
        self.ledger = self.records

    # -- construction ------------------------------------------------------
    @staticmethod
    def _create(rank, world, device, slot_bytes):
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().ul_comm_create(rank, world, device, slot_bytes, ctypes.byref(h)))
        return h

    @classmethod
    def single(cls, device: int | None = None) -> "SequenceGroup":
        """P = 1: the seq<->head flips are identities (ulysses.py:104-111 at P=1)."""
        if device is None:
            device = torch.cuda.current_device()
        return cls(0, 1, device, None, 0)

    @classmethod
    def from_process_group(cls, pg=None, slot_bytes: int = DEFAULT_SLOT_BYTES,
                           device: int | None = None, timeout_ms: int | None = None) -> "SequenceGroup":
        """Collective: every rank of ``pg`` (a torch.distributed group, any
        backend) allocates its workspace and maps every peer's over CUDA IPC."""
        import torch.distributed as dist
        reap_workspaces()
        rank = dist.get_rank(pg)
        world = dist.get_world_size(pg)
        if device is None:
            device = torch.cuda.current_device()
        if world == 1:
            return cls.single(device)
        h = cls._open_ipc(rank, world, device, slot_bytes, pg)
        g = cls(rank, world, device, h, int(_lib.lib().ul_comm_slot_bytes(h)), pg=pg)
        hc = cls._open_ipc(rank, world, device, CHANNEL_SLOT_BYTES, pg)
        g._channel = cls(rank, world, device, hc, int(_lib.lib().ul_comm_slot_bytes(hc)), pg=pg,
                         stream=torch.cuda.Stream(device=device))
        g._channel.records = g._channel.ledger = g.records   # one logical ledger for both channels
        if timeout_ms:
            g.set_timeout_ms(timeout_ms)
        dist.barrier(group=pg)
        return g

    @classmethod
    def _open_ipc(cls, rank, world, device, slot_bytes, pg):
        h = cls._create(rank, world, device, slot_bytes)
        blob = ctypes.create_string_buffer(_lib.IPC_HANDLE_BYTES)
        _lib.check(_lib.lib().ul_comm_export_handle(h, blob))
        all_blobs = gather_handles(blob.raw, pg)
        allb = ctypes.create_string_buffer(all_blobs, world * _lib.IPC_HANDLE_BYTES)
        _lib.check(_lib.lib().ul_comm_open_peers(h, allb))
        return h

    @classmethod
    def local_group(cls, world: int, slot_bytes: int = DEFAULT_SLOT_BYTES,
                    device: int | None = None) -> list["SequenceGroup"]:
        """``world`` ranks in this process on one GPU, one stream each.  The
        peer pointers are plain device pointers, so the exact kernels of the
        multi-GPU path (incl. flag waits) run at P = 2/4/8 on one B200.
        Calls of different ranks must be issued on their own ``stream``."""
        if device is None:
            device = torch.cuda.current_device()
        if world == 1:
            return [cls.single(device)]
        reap_workspaces()
        local = cls._make_local(world, device, slot_bytes)
        chans = cls._make_local(world, device, CHANNEL_SLOT_BYTES)
        for g, c in zip(local, chans):
            g._channel = c
            c.records = c.ledger = g.records   # one logical ledger for both channels
        return local

    @classmethod
    def _make_local(cls, world, device, slot_bytes):
        import weakref
        handles = cls._link_local(world, device, slot_bytes)
        sb = int(_lib.lib().ul_comm_slot_bytes(handles[0]))
        refs = []
        groups = [cls(r, world, device, handles[r], sb, stream=torch.cuda.Stream(device=device), local=refs)
                  for r in range(world)]
        refs.extend(weakref.ref(g) for g in groups)
        return groups

    @classmethod
    def _link_local(cls, world, device, slot_bytes):
        handles = [cls._create(r, world, device, slot_bytes) for r in range(world)]
        arr = (ctypes.c_void_p * world)(*[h.value for h in handles])
        _lib.check(_lib.lib().ul_comm_link_local(arr, world))
        return handles

    def set_timeout_ms(self, ms: int):
        if self._handle is not None:
            _lib.check(_lib.lib().ul_comm_set_timeout_ms(self._handle, int(ms)))
            self._timeout_ms = int(ms)
        if self._channel is not None:
            self._channel.set_timeout_ms(ms)

    @property
    def channel(self) -> "SequenceGroup":
        """The group's second exchange channel: the same ranks with their own
        workspace, epochs and stream (``channel.stream``).  The pipelined
        layer issues the seq->head exchange of head group g+1 there while
        the attention of group g (and its fused head->seq exchange on this,
        the main channel) runs on the compute stream.  Each channel is used
        from one stream, which is what the two-slot epoch protocol relies on
        (csrc/a2a.cu: a sender reuses a slot only after passing the next
        call's wait)."""
        if self._channel is None:
            raise RuntimeError("this SequenceGroup has no second channel (P = 1)")
        return self._channel

    # -- receive-slot sizing -------------------------------------------------
    def ensure_slot(self, need: int):
        """Grow the receive slots to at least `need` bytes before a call.

        Every rank issues the same calls with the same shapes, so every rank
        reaches the same decision at the same call; the regrowth is then a
        collective re-registration: all previous calls complete (a device
        sync -- their flag waits mean every peer finished writing into the
        old slots), the old workspace is released, a larger one is created
        and mapped by every peer (IPC handles over the process group, or
        direct pointers for an in-process group), and epochs restart at 0 on
        every rank."""
        if self._handle is None or need <= self.slot_bytes:
            return
        new = (int(need) + SLOT_GRANULE - 1) // SLOT_GRANULE * SLOT_GRANULE
        if self._local is not None:
            self._grow_local(need, new)
            return
        import torch.distributed as dist
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self._pg)           # every peer is done with the old slots
        self.destroy(with_channel=False)
        self._handle = self._open_ipc(self.rank, self.world, self.device, new, self._pg)
        self.slot_bytes = int(_lib.lib().ul_comm_slot_bytes(self._handle))
        if self._timeout_ms:
            self.set_timeout_ms(self._timeout_ms)
        dist.barrier(group=self._pg)

    def _grow_local(self, need: int, new: int):
        """In-process regrowth without a device sync.  The host issues the
        ranks of a local group one after the other, so when this rank reaches
        the call, its peers may not have issued their earlier calls yet, and
        this rank's own streams may hold flag waits that only those calls
        satisfy: a synchronize here would deadlock them (and a swap of every
        rank's handle now would move the peers' earlier calls onto the new
        workspace).  Instead each regrowth creates one new generation of
        linked workspaces; every rank switches to the next generation when
        IT reaches a call that does not fit -- the same call on every rank,
        since all ranks issue the same calls from the same slot size -- and
        the replaced workspaces are released with the group (their last
        calls may still be in flight)."""
        while self._pending and need > self.slot_bytes:
            self._switch(*self._pending.pop(0))
        if need <= self.slot_bytes:
            return
        peers = [ref() for ref in self._local]
        if any(g is None for g in peers):
            raise RuntimeError("in-process group: a rank's SequenceGroup was freed; cannot regrow")
        handles = self._link_local(self.world, self.device, new)
        sb = int(_lib.lib().ul_comm_slot_bytes(handles[0]))
        for g, h in zip(peers, handles):
            if g is self:
                self._switch(h, sb)
            else:
                g._pending.append((h, sb))

    def _switch(self, handle, slot_bytes: int):
        if self._handle is not None:
            self._retired.append(self._handle)
        self._handle, self.slot_bytes = handle, slot_bytes
        if self._timeout_ms:
            _lib.check(_lib.lib().ul_comm_set_timeout_ms(self._handle, int(self._timeout_ms)))

    def destroy(self, with_channel: bool = True):
        for h in self._retired + [h for h, _ in self._pending]:
            _lib.lib().ul_comm_destroy(h)
        self._retired, self._pending = [], []
        if self._handle is not None:
            _lib.lib().ul_comm_destroy(self._handle)
            self._handle = None
        if with_channel and self._channel is not None:
            self._channel.destroy()

    def __del__(self):
        # no CUDA call here: a collection can run while the ranks of another
        # in-process group are being issued, and releasing a workspace
        # (cudaFree) synchronizes the device -- which would wait on flag waits
        # that only the not-yet-issued ranks satisfy.  The handles go to the
        # graveyard, released at the next group creation or at exit.
        try:
            _GRAVEYARD.extend(self._retired + [h for h, _ in self._pending])
            if self._handle is not None:
                _GRAVEYARD.append(self._handle)
            self._retired, self._pending, self._handle = [], [], None
        except Exception:
            pass

    # -- status / metering -------------------------------------------------
    def check(self):
        """Raise GroupDesyncError if a device-side wait saw a signature
        mismatch or timed out (simgroup.py:265-298).  Errors are reported
        asynchronously, like NCCL's: poll after a synchronize."""
        if self._channel is not None:
            self._channel.check()
        if self._handle is None:
            return
        buf = ctypes.create_string_buffer(512)
        st = _lib.lib().ul_comm_status(self._handle, buf, 512)
        if st != _lib.UL_OK:
            raise GroupDesyncError(buf.value.decode(errors="replace"))

    def native_ledger(self) -> dict:
        if self._handle is None:
            return {"calls": 0, "egress_bytes": 0, "aggregate_bytes": 0}
        c, e, a = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        _lib.check(_lib.lib().ul_comm_ledger(self._handle, ctypes.byref(c), ctypes.byref(e), ctypes.byref(a)))
        return {"calls": c.value, "egress_bytes": e.value, "aggregate_bytes": a.value}

    def device_ledger(self) -> dict:
        """The byte ledger the GPU kept itself: every call's signalling CTA
        (push kernel or fused epilogue) adds the call and its bytes to this
        rank's device counters (ul_comm_ledger_device).  Read after a sync."""
        if self._handle is None:
            return {"calls": 0, "egress_bytes": 0, "aggregate_bytes": 0}
        c, e, a = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        _lib.check(_lib.lib().ul_comm_ledger_device(self._handle, ctypes.byref(c), ctypes.byref(e), ctypes.byref(a)))
        return {"calls": c.value, "egress_bytes": e.value, "aggregate_bytes": a.value}

    def _record(self, label: str, local_elements: int):
        """One logical all_to_all of `local_elements` per rank (simgroup.py:329-332)."""
        p = self.world
        self.records.append(CommRecord("all_to_all", label, p * local_elements,
                                       local_elements // p * (p - 1)))

    def _record_full(self, label: str, parent_elements: int, group: int):
        """Ledger for a head-group call: the G calls of one logical
        all_to_all are recorded once, with the whole tensor's elements."""
        if group == 0:
            self._record(label, parent_elements)

    def total_egress(self) -> int:
        return sum(r.per_rank_egress_elements for r in self.records)

    def total_aggregate(self) -> int:
        return sum(r.aggregate_elements for r in self.records)

    # -- the collective ----------------------------------------------------
    def ring_shift(self, tensors, steps: int = 1, label: str = "ring_shift", labels=None):
        """RankContext.ring_shift (simgroup.py:374-388, 464-465) for 1..4
        tensors at once: rank i receives rank (i - steps) mod P's tensors
        (fresh outputs).  A collective over peer memory (ul_ring_shift)."""
        tensors = [t.contiguous() for t in tensors]
        if not tensors or len(tensors) > _lib.MAX_FUSED:
            raise ValueError(f"ring_shift moves 1..{_lib.MAX_FUSED} tensors, got {len(tensors)}")
        if steps < 0:
            raise ValueError(f"ring_shift steps must be >= 0, got {steps}")
        outs = [torch.empty_like(t) for t in tensors]
        if self.world > 1:
            self.ensure_slot(slot_need(t.numel() * t.element_size() for t in tensors))
        for t, lab in zip(tensors, labels or [label] * len(tensors)):
            self.records.append(CommRecord("ring_shift", lab, self.world * t.numel(), t.numel() * steps))
        inp = (ctypes.c_void_p * len(tensors))(*[t.data_ptr() for t in tensors])
        outp = (ctypes.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
        nbytes = (ctypes.c_int64 * len(tensors))(*[t.numel() * t.element_size() for t in tensors])
        stream = torch.cuda.current_stream(tensors[0].device).cuda_stream
        _lib.check(_lib.lib().ul_ring_shift(self._handle, len(tensors), inp, outp, nbytes, steps,
                                            label_hash(label), stream))
        return outs

    def qkv_projection(self, x2: torch.Tensor, w: torch.Tensor, b: int, hq: int, hkv: int,
                       labels=("attn.q.seq2head", "attn.k.seq2head", "attn.v.seq2head")):
        """project(x, wq|wk|wv) (layers.py:118-122) fused with the three
        seq->head flips (ulysses.py:140-146): x2 = this rank's [nl*b, d]
        shard, w = [d, (hq + 2 hkv) hd]; returns head-layout q4 [N, b, hq/P,
        hd], k4 / v4 [N, b, hkv/P, hd].  One GEMM whose epilogue stores every
        head block at its owner rank (ul_qkv_proj_exchange); a collective."""
        from .errors import ShardError
        p = self.world
        m, d = x2.shape
        hd = d // hq
        nl = m // b
        if hq % p or hkv % p:
            raise ShardError(f"p={p} does not divide head counts ({hq}, {hkv})")
        q4 = torch.empty((nl * p, b, hq // p, hd), dtype=x2.dtype, device=x2.device)
        k4 = torch.empty((nl * p, b, hkv // p, hd), dtype=x2.dtype, device=x2.device)
        v4 = torch.empty_like(k4)
        if p > 1:
            self.ensure_slot(slot_need(t.numel() * t.element_size() for t in (q4, k4, v4)))
        for lab, hh in zip(labels, (hq, hkv, hkv)):
            self._record(lab, nl * b * hh * hd)
        stream = torch.cuda.current_stream(x2.device).cuda_stream
        _lib.check(_lib.lib().ul_qkv_proj_exchange(self._handle, x2.data_ptr(), w.data_ptr(), q4.data_ptr(),
                                                   k4.data_ptr(), v4.data_ptr(), nl, b, hq, hkv, hd,
                                                   label_hash("attn.qkv.seq2head"), stream),
                   exc_override={-1: ShardError})
        return q4, k4, v4

    def proj_exchange(self, x2: torch.Tensor, w: torch.Tensor, heads, b: int, transposed: bool = False,
                      labels=None, label: str = "proj.seq2head"):
        """GEMM fused with the seq->head exchange of its outputs
        (ul_proj_exchange): Y = x2 @ w (w [d_in, N]) or x2 @ w.T (transposed,
        w [N, d_in]); N = sum(heads)*hd is split into outputs of `heads[t]`
        heads each, returned in this rank's head layout [nl*P, b, heads[t]/P,
        hd].  x2 = this rank's [nl*b, d_in] shard; a collective."""
        from .errors import ShardError
        p = self.world
        m, d_in = x2.shape
        nl = m // b
        n_cols = w.shape[0] if transposed else w.shape[1]
        hd = n_cols // sum(heads)
        for hh in heads:
            if hh % p:
                raise ShardError(f"p={p} does not divide head count {hh}")
        outs = [torch.empty((nl * p, b, hh // p, hd), dtype=x2.dtype, device=x2.device) for hh in heads]
        if p > 1:
            self.ensure_slot(slot_need(o.numel() * o.element_size() for o in outs))
        for lab, hh in zip(labels or [label] * len(heads), heads):
            self._record(lab, nl * b * hh * hd)
        op = (ctypes.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
        hp = (ctypes.c_int64 * len(heads))(*heads)
        stream = torch.cuda.current_stream(x2.device).cuda_stream
        _lib.check(_lib.lib().ul_proj_exchange(self._handle, x2.data_ptr(), w.data_ptr(), int(transposed), len(outs),
                                               op, hp, nl, b, d_in, hd, label_hash(label), stream),
                   exc_override={-1: ShardError})
        return outs

    def all_to_all_head_group(self, tensors, group: int, groups: int, label: str = "attn.seq2head.group",
                              labels=None, ledger_group=None):
        """Seq->head exchange of head group `group` of `groups`
        (ul_all_to_all_head_group): from each rank's full shard
        [nl, b, H_t, hd] rank i receives heads i*H_t/P + group*Hg + [0, Hg)
        of every rank, Hg = H_t / (P*groups), as [nl*P, b, Hg, hd].  The
        `groups` calls of one tensor make one logical all_to_all in the
        ledger (recorded at group 0, or at `ledger_group`)."""
        tensors = [t.contiguous() for t in tensors]
        if not tensors or len(tensors) > _lib.MAX_FUSED:
            raise ValueError(f"all_to_all_head_group fuses 1..{_lib.MAX_FUSED} tensors, got {len(tensors)}")
        p = self.world
        dt = dtype_code(tensors[0].dtype)
        outs = []
        shapes = (ctypes.c_int64 * (4 * len(tensors)))()
        for t, x in enumerate(tensors):
            if x.dim() != 4 or x.dtype != tensors[0].dtype:
                raise ValueError("all_to_all_head_group needs [nl, b, H, hd] tensors of one dtype")
            nl, b, h, hd = x.shape
            if h % (p * groups):
                raise ShardError(f"p={p} x {groups} head groups does not divide head count {h}")
            outs.append(torch.empty((nl * p, b, h // (p * groups), hd), dtype=x.dtype, device=x.device))
            for kk in range(4):
                shapes[4 * t + kk] = x.shape[kk]
        if p > 1:
            self.ensure_slot(slot_need(o.numel() * o.element_size() for o in outs))
        for x, lab in zip(tensors, labels or [label] * len(tensors)):
            self._record_full(lab, x.numel(), group if ledger_group is None else ledger_group)
        inp = (ctypes.c_void_p * len(tensors))(*[x.data_ptr() for x in tensors])
        outp = (ctypes.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
        stream = torch.cuda.current_stream(tensors[0].device).cuda_stream
        _lib.check(_lib.lib().ul_all_to_all_head_group(self._handle, len(tensors), inp, outp, shapes, dt, group,
                                                       groups, label_hash(f"{label}.{group}/{groups}"), stream),
                   exc_override={-1: ShardError})
        return outs

    def all_to_all(self, tensors, split_axis: int, concat_axis: int, label: str = "all_to_all",
                   labels=None):
        """Fused all-to-all of 1..4 contiguous tensors with the same rank,
        dtype and axes (RankContext.all_to_all, simgroup.py:453-456).
        Returns freshly allocated outputs (no aliasing across ranks, like the
        reference's np.concatenate results, simgroup.py:322-327)."""
        tensors = list(tensors)
        if not tensors or len(tensors) > _lib.MAX_FUSED:
            raise ValueError(f"all_to_all fuses 1..{_lib.MAX_FUSED} tensors, got {len(tensors)}")
        ndim = tensors[0].dim()
        if ndim < 1 or ndim > 4:
            raise ValueError(f"all_to_all supports tensors of rank 1..4, got {ndim}")
        split_axis = split_axis % ndim
        concat_axis = concat_axis % ndim
        p = self.world
        dt = dtype_code(tensors[0].dtype)
        outs = []
        shapes = (ctypes.c_int64 * (4 * len(tensors)))()
        for t, x in enumerate(tensors):
            if x.dim() != ndim or x.dtype != tensors[0].dtype:
                raise ValueError("fused all_to_all needs tensors of one rank and dtype")
            if not x.is_cuda:
                raise ValueError("all_to_all operates on CUDA tensors")
            outs.append(torch.empty(a2a_out_shape(x.shape, p, split_axis, concat_axis),
                                    dtype=x.dtype, device=x.device))
            for k in range(ndim):
                shapes[4 * t + k] = x.shape[k]
        labels = labels or [label] * len(tensors)
        if p > 1:
            self.ensure_slot(slot_need(o.numel() * o.element_size() for o in outs))
        for x, lab in zip(tensors, labels):
            self._record(lab, x.numel())
        ins = [x.contiguous() for x in tensors]
        inp = (ctypes.c_void_p * len(ins))(*[x.data_ptr() for x in ins])
        outp = (ctypes.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
        stream = torch.cuda.current_stream(tensors[0].device).cuda_stream
        # P = 1 passes a NULL comm: a local copy (the reference returns a fresh array too)
        _lib.check(_lib.lib().ul_all_to_all(self._handle, len(ins), inp, outp, shapes, ndim, dt,
                                            split_axis, concat_axis, label_hash(label), stream),
                   exc_override={-1: ShardError})
        return outs
