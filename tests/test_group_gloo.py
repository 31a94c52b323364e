"""World-size-2 gloo tests of the multi-process host logic (CPU only).

Covers the setup rendezvous of SequenceGroup.from_process_group: handle
blobs gathered in rank order, validated by the native library exactly as
on a GPU box (ul_comm_validate_handles), with geometry mismatches raised as
GroupDesyncError naming the rank (simgroup.py:265-276); and the bench's
max-over-ranks timing reduction.
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2309_14509_b200 import GroupDesyncError
        from paper_2309_14509_b200.comm import gather_handles, pack_handle, validate_handles
        slot = 4096 if (case != "mismatch" or rank == 0) else 8192
        blob = pack_handle(bytes([rank]) * 64, slot, rank, world)
        allb = gather_handles(blob, None)
        res = {"len": len(allb), "first_bytes": [allb[r * 128] for r in range(world)]}
        try:
            validate_handles(allb, world, rank, 4096)
            res["ok"] = True
        except GroupDesyncError as e:
            res["ok"] = False
            res["err"] = str(e)
        # max-over-ranks timing (bench.py)
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res["max"] = float(t.item())
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def _run(case, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    return out


def test_handle_rendezvous_rank_order_and_validation():
    out = _run("ok")
    for r in (0, 1):
        assert out[r]["ok"]
        assert out[r]["len"] == 2 * 128
        assert out[r]["first_bytes"] == [0, 1]      # rank order preserved
        assert out[r]["max"] == 2.0


def test_handle_geometry_mismatch_is_desync():
    out = _run("mismatch")
    for r in (0, 1):
        assert not out[r]["ok"]
        assert "rank 1 workspace slot 8192" in out[r]["err"]
