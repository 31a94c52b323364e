"""Multi-process Ulysses group through the production setup path.

SequenceGroup.from_process_group (torch.distributed rendezvous, CUDA IPC
mapping of every peer's workspace) + DistributedAttention fwd+bwd, P = 2
processes.  The single B200 of the test box hosts both ranks, so the
cross-process flag protocol runs under GPU time-slicing -- slower, same
semantics.  Results are checked against the f64 oracle.
"""

import json
import os
import socket
import subprocess
import sys
import tempfile

import pytest

from conftest import ROOT
from helpers import BF16_MAXREL

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("mode", ["slot", "grow", "pg", "multidev"])
def test_two_process_group_ipc_fwd_bwd(mode):
    # slot: explicit workspace; grow: a 64 KiB workspace regrown collectively
    # at the first call; pg: the raw torch ProcessGroup as
    # sequence_process_group; multidev: the ranks on two different GPUs (IPC
    # peer mapping, NVLink peer stores, .sys-scope flags across devices)
    import torch
    if mode == "multidev" and torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 visible GPUs")
    with tempfile.TemporaryDirectory() as d:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
               "--master-addr=127.0.0.1", f"--master-port={_port()}",
               os.path.join(ROOT, "tests", "mp_worker.py"), d, mode]
        r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-3000:]
        res = [json.load(open(os.path.join(d, f"rank{i}.json"))) for i in range(2)]
    for x in res:
        assert "error" not in x, x
        for key in ("o", "dq", "dk", "dv"):
            assert x[key] <= BF16_MAXREL, (x["rank"], key, x[key])
        # 4 exchanges per fwd+bwd, 3 iterations (a regrown workspace regrows
        # before the first call is issued, so its ledger sees all of them)
        assert x["calls"] == 3 * 4, x
        if mode == "grow":
            assert x["slot_bytes"] > 64 << 10
        if mode == "multidev":
            assert x["device"] == x["rank"]
