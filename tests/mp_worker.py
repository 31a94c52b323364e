"""Worker for test_gpu_multiprocess.py (launched by torch.distributed.run).

Each process is one Ulysses rank.  All ranks share the box's GPU 0 here
(the test box has one B200), so torch.distributed uses gloo for the setup
rendezvous and the data path is the production one: CUDA-IPC-mapped peer
workspaces, fused push + release flags, bounded acquire waits.
"""

import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2309_14509_b200 as U  # noqa: E402
from oracle import ulysses_oracle as O  # noqa: E402


def main():
    # modes: "slot"   SequenceGroup.from_process_group with a slot big enough
    #        "grow"   ... with a 64 KiB slot: the group regrows collectively
    #        "pg"     the raw torch ProcessGroup passed to DistributedAttention
    #        "multidev" rank r on cuda:r (>= 2 GPUs: IPC + NVLink peer stores)
    out_dir = sys.argv[1]
    mode = sys.argv[2] if len(sys.argv) > 2 else "slot"
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(rank if mode == "multidev" else 0)
    n, b, hq, hkv, hd = 512, 1, 4, 2, 128
    nl = n // world
    q, k, v, do = (O.make_tensor((n, b, h, hd), 77, s, "bfloat16") for s, h in
                   ((1, hq), (2, hkv), (3, hkv), (4, hq)))
    sh = lambda x: torch.tensor(x[rank * nl:(rank + 1) * nl], dtype=torch.float32).to(torch.bfloat16).cuda()
    if mode == "pg":
        layer = U.DistributedAttention(U.FlashAttention("causal"), dist.group.WORLD, adaptive_pipeline=False)
        group = layer.spg
        assert U.DistributedAttention(U.FlashAttention("causal"), dist.group.WORLD).spg is group   # cached wrapper
        group.set_timeout_ms(60000)
    else:
        slot = 64 << 10 if mode == "grow" else 3 * nl * hq * hd * 2 + (1 << 20)
        group = U.SequenceGroup.from_process_group(None, slot_bytes=slot, timeout_ms=60000)
        layer = U.DistributedAttention(U.FlashAttention("causal"), group, adaptive_pipeline=False)
    res = {"rank": rank, "device": torch.cuda.current_device()}
    tq, tk, tv = (sh(x).requires_grad_(True) for x in (q, k, v))
    try:
        for _ in range(3):              # several calls: epochs and slot parity
            for t in (tq, tk, tv):
                t.grad = None
            o = layer(tq, tk, tv)
            o.backward(sh(do))
        torch.cuda.synchronize()
        group.check()
        ref, _ = O.local_attention(q, k, v, "causal", exact=False)
        gref = O.local_attention_backward(q, k, v, do, "causal", exact=False)
        sl = slice(rank * nl, (rank + 1) * nl)
        rel = lambda a, r: float(np.abs(a.detach().float().cpu().numpy() - r[sl]).max() / np.abs(r).max())
        res.update(o=rel(o, ref), dq=rel(tq.grad, gref[0]), dk=rel(tk.grad, gref[1]), dv=rel(tv.grad, gref[2]),
                   calls=group.native_ledger()["calls"], slot_bytes=group.slot_bytes)
    except Exception as e:  # reported to the test
        res["error"] = repr(e)
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump(res, f)
    dist.barrier()
    group.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
