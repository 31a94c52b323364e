"""Child process of test_gpu_ring.py::test_hybrid_ulysses_ring (eager CUDA
module loading): HybridAttention on pu x pr in-process ranks vs the oracle."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from helpers import BF16_MAXREL, rel_max_err, to_dev, to_np, warm_streams  # noqa: E402
from oracle import ulysses_oracle as O  # noqa: E402
import paper_2309_14509_b200 as U  # noqa: E402

def run_config(pu, pr, dname):
    dtype = getattr(torch, dname)
    hd = 128 if dtype == torch.bfloat16 else 16
    h = 8
    d, b, n, seed = h * hd, 1, 64 * pu * pr, 6
    P = pu * pr
    nl = n // P
    w = {k: O.bf16_round(v) for k, v in O.make_weights(d, seed).items()}
    x = O.bf16_round(O.make_input(n, b, d, seed))
    ug = [U.SequenceGroup.local_group(pu, slot_bytes=16 << 20) for _ in range(pr)]   # ug[i][j]
    rg = [U.SequenceGroup.local_group(pr, slot_bytes=16 << 20) for _ in range(pu)]   # rg[j][i]
    ranks = [(i, j) for i in range(pr) for j in range(pu)]
    for i, j in ranks:
        rg[j][i].stream = ug[i][j].stream   # one stream per rank for both of its groups
    if os.environ.get("UL_WORKER_TIMEOUT_MS"):
        for grp in ug + rg:
            for g in grp:
                g.set_timeout_ms(int(os.environ["UL_WORKER_TIMEOUT_MS"]))
    flat = [ug[i][j] for i, j in ranks]


    def run_all(fn):
        """fn(flat rank) on every rank, each on its own stream (run_ranks passes
        the group-local rank, which is not unique across sub-groups)."""
        torch.cuda.synchronize()
        out = []
        for r, g in enumerate(flat):
            with torch.cuda.stream(g.stream):
                out.append(fn(r))
        torch.cuda.synchronize()
        for grp in ug + rg:
            for g in grp:
                g.check()
        return out


    # per-stream library setup (cuBLAS handles/workspaces) and a single-rank pass first
    warm_streams(flat)
    _t = to_dev(x[:nl], dtype).requires_grad_(True)
    _o = U.HybridAttention(d, h, None, None, "causal", weights=w, dtype=dtype)(_t)
    _o.backward(torch.ones_like(_o))
    torch.cuda.synchronize()
    mods = run_all(lambda r: U.HybridAttention(d, h, ug[r // pu][r % pu], rg[r % pu][r // pu], "causal",
                                               weights=w, dtype=dtype))
    go = O.bf16_round(O.make_input(n, b, d, seed + 1))
    xs = run_all(lambda r: to_dev(x[r * nl:(r + 1) * nl], dtype).requires_grad_(True))
    gs = run_all(lambda r: to_dev(go[r * nl:(r + 1) * nl], dtype))
    outs = run_all(lambda r: mods[r](xs[r]))
    run_all(lambda r: torch.autograd.backward([outs[r]], [gs[r]]))
    out = np.concatenate([to_np(o) for o in outs], 0)
    ref = np.concatenate(O.ring_attention_layer([x], w, h, "causal", exact=False))   # P = 1: plain attention layer
    err = rel_max_err(out, ref)
    # gradients: the same function's, oracle = the attention layer's backward at P = 1
    _, st = O.ulysses_attention_layer([x], w, h, "causal", exact=False)
    rgx, rgw = O.ulysses_attention_layer_backward([go], st, w, "causal", exact=False)
    gx = np.concatenate([to_np(t.grad) for t in xs], 0)
    gerr = max([rel_max_err(gx, rgx[0])] + [rel_max_err(sum(to_np(getattr(m, k).grad) for m in mods), rgw[k])
                                            for k in ("wq", "wk", "wv", "wo")])
    tol = 1e-4 if dtype == torch.float32 else BF16_MAXREL
    return {"cfg": [pu, pr, dname], "ok": bool(err <= tol and gerr <= tol), "err": err, "grad_err": gerr,
            "tol": tol}


if __name__ == "__main__":
    cfgs = [a.split(",") for a in sys.argv[1:]]   # "pu,pr,dtype" ...
    res = [run_config(int(c[0]), int(c[1]), c[2]) for c in cfgs]
    print(json.dumps({"ok": all(r["ok"] for r in res), "results": res}))
