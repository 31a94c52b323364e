"""A/B of kernel variants: per-stage device time (CUDA events, L2 flushed
before each launch) of the local attention at config 2 for every library
passed, plus a numerics check against a torch fp32 reference on 2 heads.

    python tools/ab_kernels.py ab_libs/a ab_libs/b ...   (each runs in its own process)
"""
import json
import math
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(n, H, hd, reps):
    sys.path.insert(0, ROOT)
    import torch
    from paper_2309_14509_b200 import _lib
    lib = _lib.lib()
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(2024)
    mk = lambda: torch.randn((n, 1, H, hd), generator=g, device=dev).to(torch.bfloat16)
    q, k, v, do = mk(), mk(), mk(), mk()
    o = torch.empty_like(q)
    lse = torch.empty((1, H, n), dtype=torch.float32, device=dev)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    wsb = int(lib.ul_attn_bwd_workspace_bytes(n, 1, H, H, hd, 1))
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    scale = 1.0 / math.sqrt(hd)
    flush = torch.empty(1 << 30, dtype=torch.uint8, device=dev)

    def run(stage):
        if stage == 0:
            _lib.check(lib.ul_attn_fwd(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), lse.data_ptr(),
                                       n, 1, H, H, hd, 1, 1, scale, None, st))
        else:
            _lib.check(lib.ul_attn_bwd_stages(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), do.data_ptr(),
                                              lse.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(),
                                              ws.data_ptr(), wsb, n, 1, H, H, hd, 1, 1, scale, stage,
                                              int(os.environ.get("AB_DET", "0")), st))
    names = {0: "fwd", 1: "prep", 2: "dkdv", 4: "dq"}
    t = {s: [] for s in names}
    for it in range(3 + reps):
        for s in names:
            flush.zero_()
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            run(s)
            e.record()
            torch.cuda.synchronize()
            if it >= 3:
                t[s].append(a.elapsed_time(e))
    res = {names[s]: round(statistics.median(v_), 4) for s, v_ in t.items()}
    res["total"] = round(sum(res.values()), 4)
    # numerics: torch fp32 reference on heads 0 and H-1
    errs = {}
    for h in (0, H - 1):
        qf, kf, vf, dof = (x[:, 0, h].float().requires_grad_(True) for x in (q, k, v, do))
        s_ = (qf @ kf.T) * scale
        s_ = s_.masked_fill(torch.ones(n, n, device=dev, dtype=torch.bool).triu(1), float("-inf"))
        of = torch.softmax(s_, -1) @ vf
        of.backward(dof)
        for nm, a_, r_ in (("o", o[:, 0, h], of), ("dq", dq[:, 0, h], qf.grad), ("dk", dk[:, 0, h], kf.grad),
                           ("dv", dv[:, 0, h], vf.grad)):
            e_ = float((a_.float() - r_).abs().max() / r_.abs().max())
            errs[nm] = max(errs.get(nm, 0.0), round(e_, 6))
    res["err"] = errs
    print("RESULT " + json.dumps(res), flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]))
        sys.exit(0)
    n = int(os.environ.get("AB_N", "8192"))
    H = int(os.environ.get("AB_H", "16"))
    reps = int(os.environ.get("AB_REPS", "20"))
    for rnd in range(int(os.environ.get("AB_ROUNDS", "2"))):
        for path in sys.argv[1:]:
            env = dict(os.environ, UL_LIB=os.path.join(os.path.abspath(path), "libulysses_b200.so"))
            out = subprocess.run([sys.executable, __file__, "--child", str(n), str(H), os.environ.get("AB_HD", "128"), str(reps)],
                                 env=env, capture_output=True, text=True)
            line = [l for l in out.stdout.splitlines() if l.startswith("RESULT ")]
            print(rnd, os.path.basename(path.rstrip("/")), line[0][7:] if line else out.stderr[-2000:], flush=True)
