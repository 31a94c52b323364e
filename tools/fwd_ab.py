"""A/B of the forward kernels (UL_FWD_H2=1 half-unit kernel vs =0 full-tile
persistent kernel; UL_FWD_ALT=1/0 softmax ping-pong on/off; softmax warps per
row, UL_FWD_WPR / UL_FWD_FULL_WPR): device time per launch (CUDA events, L2 flushed by a
read before each), TF/s, and max error of O / LSE against a torch fp32
reference on a few heads.  Each variant runs in its own process (the env
switch is read once).
    python tools/fwd_ab.py [n] [heads] [causal 1|0]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(n, h, causal, reps=20):
    sys.path.insert(0, ROOT)
    import torch
    import paper_2309_14509_b200 as U
    g = torch.Generator(device="cuda")
    g.manual_seed(2024)
    q, k, v = (torch.randn((n, 1, h, 128), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
    attn = U.FlashAttention("causal" if causal else "none")
    flush = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        o, lse = attn.forward_with_lse(q, k, v)
    ts = []
    for _ in range(reps):
        flush.view(torch.int64).sum()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        o, lse = attn.forward_with_lse(q, k, v)
        e.record()
        ts.append((a, e))
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(e) for a, e in ts)[reps // 2]
    flops = 4.0 * n * n * 128 * h * (0.5 if causal else 1.0)
    errs = {}
    for hh in sorted({0, h // 2, h - 1}):
        qf, kf, vf = (x[:, 0, hh].float() for x in (q, k, v))
        s = (qf @ kf.T) / 128 ** 0.5
        if causal:
            s = s.masked_fill(torch.ones(n, n, device="cuda", dtype=torch.bool).triu(1), float("-inf"))
        ref = torch.softmax(s, -1) @ vf
        lref = torch.logsumexp(s, -1)
        errs[hh] = {"o": float((o[:, 0, hh].float() - ref).abs().max() / ref.abs().max()),
                    "lse": float((lse[0, hh] - lref).abs().max())}
    print(json.dumps({"h2": os.environ.get("UL_FWD_H2", "1"), "alt": os.environ.get("UL_FWD_ALT", "0"),
                      "wpr": os.environ.get("UL_FWD_WPR", "2"),
                      "ms": round(ms, 4),
                      "tflops": round(flops / ms / 1e9, 1), "err": errs}))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child(int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]))
        sys.exit(0)
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    h = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    causal = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    variants = os.environ.get("AB_VARIANTS", "1:0:2,1:0:1,0:0:2,1:0:2,1:0:1").split(",")
    for var in variants:
        h2, alt, wpr = var.split(":")
        env = dict(os.environ, UL_FWD_H2=h2, UL_FWD_ALT=alt, UL_FWD_WPR=wpr, UL_FWD_FULL_WPR=wpr)
        r = subprocess.run([sys.executable, __file__, "--child", str(n), str(h), str(causal)], env=env,
                           capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-2000:], flush=True)
