"""Pipeline trace of the backward kernels (profiling tool, not product).

Loads the -DUL_TRACE build (make trace), runs fwd + each bwd kernel on the
config-2 per-head shape, and prints the steady-state hand-off timing of the
MMA thread and two softmax warps (clock64 deltas, SM cycles):

  ev0 MMA: operands of sub-tile j landed, S/dP issue starts
  ev1 MMA: p_full(j) observed, dK/dV (or dQ) issue starts
  ev2/ev4 softmax warp 2 / 9: s_full(j) observed
  ev3/ev5 softmax warp 2 / 9: dS(j) stored, arriving on p_full(j)
  ev6 MMA: dK/dV (dQ) of j issued and committed;  ev7 MMA: S/dP of j issued
  ev8 TMA (dQ kernel): stage of j free, loads of j issued

    python tools/trace_bwd.py [n] [heads]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_14509_b200 import _lib  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, os.environ.get("TRACE_LIB", "ab_libs/trace/libulysses_b200.so")))
_lib._declare(lib)
lib.ul_debug_trace.restype = ctypes.c_int
lib.ul_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
H = int(sys.argv[2]) if len(sys.argv) > 2 else 16
hd = 128
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(1)
mk = lambda: torch.randn((n, 1, H, hd), generator=g, device=dev).to(torch.bfloat16)
q, k, v, do = mk(), mk(), mk(), mk()
o = torch.empty_like(q)
lse = torch.empty((1, H, n), device=dev, dtype=torch.float32)
dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
scale = hd ** -0.5
st = torch.cuda.current_stream().cuda_stream
P = lambda t: ctypes.c_void_p(t.data_ptr())


def chk(rc):
    if rc != 0:
        raise RuntimeError(lib.ul_last_error().decode())


chk(lib.ul_attn_fwd(P(q), P(k), P(v), P(o), P(lse), n, 1, H, H, hd, 1, 1, ctypes.c_float(scale), None, st))
FLAGS = 0   # per-call backward flags (UL_ATTN_DETERMINISTIC = 1)
wsb = lib.ul_attn_bwd_workspace_bytes(n, 1, H, H, hd, 1)
ws = torch.empty(wsb, device=dev, dtype=torch.uint8)


def run(stages):
    chk(lib.ul_attn_bwd_stages(P(q), P(k), P(v), P(o), P(do), P(lse), P(dq), P(dk), P(dv), P(ws), ctypes.c_size_t(wsb),
                               n, 1, H, H, hd, 1, 1, ctypes.c_float(scale), stages, FLAGS, st))
    torch.cuda.synchronize()
    buf = np.zeros(8 * 16 * 256, dtype=np.uint64)
    chk(lib.ul_debug_trace(buf.ctypes.data, buf.nbytes))
    return buf.reshape(8, 16, 256).astype(np.int64)


def report(name, tr):
    print(f"== {name}")
    for cta in range(8):
        ev = tr[cta]
        cnt = int((ev[0] > 0).sum())
        if cnt < 16:
            print(f" cta {cta}: {cnt} sub-tiles (skipped)")
            continue
        lo, hi = 4, cnt - 4
        j = np.arange(lo, hi)
        d = lambda a, b, sa=0, sb=0: np.median(ev[a][j + sa] - ev[b][j + sb])
        print(f" cta {cta}: n={cnt} period(ev0)={d(0, 0, 1, 0):.0f}"
              f" S-issue->s_full seen={d(2, 0):.0f} softmax(w2)={d(3, 2):.0f} softmax(w9)={d(5, 4):.0f}"
              f" w2 idle={d(2, 3, 1, 0):.0f} arrive->MMA sees p_full={d(1, 3):.0f}/{d(1, 5):.0f}"
              f" p_full(j)->S issue(j+1)={d(0, 1, 1, 0):.0f} w9-w2 start skew={d(4, 2):.0f}")
        print(f"        grads issue={d(6, 1):.0f} S/dP issue={d(7, 0):.0f} grads(j)done->S(j+2) start={d(0, 6, 2, 0):.0f}"
              f" S/dP(j) issued->p_full(j-1) seen={d(1, 7, -1, 0):.0f}")
        if (ev[8] > 0).sum() > 16:
            print(f"        TMA: stage free(j)->data seen(j)={d(0, 8):.0f}  dQ/grads(j-K) issued->stage free(j)="
                  f"{d(8, 6, 0, -4):.0f}/{d(8, 6, 0, -3):.0f}")
        print(f"        MMA: loop top->operands seen={d(0, 10):.0f}")
        if (ev[14] > 0).sum() > 16:
            print(f"        w2: tmem ld data={d(12, 2):.0f} L/D data={d(15, 2):.0f} compute={d(14, 15):.0f}"
                  f" st+wait={d(3, 14):.0f}")
        if (ev[11] > 0).sum() > 16:
            print(f"        w2: phase1={d(12, 2):.0f} wait dP={d(11, 12):.0f} phase2={d(3, 11):.0f}")


def report_fused(tr):
    print("== fused (dK/dV/dQ)")
    for cta in range(8):
        ev = tr[cta]
        cnt = int((ev[0] > 0).sum())
        if cnt < 16:
            continue
        j = np.arange(4, cnt - 4)
        d = lambda a, b, sa=0, sb=0: np.median(ev[a][j + sa] - ev[b][j + sb])
        print(f" cta {cta}: n={cnt} period={d(0, 0, 1, 0):.0f}  MMA: top->q_full={d(0, 10):.0f}"
              f" S issue->dq_free ok={d(9, 0):.0f} s_full commit={d(7, 9):.0f} p_full(j-1) seen after s_full(j)="
              f"{d(1, 7, -1, 0):.0f} grads issue={d(6, 1):.0f}")
        print(f"   softmax w6: s_full seen after commit={d(2, 7):.0f} ld={d(12, 2):.0f} compute={d(13, 12):.0f}"
              f" ds_free wait={d(14, 13):.0f} st+arrive={d(3, 14):.0f}  w21 arrive-w6={d(5, 3):.0f}"
              f"  p_full seen-arrive={d(1, 3):.0f}")
        print(f"   drain w2: dq_full seen after grads issue={d(4, 6):.0f} ld+32red+ld={d(11, 4):.0f}"
              f" 32 red={d(15, 11):.0f}  dq_free(j) arrive -> MMA dP(j+2)={d(9, 11, 2, 0):.0f}")
        print(f"   TMA: stage free seen -> q_full at MMA={d(0, 8):.0f}")


def timeline_fused(tr, j0=60, span=3):
    ev = tr[0]
    t0 = ev[10][j0]
    names = {10: "MMA top", 0: "MMA q_full seen", 9: "MMA dq_free(j-2) ok -> dP^T(j) issue", 7: "MMA dP^T(j) issued",
             1: "MMA p_full(j) seen", 6: "MMA grads+dQ^T(j) issued", 2: "w6 s_full seen", 12: "w6 S^T loaded",
             13: "w6 dS computed", 14: "w6 ds_free ok", 3: "w6 p_full arrive", 5: "w21 p_full arrive",
             4: "drain dq_full seen", 11: "drain dq_free arrive", 15: "drain reds issued", 8: "TMA stage free"}
    rows = []
    for j in range(j0 - 2, j0 + span):
        for e, nm in names.items():
            if ev[e][j] > 0:
                rows.append((ev[e][j] - t0, f"{nm} [{j}]"))
    print("== timeline fused (cta 0)")
    for t, nm in sorted(rows):
        if -2500 < t < 5000:
            print(f"  {t:6d}  {nm}")


FLAGS = 0
run(1 | 2)
tr = run(1 | 2)
report_fused(tr)
timeline_fused(tr)
lib.ul_debug_warp.restype = ctypes.c_int
lib.ul_debug_warp.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
wb = np.zeros(32 * 256, dtype=np.uint64)
chk(lib.ul_debug_warp(wb.ctypes.data, wb.nbytes))
w = wb.reshape(32, 256).astype(np.int64)
for j in (59, 60, 61):
    ref = tr[0][10][60]
    print(f"  arrivals [{j}] (rel. MMA top 60): p_full " +
          " ".join(f"w{x}:{w[x][j] - ref}" for x in range(6, 22)) + "  dq_free " +
          " ".join(f"w{x}:{w[x][j] - ref}" for x in range(2, 6)))
FLAGS = 1
for stages, name in ((1 | 2, "dkdv"), (4, "dq")):
    run(stages)  # warm
    report(name, run(stages))


def timeline(name, tr, j0=60, span=3):
    """Raw event times of CTA 0 for sub-tiles j0..j0+span, relative to the
    MMA loop top of j0 (ev10)."""
    ev = tr[0]
    t0 = ev[10][j0]
    names = {10: "MMA top", 0: "MMA kv seen", 1: "MMA p_full seen (dQ/grads j)", 6: "MMA dQ/grads(j) issued",
             7: "MMA S/dP(j) issued", 2: "w2 s_full seen", 3: "w2 p_full arrive", 4: "w9 s_full seen",
             5: "w9 p_full arrive", 8: "TMA stage free", 9: "MMA s_free seen", 13: "MMA S(j) issued"}
    rows = []
    for j in range(j0 - 2, j0 + span):
        for e, nm in names.items():
            if ev[e][j] > 0:
                rows.append((ev[e][j] - t0, f"{nm} [{j}]"))
    print(f"== timeline {name}")
    for t, nm in sorted(rows):
        if -3000 < t < 4000:
            print(f"  {t:6d}  {nm}")


if os.environ.get("TIMELINE"):
    for stages, name in ((1 | 2, "dkdv"), (4, "dq")):
        timeline(name, run(stages))


def cta_report(name):
    """Per-CTA life of the last launch (globaltimer ns): prologue (start ->
    first operands), main loop, epilogue, and the per-SM occupancy/tail."""
    lib.ul_debug_cta.restype = ctypes.c_int
    lib.ul_debug_cta.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    buf = np.zeros(8192 * 7, dtype=np.uint64)
    chk(lib.ul_debug_cta(buf.ctypes.data, buf.nbytes))
    c = buf.reshape(8192, 7).astype(np.int64)
    c = c[c[:, 0] > 0]
    t0 = c[:, 0].min()
    start, first, epi, end, sm, ck0, ck1 = (c[:, i] for i in range(7))
    print(f"   SM clock over CTA lifetimes: median {np.median((ck1 - ck0) / (end - start)):.3f} GHz")
    span = end.max() - t0
    print(f"== CTA life {name}: {len(c)} CTAs, kernel span {span / 1e3:.1f} us")
    print(f"   prologue (start->first operands) median {np.median(first - start) / 1e3:.2f} us,"
          f" epilogue (q_done->end) median {np.median(end - epi) / 1e3:.2f} us,"
          f" main median {np.median(epi - first) / 1e3:.2f} us")
    busy = np.zeros(int(sm.max()) + 1)
    last = np.zeros_like(busy)
    for s_, a, e in zip(sm, start, end):
        busy[s_] += e - a
        last[s_] = max(last[s_], e - t0)
    print(f"   per-SM busy mean {busy.mean() / 1e3:.1f} us (min {busy.min() / 1e3:.1f}, max {busy.max() / 1e3:.1f}),"
          f" SM finish min {last.min() / 1e3:.1f} us / max {last.max() / 1e3:.1f} us")
    gaps = []
    order = np.argsort(start)
    for s_ in range(len(busy)):
        idx = [i for i in order if sm[i] == s_]
        for a, b in zip(idx, idx[1:]):
            gaps.append(start[b] - end[a])
    if gaps:
        print(f"   gap between consecutive CTAs on an SM: median {np.median(gaps) / 1e3:.2f} us")


if os.environ.get("CTA"):
    run(4)
    cta_report("dq")


if os.environ.get("CTA_FUSED"):
    FLAGS = 0
    run(1 | 2)
    cta_report("fused")
