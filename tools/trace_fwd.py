"""Pipeline trace of the forward kernel (profiling tool, not product).

Loads the -DUL_TRACE build (make trace), runs the config-2 forward and prints
the steady-state hand-off timing (clock64, SM cycles) of the first CTAs plus
a raw timeline and the per-CTA life summary:

  ev10/0 MMA: loop top / V(j), K(j+1) landed     ev1/ev2 MMA: p_full A/B(j) seen
  ev6 MMA: PV_A(j), S_A(j+1) issued               ev7 MMA: iteration issued
  ev3/ev4 softmax tile A (warp 2): s_full seen / p_full arrive
  ev5/ev11 softmax tile B (warp 6): s_full seen / p_full arrive
  ev8/ev9 TMA: K / V stage of j free

    python tools/trace_fwd.py [n] [heads]
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
for fn in ("ul_debug_trace_fwd", "ul_debug_cta_fwd"):
    getattr(lib, fn).restype = ctypes.c_int
    getattr(lib, fn).argtypes = [ctypes.c_void_p, ctypes.c_size_t]

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
H = int(sys.argv[2]) if len(sys.argv) > 2 else 16
hd = 128
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(1)
mk = lambda: torch.randn((n, 1, H, hd), generator=g, device=dev).to(torch.bfloat16)
q, k, v = mk(), mk(), mk()
o = torch.empty_like(q)
lse = torch.empty((1, H, n), device=dev, dtype=torch.float32)
st = torch.cuda.current_stream().cuda_stream
sched = torch.zeros(4, dtype=torch.int32, device=dev)   # persistent-forward work counter
P = lambda t: ctypes.c_void_p(t.data_ptr())


def chk(rc):
    if rc != 0:
        raise RuntimeError(lib.ul_last_error().decode())


def run():
    chk(lib.ul_attn_fwd(P(q), P(k), P(v), P(o), P(lse), n, 1, H, H, hd, 1, 1, ctypes.c_float(hd ** -0.5),
                        P(sched) if os.environ.get("PERSIST", "1") == "1" else None, st))
    torch.cuda.synchronize()


run()
run()
buf = np.zeros(8 * 16 * 256, dtype=np.uint64)
chk(lib.ul_debug_trace_fwd(buf.ctypes.data, buf.nbytes))
tr = buf.reshape(8, 16, 256).astype(np.int64)
for cta in range(4):
    ev = tr[cta]
    cnt = int((ev[0] > 0).sum())
    if cnt < 12:
        continue
    j = np.arange(3, cnt - 3)
    d = lambda a, b, sa=0, sb=0: np.median(ev[a][j + sa] - ev[b][j + sb])
    print(f"cta {cta}: kv tiles={cnt} period={d(0, 0, 1, 0):.0f}  softmax A={d(4, 3):.0f} B={d(11, 5):.0f}"
          f"  A arrive->MMA sees={d(1, 4):.0f}  B arrive->MMA sees={d(2, 11):.0f}"
          f"  MMA wait V/K={d(0, 10):.0f}  S_A(j+1) issued->s_full seen A={d(3, 6, 1, 0):.0f}")
    print(f"   A(w2): ld={d(12, 3):.0f} max={d(13, 12):.0f} exp+st={d(14, 13):.0f} wait_st..arrive={d(4, 14):.0f}"
          f"  w4 arrive - w2 arrive={d(15, 4):.0f}")
ev = tr[0]
j0 = 30
t0 = ev[10][j0]
names = {10: "MMA top", 0: "MMA V/K landed", 1: "MMA p_full A seen", 6: "MMA PV_A+S_A issued",
         2: "MMA p_full B seen", 7: "MMA all issued", 3: "A s_full seen", 4: "A arrive", 5: "B s_full seen",
         11: "B arrive", 8: "TMA K stage free", 9: "TMA V stage free", 12: "A ld done", 13: "A max done",
         14: "A exp done", 15: "A w4 arrive"}
rows = []
for jj in range(j0 - 1, j0 + 3):
    for e, nm in names.items():
        if ev[e][jj] > 0:
            rows.append((ev[e][jj] - t0, f"{nm} [{jj}]"))
print("== timeline cta 0")
for t, nm in sorted(rows):
    if -2500 < t < 6000:
        print(f"  {t:6d}  {nm}")

cb = np.zeros(8192 * 7, dtype=np.uint64)
chk(lib.ul_debug_cta_fwd(cb.ctypes.data, cb.nbytes))
c = cb.reshape(8192, 7).astype(np.int64)
c = c[c[:, 0] > 0]
start, first, epi, end, sm, ck0, ck1 = (c[:, i] for i in range(7))
print(f"== CTA life: {len(c)} CTAs, span {(end.max() - start.min()) / 1e3:.1f} us,"
      f" clock {np.median((ck1 - ck0) / (end - start)):.3f} GHz, prologue {np.median(first - start) / 1e3:.2f} us,"
      f" epilogue {np.median(end - epi) / 1e3:.2f} us, main {np.median(epi - first) / 1e3:.2f} us")
if os.environ.get("CTA_PERSIST"):
    # persistent grid: one CTA per SM; the spread of their end times is the
    # static schedule's imbalance
    print(f"== persistent CTAs: end spread {(end.max() - end.min()) / 1e3:.1f} us "
          f"(p10 {np.percentile(end - start.min(), 10) / 1e3:.1f}, median {np.median(end - start.min()) / 1e3:.1f}, "
          f"max {(end.max() - start.min()) / 1e3:.1f} us)")
