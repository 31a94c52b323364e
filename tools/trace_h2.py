"""Pipeline trace of the half-unit forward (profiling tool, not product).

Loads the -DUL_TRACE build (tools/ab_build.sh trace "-DUL_TRACE"), runs the
config-2 forward on the persistent half-unit kernel and prints, for CTA 0,
the clock64 timeline of units U0..U0+span of both query tiles:

  ev0/ev2 MMA: p_full(A/B, unit) seen      ev1/ev3 MMA: PV(A/B, unit) issued
  ev4/ev7 softmax A/B (warp 2/10): s_full seen
  ev5/ev8 softmax A/B: exponentials start  ev6/ev9 softmax A/B: p_full arrive

    python tools/trace_h2.py [n] [heads] [U0] [span]
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2309_14509_b200 import _lib  # noqa: E402

lib = ctypes.CDLL(os.path.join(ROOT, os.environ.get("TRACE_LIB", "ab_libs/trace/libulysses_b200.so")))
_lib._declare(lib)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
H = int(sys.argv[2]) if len(sys.argv) > 2 else 16
U0 = int(sys.argv[3]) if len(sys.argv) > 3 else 40
span = int(sys.argv[4]) if len(sys.argv) > 4 else 4
hd = 128
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(1)
q, k, v = (torch.randn((n, 1, H, hd), generator=g, device=dev).to(torch.bfloat16) for _ in range(3))
o = torch.empty_like(q)
lse = torch.empty((1, H, n), device=dev, dtype=torch.float32)
sched = torch.zeros(4, dtype=torch.int32, device=dev)
st = torch.cuda.current_stream().cuda_stream
P = lambda t: ctypes.c_void_p(t.data_ptr())
for _ in range(3):
    rc = lib.ul_attn_fwd(P(q), P(k), P(v), P(o), P(lse), n, 1, H, H, hd, 1, 1, ctypes.c_float(hd ** -0.5), P(sched), st)
    assert rc == 0, lib.ul_last_error()
torch.cuda.synchronize()
lib.ul_debug_trace_fwd.restype = ctypes.c_int
buf = np.zeros(8 * 16 * 256, dtype=np.uint64)
assert lib.ul_debug_trace_fwd(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes)) == 0
tr = buf.reshape(8, 16, 256).astype(np.int64)
names = {0: "MMA p_full(A) seen", 1: "MMA PV(A)+S issued", 2: "MMA p_full(B) seen", 3: "MMA PV(B)+S issued",
         4: "A s_full seen", 5: "A exps start", 6: "A p_full arrive (w2, SMSP2)",
         7: "B s_full seen", 8: "B exps start", 9: "B p_full arrive",
         10: "MMA loop top", 11: "MMA V landed", 12: "MMA K+V landed"}
# producer events (indexed by kv tile, not unit): 13 K slot free, 14 V slot free
for cta in range(2):
    ev = tr[cta]
    t0 = ev[4][U0]
    rows = []
    for u in range(U0 - 1, U0 + span):
        for e, nm in names.items():
            if ev[e][u] > 0:
                rows.append((ev[e][u] - t0, f"{nm} [{u}]"))
    print(f"== cta {cta} timeline (clock64, rel. A s_full seen [{U0}])")
    for t, nm in sorted(rows):
        print(f"  {t:7d}  {nm}")
    j = np.arange(8, 120)
    med = lambda a, b, sa=0: int(np.median(ev[a][j + sa] - ev[b][j]))
    print(f"  medians: A unit period={med(4, 4, 1)}  A s_full->exps={med(5, 4)} A exps->arrive={med(6, 5)}"
          f"  A arrive->MMA sees={med(0, 6)}  MMA sees->issued={med(1, 0)}  A arrive->next s_full seen={med(4, 6, 1)}")
    print(f"           B: s_full->exps={med(8, 7)} exps->arrive={med(9, 8)} B arrive->MMA sees={med(2, 9)}"
          f"  MMA: loop top->K+V landed={med(12, 10)} K+V landed->p_full(A) seen={med(0, 12)}"
          f"  PV(A) issued->p_full(B) seen={med(2, 1)} PV(B) issued->next loop top={med(10, 3, 1)}")
