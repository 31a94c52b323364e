"""Pipeline trace of the full-tile persistent forward (profiling tool, not
product).  Loads the -DUL_TRACE build (tools/ab_build.sh trace "-DUL_TRACE"),
runs the config-2 forward and prints, for CTAs 0-1, the clock64 timeline of
steps J0..J0+span (per-tile kv step counters) and median phase lengths:

  softmax A/B (warp 2 / 2 + kSoft): 4/7 s_full seen, 5/8 exponentials start,
      11/14 split P arrive, 6/9 p_full arrive
  MMA thread: 0/2 split P seen, 12/13 p_full seen, 1/3 PV issued, 10 loop top

    UL_FWD_H2=0 python tools/trace_full.py [n] [heads] [J0] [span]
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
J0 = int(sys.argv[3]) if len(sys.argv) > 3 else 40
span = int(sys.argv[4]) if len(sys.argv) > 4 else 3
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
buf = np.zeros(8 * 16 * 256, dtype=np.uint64)
assert lib.ul_debug_trace_fwd(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes)) == 0
tr = buf.reshape(8, 16, 256).astype(np.int64)
names = {4: "A s_full seen", 5: "A exps start", 11: "A split P arrive", 6: "A p_full arrive",
         7: "B s_full seen", 8: "B exps start", 14: "B split P arrive", 9: "B p_full arrive",
         0: "MMA split P(A) seen", 12: "MMA p_full(A) seen", 1: "MMA PV(A) issued",
         2: "MMA split P(B) seen", 13: "MMA p_full(B) seen", 3: "MMA PV(B) issued"}
for cta in range(2):
    ev = tr[cta]
    t0 = ev[4][J0]
    rows = [(ev[e][j] - t0, f"{nm} [{j}]") for j in range(J0 - 1, J0 + span) for e, nm in names.items() if ev[e][j] > 0]
    print(f"== cta {cta} timeline (clock64, rel. A s_full seen [{J0}])")
    for t, nm in sorted(rows):
        print(f"  {t:7d}  {nm}")
    j = np.arange(8, 100)
    med = lambda a, b, sa=0: int(np.median(ev[a][j + sa] - ev[b][j]))
    for T, (sf, ex, sp, pf, ms, mf, mi) in (("A", (4, 5, 11, 6, 0, 12, 1)), ("B", (7, 8, 14, 9, 2, 13, 3))):
        print(f"  {T}: period={med(sf, sf, 1)} s_full->exps={med(ex, sf)} exps->splitP={med(sp, ex)} "
              f"splitP->p_full={med(pf, sp)} | splitP arrive->MMA sees={med(ms, sp)} p_full arrive->MMA sees={med(mf, pf)}"
              f" MMA p_full seen->PV issued={med(mi, mf)} | p_full arrive->next s_full seen={med(sf, pf, 1)}")
