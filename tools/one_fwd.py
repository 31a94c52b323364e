"""One config-2 forward (or backward) launch sequence for ncu captures:
python tools/one_fwd.py [fwd|bwd] [n] [heads]"""
import sys
import torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2309_14509_b200 as U

what = sys.argv[1] if len(sys.argv) > 1 else "fwd"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
h = int(sys.argv[3]) if len(sys.argv) > 3 else 16
g = torch.Generator(device="cuda")
g.manual_seed(1)
q, k, v, do = (torch.randn((n, 1, h, 128), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
attn = U.FlashAttention("causal")
for _ in range(3):
    o, lse = attn.forward_with_lse(q, k, v)
    if what == "bwd":
        attn.backward(q, k, v, o, lse, do)
torch.cuda.synchronize()
