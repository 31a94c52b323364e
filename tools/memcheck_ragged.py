"""compute-sanitizer memcheck companion (tool, not product): ragged / GQA /
hd-64 forwards against the oracle.
    compute-sanitizer --tool memcheck python tools/memcheck_ragged.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2309_14509_b200 as U  # noqa: E402
from oracle import ulysses_oracle as O  # noqa: E402

for n, hq, hkv, hd, mask in ((1000, 4, 2, 128, "causal"), (333, 2, 1, 64, "causal"), (640, 2, 2, 128, "none")):
    q = O.make_tensor((n, 1, hq, hd), 5, 1, "bfloat16")
    k = O.make_tensor((n, 1, hkv, hd), 5, 2, "bfloat16")
    v = O.make_tensor((n, 1, hkv, hd), 5, 3, "bfloat16")
    dev = lambda x: torch.tensor(x, dtype=torch.float32).to(torch.bfloat16).cuda()
    o, lse = U.FlashAttention(mask).forward_with_lse(dev(q), dev(k), dev(v))
    torch.cuda.synchronize()
    ref, _ = O.local_attention(q, k, v, mask, exact=False)
    print(n, hd, mask, float(np.abs(o.float().cpu().numpy() - ref).max() / np.abs(ref).max()))
