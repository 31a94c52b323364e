"""Debug: the first in-process layer call of a process (faulthandler dumps
where the host thread is blocked)."""
import faulthandler
import os
import sys
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
faulthandler.dump_traceback_later(25, exit=False)
import torch  # noqa: E402
from oracle import ulysses_oracle as O  # noqa: E402
import test_gpu_pipeline as T  # noqa: E402
import paper_2309_14509_b200 as U  # noqa: E402
W = os.environ.get("WARM", "")
if W == "fwd":
    x = torch.randn((1024, 1, 4, 128), device="cuda").to(torch.bfloat16)
    U.FlashAttention("causal").forward_with_lse(x, x, x)
    torch.cuda.synchronize()
    print("fwd warm done", flush=True)
if W == "fwdns":   # forward without the dynamic schedule counter (static items)
    x = torch.randn((1024, 1, 4, 128), device="cuda").to(torch.bfloat16)
    o_ = torch.empty_like(x)
    l_ = torch.empty((1, 4, 1024), device="cuda")
    from paper_2309_14509_b200 import _lib
    _lib.check(_lib.lib().ul_attn_fwd(x.data_ptr(), x.data_ptr(), x.data_ptr(), o_.data_ptr(), l_.data_ptr(),
                                      1024, 1, 4, 4, 128, 1, 1, 0.088, None, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    print("fwd (static) warm done", flush=True)
if W == "zeros":
    torch.zeros(2, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
if W == "p1":
    x = torch.randn((1024, 1, 4, 128), device="cuda").to(torch.bfloat16)
    fa = U.FlashAttention("causal")
    o_, l_ = fa.forward_with_lse(x, x, x)
    fa.backward(x, x, x, o_, l_, x)
    torch.cuda.synchronize()
    print("p1 warm done", flush=True)
n, hd, p, hq, hkv = 1024, 128, 2, 8, 8
q, k, v, do = (O.make_tensor((n, 1, h, hd), 41, s, "bfloat16") for s, h in ((1, hq), (2, hkv), (3, hkv), (4, hq)))
o1, g1, groups1 = T._layer(p, q, k, v, do, pipeline=1)
print("layer ok", flush=True)
