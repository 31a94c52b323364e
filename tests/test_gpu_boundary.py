"""Boundary hardening on the GPU: self-sizing receive slots, the DeepSpeed
signature (*args passthrough to local_attn), per-call deterministic flags,
the caller-owned forward schedule counter, odd-byte ring shifts and the
empty-shard projection exchange."""

import numpy as np
import pytest
import torch

from helpers import run_ranks, rel_max_err, BF16_MAXREL
from oracle import ulysses_oracle as O

pytestmark = pytest.mark.gpu


def U():
    import paper_2309_14509_b200 as mod
    return mod


def test_receive_slot_grows_on_demand_in_process():
    # a 1 MiB workspace and a 3 x 1 MiB call: the group regrows (collectively)
    # instead of failing, and the routing stays bit-exact
    p, nl, h, hd = 4, 512, 8, 128
    rng = np.random.default_rng(3)
    xs = [[torch.from_numpy(rng.standard_normal((nl, 1, h, hd)).astype(np.float32)).to(torch.bfloat16).cuda()
           for _ in range(3)] for _ in range(p)]
    groups = U().SequenceGroup.local_group(p, slot_bytes=1 << 20)
    assert groups[0].slot_bytes < 3 * nl * h * hd * 2
    outs = run_ranks(groups, lambda r: groups[r].all_to_all(xs[r], 2, 0))
    assert all(g.slot_bytes >= 3 * nl * h * hd * 2 for g in groups)
    for t in range(3):
        exp = O.all_to_all([x[t].cpu().view(torch.int16).numpy() for x in xs], 2, 0)
        for r in range(p):
            assert np.array_equal(outs[r][t].cpu().view(torch.int16).numpy(), exp[r])
    # and keeps working (epochs restarted on every rank)
    back = run_ranks(groups, lambda r: groups[r].all_to_all([outs[r][0]], 0, 2))
    for r in range(p):
        assert torch.equal(back[r][0], xs[r][0])


def test_distributed_attention_small_slot_fused_layer_grows():
    # DistributedAttention over a group created with a slot far below what
    # the fused Q/K/V exchange needs: no slot arithmetic by the caller
    from test_gpu_distributed import run_layer
    p, n, h, hd = 2, 2048, 4, 128
    q, k, v, do = (O.make_tensor((n, 1, h, hd), 2024, s, "bfloat16") for s in (1, 2, 3, 4))
    o, (dq, dk, dv), groups = run_layer(p, q, k, v, do, "causal", torch.bfloat16, slot_bytes=256 << 10)
    assert all(g.slot_bytes >= 3 * (n // p) * h * hd * 2 for g in groups)
    ref, _ = O.local_attention(q, k, v, "causal", exact=False)
    assert rel_max_err(o, ref) <= BF16_MAXREL
    for got, exp in zip((dq, dk, dv), O.local_attention_backward(q, k, v, do, "causal", exact=False)):
        assert rel_max_err(got, exp) <= BF16_MAXREL


def test_args_pass_through_to_local_attention():
    # DeepSpeed's DistributedAttention.forward(query, key, value, *args):
    # extra arguments reach local_attn (the generic route)
    seen = {}
    fa = U().FlashAttention("causal")

    def local_attn(q4, k4, v4, tag, scale_by=1.0):
        seen["tag"], seen["scale_by"] = tag, scale_by
        return fa(q4, k4, v4) * scale_by

    layer = U().DistributedAttention(local_attn, U().SequenceGroup.single())
    x = torch.randn((256, 1, 2, 128), device="cuda").to(torch.bfloat16)
    out = layer(x, x, x, "mark", scale_by=2.0)
    assert seen == {"tag": "mark", "scale_by": 2.0}
    ref = fa(x, x, x) * 2.0
    assert torch.equal(out, ref)


def test_deterministic_flag_is_per_call():
    # two plugins with different modes interleaved on one stream: each call
    # carries its own mode (no process-global switch); the deterministic one
    # reproduces itself bitwise
    n, h, hd = 1024, 2, 128
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    q, k, v, do = (torch.randn((n, 1, h, hd), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
    det, fused = U().FlashAttention("causal", deterministic=True), U().FlashAttention("causal")
    o, lse = det.forward_with_lse(q, k, v)
    a = det.backward(q, k, v, o, lse, do)
    fused.backward(q, k, v, o, lse, do)
    b = det.backward(q, k, v, o, lse, do)
    for x, y in zip(a, b):
        assert torch.equal(x, y)


def test_forward_schedule_counter_is_caller_memory():
    # the persistent forward's work counter is passed in (no library
    # allocation): same result with the dynamic counter, with NULL (static
    # schedule), and the counter is left zeroed
    from paper_2309_14509_b200 import _lib
    n, h, hd = 4096, 4, 128
    g = torch.Generator(device="cuda")
    g.manual_seed(6)
    q, k, v = (torch.randn((n, 1, h, hd), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
    L = _lib.lib()
    st = torch.cuda.current_stream().cuda_stream
    outs = []
    sched = torch.zeros(2, dtype=torch.int32, device="cuda")
    for ptr in (sched.data_ptr(), None):
        o = torch.empty_like(q)
        lse = torch.empty((1, h, n), dtype=torch.float32, device="cuda")
        _lib.check(L.ul_attn_fwd(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), lse.data_ptr(),
                                 n, 1, h, h, hd, 1, 1, hd ** -0.5, ptr, st))
        outs.append((o, lse))
    torch.cuda.synchronize()
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    assert int(sched.abs().sum()) == 0


@pytest.mark.parametrize("numel", [1, 7, 4097])
def test_ring_shift_odd_byte_counts(numel):
    # uint8 payloads with odd byte counts move completely (1-byte vector path)
    p = 2
    groups = U().SequenceGroup.local_group(p, slot_bytes=1 << 20)
    xs = [torch.randint(0, 255, (numel,), dtype=torch.uint8, device="cuda") for _ in range(p)]
    outs = run_ranks(groups, lambda r: groups[r].ring_shift([xs[r]], 1))
    for r in range(p):
        assert torch.equal(outs[r][0], xs[(r - 1) % p])


def test_qkv_projection_empty_shard_still_signals():
    # nl == 0 on every rank: no GEMM tile runs, yet the exchange completes
    # (signal-only push) instead of timing out as a false desync
    p, hq, hd = 2, 4, 128
    d = hq * hd
    groups = U().SequenceGroup.local_group(p, slot_bytes=1 << 20)
    for g_ in groups:
        g_.set_timeout_ms(5000)
    x = torch.empty((0, d), dtype=torch.bfloat16, device="cuda")
    w = torch.randn((d, 3 * d), device="cuda").to(torch.bfloat16)
    outs = run_ranks(groups, lambda r: groups[r].qkv_projection(x, w, 1, hq, hq))
    for o in outs:
        assert o[0].shape == (0, 1, hq // p, hd)
