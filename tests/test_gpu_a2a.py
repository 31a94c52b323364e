"""K1/K2 all-to-all on the GPU: bit-exact routing vs the reference goldens.

P > 1 runs as an in-process group on one B200 (each rank on its own stream,
peer pointers = plain device pointers): the same push / flag-wait / drain
kernels as the multi-GPU path.  Mirrors test_simgroup.py TestAllToAll and
test_ulysses.py TestLayoutFlips.
"""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from helpers import run_ranks
from oracle import ulysses_oracle as O

pytestmark = pytest.mark.gpu


def U():
    import paper_2309_14509_b200 as mod
    return mod


def golden():
    return np.load(os.path.join(GOLDEN, "a2a.npz"))


@pytest.mark.parametrize("ci", range(8))
def test_golden_cases_bitwise_f32(ci):
    g = golden()
    meta = g[f"case{ci}_meta"]
    p, split, concat = (int(x) for x in meta[:3])
    ins = [torch.from_numpy(g[f"case{ci}_in{r}"]).cuda() for r in range(p)]
    groups = U().SequenceGroup.local_group(p, slot_bytes=1 << 20)
    outs = run_ranks(groups, lambda r: groups[r].all_to_all([ins[r]], split, concat, label="golden")[0])
    for r in range(p):
        exp = g[f"case{ci}_out{r}"]
        got = outs[r].cpu().numpy()
        assert got.shape == exp.shape
        assert got.tobytes() == exp.tobytes(), f"rank {r} routing differs"


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("nl,b,h,hd", [(64, 1, 16, 128), (33, 2, 8, 64), (5, 1, 8, 8)])
def test_seq2head_bf16_bitwise_and_self_inverse(p, nl, b, h, hd):
    rng = np.random.default_rng([p, nl, h])
    xs = [rng.standard_normal((nl, b, h, hd)).astype(np.float32) for _ in range(p)]
    ins = [torch.from_numpy(x).to(torch.bfloat16).cuda() for x in xs]
    exp = O.all_to_all([x.cpu().view(torch.int16).numpy() for x in ins], 2, 0)
    groups = U().SequenceGroup.local_group(p, slot_bytes=4 << 20)
    heads = run_ranks(groups, lambda r: groups[r].all_to_all([ins[r]], 2, 0)[0])
    for r in range(p):
        assert np.array_equal(heads[r].cpu().view(torch.int16).numpy(), exp[r])
    back = run_ranks(groups, lambda r: groups[r].all_to_all([heads[r]], 0, 2)[0])
    for r in range(p):
        assert torch.equal(back[r].view(torch.int16), ins[r].view(torch.int16))


def test_fused_qkv_gqa_and_ledger():
    p, nl, b, hq, hkv, hd = 4, 16, 1, 8, 4, 64
    rng = np.random.default_rng(11)
    mk = lambda h: [torch.from_numpy(rng.standard_normal((nl, b, h, hd)).astype(np.float32)).to(torch.bfloat16).cuda()
                    for _ in range(p)]
    q, k, v = mk(hq), mk(hkv), mk(hkv)
    groups = U().SequenceGroup.local_group(p, slot_bytes=4 << 20)
    outs = run_ranks(groups, lambda r: groups[r].all_to_all([q[r], k[r], v[r]], 2, 0))
    for name, src in (("q", q), ("k", k), ("v", v)):
        exp = O.all_to_all([x.cpu().view(torch.int16).numpy() for x in src], 2, 0)
        idx = "qkv".index(name)
        for r in range(p):
            assert np.array_equal(outs[r][idx].cpu().view(torch.int16).numpy(), exp[r])
    # metering == simgroup.py:329-332 per logical tensor; native egress in bytes
    led = groups[0].native_ledger()
    local_bytes = (nl * b * (hq + 2 * hkv) * hd) * 2
    assert led["calls"] == 1
    assert led["egress_bytes"] == local_bytes // p * (p - 1)
    recs = groups[0].records
    assert [r.aggregate_elements for r in recs] == [p * nl * b * h * hd for h in (hq, hkv, hkv)]


def test_p1_identity_and_zero_egress():
    x = torch.randn(8, 1, 4, 16, device="cuda")
    g = U().SequenceGroup.single()
    y = g.all_to_all([x], 2, 0)[0]
    assert torch.equal(x, y) and y.data_ptr() != x.data_ptr()
    assert g.total_egress() == 0


def test_shard_error():
    groups = U().SequenceGroup.local_group(2, slot_bytes=1 << 20)
    with pytest.raises(U().ShardError):
        groups[0].all_to_all([torch.zeros(3, 2, device="cuda")], 0, 1)


def test_desync_signature_mismatch_is_error_not_hang():
    # test_simgroup.py:196-204: inconsistent shapes name the rank and the collective
    groups = U().SequenceGroup.local_group(2, slot_bytes=1 << 20)
    for g in groups:
        g.set_timeout_ms(5000)
    xs = [torch.zeros(4, 2, device="cuda"), torch.zeros(2, 4, device="cuda")]
    with pytest.raises(U().GroupDesyncError, match="rank 1.*all_to_all"):
        run_ranks(groups, lambda r: groups[r].all_to_all([xs[r]], 0, 1, label="oops"))


def test_desync_timeout_when_a_rank_never_arrives():
    # test_simgroup.py:206-213: an absent rank -> timeout error naming it
    groups = U().SequenceGroup.local_group(2, slot_bytes=1 << 20)
    groups[0].set_timeout_ms(300)
    x = torch.zeros(4, 2, device="cuda")
    torch.cuda.synchronize()
    with torch.cuda.stream(groups[0].stream):
        groups[0].all_to_all([x], 0, 1, label="late")
    torch.cuda.synchronize()
    with pytest.raises(U().GroupDesyncError, match="timeout.*ranks \\[1\\]"):
        groups[0].check()


def test_many_back_to_back_calls_ping_pong_slots():
    # epochs / slot parity across many calls without host syncs in between
    p = 4
    groups = U().SequenceGroup.local_group(p, slot_bytes=1 << 20)
    xs = [torch.randn(16, 1, 8, 32, device="cuda") for _ in range(p)]
    torch.cuda.synchronize()

    def step(r):
        y = xs[r]
        for _ in range(20):
            y = groups[r].all_to_all([y], 2, 0)[0]
            y = groups[r].all_to_all([y], 0, 2)[0]
        return y

    outs = run_ranks(groups, step)
    for r in range(p):
        assert torch.equal(outs[r], xs[r])
