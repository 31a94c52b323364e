"""The pipelined layer (exchanges over head groups overlapped with the
attention, north star item 3) against the unpipelined one and the oracle:
bitwise equal outputs and gradients (deterministic backward), the ledger
law unchanged (one logical all_to_all per tensor per direction), and the
head-group exchange routing bit-exact against the reference all_to_all of
the same heads."""

import numpy as np
import pytest
import torch

from helpers import BF16_MAXREL, rel_max_err, run_ranks, to_dev, to_np
from oracle import ulysses_oracle as O

pytestmark = pytest.mark.gpu


def U():
    import paper_2309_14509_b200 as mod
    return mod


def _layer(p, q, k, v, do, pipeline, deterministic=True):
    n = q.shape[0]
    nl = n // p
    groups = U().SequenceGroup.local_group(p, slot_bytes=1 << 20)
    attn = U().FlashAttention("causal", deterministic=deterministic)
    layers = [U().DistributedAttention(attn, g, pipeline=pipeline, adaptive_pipeline=False) for g in groups]
    sh = lambda x, r: to_dev(x[r * nl:(r + 1) * nl], torch.bfloat16).requires_grad_(True)
    ins = run_ranks(groups, lambda r: [sh(x, r) for x in (q, k, v)])
    dos = run_ranks(groups, lambda r: to_dev(do[r * nl:(r + 1) * nl], torch.bfloat16))
    outs = run_ranks(groups, lambda r: layers[r](*ins[r]))

    def bwd(r):
        torch.autograd.backward([outs[r]], [dos[r]])
        return [t.grad for t in ins[r]]
    gr = run_ranks(groups, bwd)
    cat = lambda xs: torch.cat([x.detach() for x in xs], 0)
    return cat(outs), [cat([gr[r][i] for r in range(p)]) for i in range(3)], groups


@pytest.mark.parametrize("p,hq,hkv,want", [(2, 8, 8, 2), (2, 8, 4, 2), (4, 16, 8, 2), (2, 8, 8, 4)])
def test_pipelined_equals_unpipelined_bitwise(p, hq, hkv, want):
    n, hd = 1024, 128
    q, k, v, do = (O.make_tensor((n, 1, h, hd), 41, s, "bfloat16") for s, h in ((1, hq), (2, hkv), (3, hkv), (4, hq)))
    o1, g1, groups1 = _layer(p, q, k, v, do, pipeline=1)
    o2, g2, groups2 = _layer(p, q, k, v, do, pipeline=want)
    assert U().attention.pipeline_groups(hq // p, hkv // p, want) > 1
    # (the default layer would not split a problem this small)
    assert U().attention.pipeline_groups(hq // p, hkv // p, want, n=n, sms=148) == 1
    assert torch.equal(o1, o2)
    for a, b in zip(g1, g2):
        assert torch.equal(a, b)
    ref, _ = O.local_attention(q, k, v, "causal", exact=False)
    assert rel_max_err(to_np(o2), ref) <= BF16_MAXREL
    # the ledger law (verify.check_ledger): 4 logical all_to_all per direction
    for g in groups2:
        recs = g.records
        assert len(recs) == 8
        assert sum(r.per_rank_egress_elements for r in recs) == sum(r.per_rank_egress_elements for r in groups1[0].records)


@pytest.mark.parametrize("p,groups_,h", [(2, 2, 8), (4, 2, 8), (2, 4, 8), (4, 1, 4)])
def test_head_group_exchange_routing_bitwise(p, groups_, h):
    nl, b, hd = 48, 2, 64
    rng = np.random.default_rng([p, groups_, h])
    xs = [rng.standard_normal((nl, b, h, hd)).astype(np.float32) for _ in range(p)]
    ins = [torch.from_numpy(x).to(torch.bfloat16).cuda() for x in xs]
    groups = U().SequenceGroup.local_group(p, slot_bytes=1 << 20)
    hl, hg = h // p, h // (p * groups_)
    for gi in range(groups_):
        outs = run_ranks(groups, lambda r: groups[r].channel.all_to_all_head_group([ins[r]], gi, groups_)[0])
        # reference: the all_to_all (simgroup.py:322-327) of each rank's heads of this group
        sel = [np.concatenate([x.cpu().view(torch.int16).numpy()[:, :, i * hl + gi * hg:i * hl + (gi + 1) * hg]
                               for i in range(p)], axis=2) for x in ins]
        exp = O.all_to_all(sel, 2, 0)
        for r in range(p):
            assert np.array_equal(outs[r].cpu().view(torch.int16).numpy(), exp[r])
