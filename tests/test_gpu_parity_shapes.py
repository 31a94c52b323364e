"""Backward (and forward) parity at BASELINE.json's per-rank shapes against
the float64 oracle, on sampled row blocks.

  config 2  16 heads x 128, N = 8192            (the single-GPU workload)
  config 3   4 heads x 128, N = 32K and 64K      (per rank of P = 8, 32 heads)
  config 4   4 q / 1 kv heads x 128, N = 128K    (per rank of P = 8, GQA 32/8)

Both backward modes (fused atomic-dQ default, deterministic two-kernel).
Checks (kernels.py:89-111 restricted with the reference's row_offset
convention, tensor.py:151-156 / 227-249; oracle/ulysses_oracle.py):
  * O, LSE and dQ on query-row blocks (start, middle, end): independent --
    each row's result depends only on that row;
  * dK / dV on the LAST kv-row block: independent (the only query rows that
    see it are the last ones, whose full-row normalisers the oracle computes
    exactly);
  * dK / dV on a middle kv-row block: chained -- the oracle uses the
    device's LSE and D = rowsum(dO * O) for the n/2 query rows that see the
    block (both verified on the sampled rows above), everything else in
    float64.
bf16 contract: max|a - o| <= 2e-2 * max|o| per block (tests/helpers.py).
Per-shape errors are printed and, with UL_PARITY_REPORT=<path>, appended
as JSON lines.
"""

import json
import math
import os

import numpy as np
import pytest
import torch

from helpers import BF16_MAXREL, rel_max_err
from oracle import ulysses_oracle as O

pytestmark = pytest.mark.gpu

SHAPES = [   # (config, n, hq, hkv)
    ("config2", 8192, 16, 16),
    ("config3_32k", 32768, 4, 4),
    ("config3_64k", 65536, 4, 4),
    ("config4_gqa_128k", 131072, 4, 1),
]
HD = 128
BLK = 64


def U():
    import paper_2309_14509_b200 as mod
    return mod


def _report(rec):
    print(json.dumps(rec))
    path = os.environ.get("UL_PARITY_REPORT")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


@pytest.fixture(scope="module")
def cache():
    return {}


def _run(cache, n, hq, hkv):
    key = (n, hq, hkv)
    if key in cache:
        return cache[key]
    cache.clear()
    g = torch.Generator(device="cuda")
    g.manual_seed(2024 + n + hq)
    mk = lambda h: torch.randn((n, 1, h, HD), generator=g, device="cuda").to(torch.bfloat16)
    q, k, v, do = mk(hq), mk(hkv), mk(hkv), mk(hq)
    fused, det = U().FlashAttention("causal"), U().FlashAttention("causal", deterministic=True)
    o, lse = fused.forward_with_lse(q, k, v)
    grads = {"fused": fused.backward(q, k, v, o, lse, do), "deterministic": det.backward(q, k, v, o, lse, do)}
    torch.cuda.synchronize()
    host = lambda t: t[:, 0].float().cpu().numpy()          # [n, h, hd], exact bf16 values
    res = {"q": host(q), "k": host(k), "v": host(v), "do": host(do), "o": host(o),
           "lse": lse[0].cpu().numpy().astype(np.float64),
           "grads": {m: tuple(host(t) for t in gr) for m, gr in grads.items()}}
    cache[key] = res
    return res


def _heads(hq):
    return sorted({0, hq // 2, hq - 1})


@pytest.mark.parametrize("cfg,n,hq,hkv", SHAPES)
def test_forward_and_dq_rows(cache, cfg, n, hq, hkv):
    r = _run(cache, n, hq, hkv)
    scale = 1.0 / math.sqrt(HD)
    grp = hq // hkv
    errs = {"o": 0.0, "lse_abs": 0.0, "dq_fused": 0.0, "dq_deterministic": 0.0}
    for h in _heads(hq):
        gk = h // grp
        qh, kh, vh, dh = r["q"][:, h], r["k"][:, gk], r["v"][:, gk], r["do"][:, h]
        for r0 in (0, (n // 3) // BLK * BLK, n - BLK):
            rows = (r0, r0 + BLK)
            ctx, lse = O.attention_head(qh[:, None], kh[:, None], vh[:, None], "causal", scale, exact=False,
                                        rows=rows)
            errs["o"] = max(errs["o"], rel_max_err(r["o"][r0:r0 + BLK, h], ctx[:, 0]))
            errs["lse_abs"] = max(errs["lse_abs"], float(np.abs(r["lse"][h, r0:r0 + BLK] - lse[0]).max()))
            dq = O.attention_head_backward_rows(qh, kh, vh, dh, "causal", scale, rows)
            for m in ("fused", "deterministic"):
                errs["dq_" + m] = max(errs["dq_" + m], rel_max_err(r["grads"][m][0][r0:r0 + BLK, h], dq))
    _report({"test": "fwd_dq_rows", "config": cfg, "n": n, "hq": hq, "hkv": hkv, **errs})
    assert errs["o"] <= BF16_MAXREL and errs["lse_abs"] <= 2e-2
    assert errs["dq_fused"] <= BF16_MAXREL and errs["dq_deterministic"] <= BF16_MAXREL


@pytest.mark.parametrize("cfg,n,hq,hkv", SHAPES)
def test_dk_dv_kv_blocks(cache, cfg, n, hq, hkv):
    r = _run(cache, n, hq, hkv)
    scale = 1.0 / math.sqrt(HD)
    grp = hq // hkv
    errs = {}
    kv_heads = sorted({0, hkv - 1})
    for kind, c0 in (("tail", n - 2 * BLK), ("middle_chained", (n // 2) // BLK * BLK)):
        cols = (c0, c0 + BLK if kind != "tail" else n)
        for gk in kv_heads:
            dk = np.zeros((cols[1] - cols[0], HD))
            dv = np.zeros_like(dk)
            for h in range(gk * grp, (gk + 1) * grp):       # GQA: sum over the kv head's query group
                qh, dh = r["q"][:, h], r["do"][:, h]
                if kind == "tail":
                    a, b = O.attention_head_backward_cols(qh, r["k"][:, gk], r["v"][:, gk], dh, "causal", scale,
                                                          cols)
                else:
                    dot = (r["o"][:, h].astype(np.float64) * dh.astype(np.float64)).sum(axis=1)
                    a, b = O.attention_head_backward_cols(qh, r["k"][:, gk], r["v"][:, gk], dh, "causal", scale,
                                                          cols, lse=r["lse"][h], dot=dot)
                dk += a
                dv += b
            for m in ("fused", "deterministic"):
                _, gdk, gdv = r["grads"][m]
                for nm, got, ref in (("dk", gdk, dk), ("dv", gdv, dv)):
                    key = f"{nm}_{kind}_{m}"
                    errs[key] = max(errs.get(key, 0.0), rel_max_err(got[cols[0]:cols[1], gk], ref))
    _report({"test": "dk_dv_blocks", "config": cfg, "n": n, "hq": hq, "hkv": hkv, **errs})
    bad = {k_: e for k_, e in errs.items() if not e <= BF16_MAXREL}
    assert not bad, bad
