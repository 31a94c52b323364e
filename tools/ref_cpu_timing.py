"""BASELINE.md section 3 / SURVEY 8(d) CPU-baseline plan, timed with the
UNMODIFIED reference (seqlab, imported from /root/reference -- this container
only; the GPU box has no /root/reference, so the bench's reference arm times
the oracle port instead).  Test/measurement tooling, not product.

  * config 1 (P = 2, N = 1024, 8 heads x 64): run_ulysses_attention
    (ulysses.py:249-260, includes the d x d projections) and
    run_ulysses_attention_backward (:281-307), lockstep and concurrent,
    dense and causal, best of 3 (fwd) / best of 2 (fwd+bwd);
  * the boundary harness: q, k, v given -> 3 seq->head all_to_all, the
    per-head kernel, 1 head->seq (ulysses.py:144-154 without projections);
  * the reference all_to_all (RankContext.all_to_all, simgroup.py:313-335)
    at the full per-rank sizes of configs 3, 4 and 5: GB/s per rank.

    PYTHONPATH=/root/reference/pkg/src python tools/ref_cpu_timing.py [out.json]
"""
import json
import os
import platform
import subprocess
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
import numpy as np  # noqa: E402
from seqlab import kernels as K  # noqa: E402
from seqlab import layers as L  # noqa: E402
from seqlab import simgroup as SG  # noqa: E402
from seqlab import tensor as T  # noqa: E402
from seqlab import ulysses as UL  # noqa: E402


def best(fn, reps):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts)


def mask_of(name):
    return T.Mask.causal() if name == "causal" else T.Mask.none()


def config1(out):
    n, b, h, hd, p = 1024, 1, 8, 64, 2
    d = h * hd
    x = L.make_input(n, b, d, 2024)
    w = L.make_weights(d, 2024)
    g = L.make_input(n, b, d, 7)
    for kname in ("dense", "causal"):
        spec = L.AttentionSpec(n=n, b=b, d=d, h_heads=h, mask=mask_of(kname))
        for mode in ("lockstep", "concurrent"):
            out[f"config1_{kname}_{mode}_fwd_s"] = round(
                best(lambda: UL.run_ulysses_attention(x, w, spec, kname, p, mode=mode), 3), 3)
            out[f"config1_{kname}_{mode}_fwd_bwd_s"] = round(
                best(lambda: UL.run_ulysses_attention_backward(x, g, w, spec, kname, p, mode=mode), 2), 3)
        # boundary harness: q, k, v given (no projections), concurrent ranks
        rng = np.random.default_rng(2024)
        qkv = [rng.standard_normal((n, b, d)) for _ in range(3)]
        kern = K.get_kernel(kname)

        def program(ctx):
            nl = n // p
            sh = [a[ctx.rank * nl:(ctx.rank + 1) * nl] for a in qkv]
            q4, k4, v4 = (UL._to_head(a, spec, ctx, f"b.{i}") for i, a in enumerate(sh))
            c4 = np.empty_like(q4)
            for hh in range(q4.shape[2]):
                c4[:, :, hh, :] = kern(q4[:, :, hh, :], k4[:, :, hh, :], v4[:, :, hh, :], spec.mask, spec.scale)
            return UL._to_seq(c4, spec, ctx, "b.ctx")

        for mode in ("lockstep", "concurrent"):
            out[f"boundary_{kname}_{mode}_fwd_s"] = round(best(lambda: SG.RankGroup(p, mode=mode).run(program), 3), 3)
    out["config1_tokens_per_s_fwd_bwd_causal_concurrent"] = round(n / out["config1_causal_concurrent_fwd_bwd_s"], 2)


def a2a_full(out):
    # per-rank seq shards [N/P, 1, H, 128] f64; the seq->head all_to_all of one tensor
    for name, p, n, h in (("config3_N32K", 8, 32768, 32), ("config4_kv_N128K", 8, 131072, 8),
                          ("config5_P2_N128K", 2, 131072, 56)):
        nl = n // p
        shards = [np.random.default_rng(r).standard_normal((nl, 1, h, 128)) for r in range(p)]

        def program(ctx):
            return ctx.all_to_all(shards[ctx.rank], split_axis=2, concat_axis=0, label="a2a")

        t = best(lambda: SG.RankGroup(p, mode="concurrent").run(program), 2)
        local = shards[0].nbytes
        egress = local // p * (p - 1)
        out[f"a2a_{name}"] = {"P": p, "per_rank_shape": [nl, 1, h, 128], "dtype": "f64", "seconds": round(t, 3),
                              "local_bytes_per_rank": local, "egress_gbs_per_rank": round(egress / t / 1e9, 3)}


def main():
    out = {"host": {"cpu_count": os.cpu_count(), "python": platform.python_version(), "numpy": np.__version__}}
    try:
        out["host"]["lscpu_model"] = [ln.split(":", 1)[1].strip() for ln in
                                      subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines()
                                      if ln.startswith("Model name")][0]
    except Exception:
        pass
    config1(out)
    a2a_full(out)
    text = json.dumps(out, indent=1)
    print(text)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            f.write(text + "\n")


if __name__ == "__main__":
    main()
