"""Per-GPU work of BASELINE configs 2-5 measured on ONE B200.

A Ulysses rank at SP degree P runs (a) the fused seq->head / head->seq
exchanges and (b) local attention over the full sequence for H/P heads.
With one GPU available, this tool times (b) at each config's per-rank shape
(exactly the work one of the P GPUs does) and (a) with the same kernels as an
in-process group of P ranks on one device (traffic lands in local HBM, so it
is an HBM-bound lower bound for the NVLink exchange, not an NVLink number).

    python tools/sweep.py [--out profiles/r1_sweep.json] [--quick]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# (name, P, N, Hq, Hkv, hd)
CONFIGS = [
    ("config2 local attn 16x128 N=8K", 1, 8192, 16, 16, 128),
    ("config3 P=8 32x128 N=32K", 8, 32768, 32, 32, 128),
    ("config3 P=8 32x128 N=64K", 8, 65536, 32, 32, 128),
    ("config3 P=8 32x128 N=128K", 8, 131072, 32, 32, 128),
    ("config3 P=8 32x128 N=256K", 8, 262144, 32, 32, 128),
    ("config4 GQA 32q/8kv P=8 N=128K", 8, 131072, 32, 8, 128),
    ("config5 56x128 P=1 N=64K", 1, 65536, 56, 56, 128),
    ("config5 56x128 P=2 N=128K", 2, 131072, 56, 56, 128),
    ("config5 56x128 P=4 N=256K", 4, 262144, 56, 56, 128),
    ("config5 56x128 P=8 N=512K", 8, 524288, 56, 56, 128),
]


def main():
    import torch

    import paper_2309_14509_b200 as U

    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_sweep.json"))
    ap.add_argument("--quick", action="store_true", help="skip the 256K/512K points")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    dev = torch.device("cuda", 0)
    attn = U.FlashAttention("causal")
    res = []
    for name, P, N, Hq, Hkv, hd in CONFIGS:
        if args.quick and N > 131072:
            continue
        hq_l, hkv_l = Hq // P, Hkv // P
        g = torch.Generator(device=dev)
        g.manual_seed(2024)
        mk = lambda h: torch.randn((N, 1, h, hd), generator=g, device=dev).to(torch.bfloat16)
        q, k, v, do = mk(hq_l), mk(hkv_l), mk(hkv_l), mk(hq_l)
        ev = lambda: torch.cuda.Event(enable_timing=True)
        tf, tb = [], []
        for it in range(1 + args.reps):
            a, b, c = ev(), ev(), ev()
            a.record()
            o, lse = attn.forward_with_lse(q, k, v)
            b.record()
            attn.backward(q, k, v, o, lse, do)
            c.record()
            torch.cuda.synchronize()
            if it:
                tf.append(a.elapsed_time(b))
                tb.append(b.elapsed_time(c))
        fwd_ms, bwd_ms = statistics.mean(tf), statistics.mean(tb)
        ff = 4.0 * hq_l * N * N * hd * 0.5
        fb = 2.0 * ff
        step_ms = fwd_ms + bwd_ms
        rec = {"config": name, "P": P, "N": N, "heads_q_per_gpu": hq_l, "heads_kv_per_gpu": hkv_l,
               "attn_fwd_ms": round(fwd_ms, 3), "attn_bwd_ms": round(bwd_ms, 3),
               "attn_tflops_per_gpu": round((ff + fb) / (step_ms / 1e3) / 1e12, 1),
               "frac_of_measured_peak": round((ff + fb) / (step_ms / 1e3) / 1e12 / peaks["bf16_tflops"], 4),
               "tokens_per_s_job_attn_only": round(N / (step_ms / 1e3), 1)}
        # exchange: one fused QKV seq->head call of the P-rank group, in-process on one GPU
        if P > 1:
            nl = N // P
            groups = U.SequenceGroup.local_group(P, slot_bytes=(hq_l * P + 2 * hkv_l * P) * nl * hd * 2 + (1 << 20))
            xs = [[torch.randn((nl, 1, h, hd), device=dev).to(torch.bfloat16) for h in (Hq, Hkv, Hkv)]
                  for _ in range(P)]
            torch.cuda.synchronize()
            times = []
            cover = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
            for it in range(1 + args.reps):
                torch.cuda.synchronize()
                for _ in range(P):   # keep the GPU busy while the host enqueues every rank
                    cover.view(torch.int64).sum()
                evs = []
                for r in range(P):
                    with torch.cuda.stream(groups[r].stream):
                        a, b = ev(), ev()
                        groups[r].stream.wait_stream(torch.cuda.current_stream(dev))
                        a.record()
                        groups[r].all_to_all(xs[r], 2, 0)
                        b.record()
                        evs.append((a, b))
                torch.cuda.synchronize()
                if it:
                    times.append(max(evs[0][0].elapsed_time(b) for _, b in evs))
            for gr in groups:
                gr.check()
            ms = statistics.mean(times)
            local = (Hq + 2 * Hkv) * nl * hd * 2
            egress = local // P * (P - 1)
            rec["a2a_qkv_in_process_ms"] = round(ms, 3)
            rec["a2a_egress_bytes_per_gpu"] = egress
            rec["a2a_volume_exact_per_layer_fwd_elements"] = 4 * N * 1 * Hq * hd * (P - 1) // (P * P)
            # whole layer fwd+bwd: q,k,v,o then dO,dq,dk,dv cross the group once each
            layer_egress = (2 * (Hq + 2 * Hkv) + 2 * Hq) * nl * hd * 2 // P * (P - 1)
            rec["a2a_layer_egress_bytes_per_gpu"] = layer_egress
            # (770 GB/s: the pool's measured B200 peer copy per direction, B200_PROFILING.md --
            #  not measured by this tool, which has one GPU)
            rec["a2a_layer_time_at_guide_peer_copy_770GBs_ms"] = round(layer_egress / 770e9 * 1e3, 3)
            rec["a2a_layer_share_at_guide_peer_copy_770GBs"] = round(
                layer_egress / 770e9 * 1e3 / (step_ms + layer_egress / 770e9 * 1e3), 4)
            for gr in groups:
                gr.destroy()
            del xs
        res.append(rec)
        print(json.dumps(rec), flush=True)
        del q, k, v, do, o, lse
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump({"device": torch.cuda.get_device_name(0), "results": res}, f, indent=1)


if __name__ == "__main__":
    main()
