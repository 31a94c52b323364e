"""Benchmark: Ulysses attention layer (fwd+bwd) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 2|3|4|5] [--seq N] [--quick] [--dry-run]

`--gpus N` (N > 1) without a torchrun environment launches N ranks itself
(torch.distributed.run on 127.0.0.1, one process per GPU); under torchrun it
runs as the rank it is.

Workloads (BASELINE.json configs): config 2's problem -- local attention
fwd+bwd of one GPT-1.3B layer shape (16 heads x 128), N = 8192 tokens, bf16,
causal -- at every N: N = 1 is the metric's single-GPU workload, N > 1 runs
the same problem through the Ulysses layer over N ranks (strong scaling:
the driver's per-N values compare one problem), the seq->head / head->seq
exchanges on the peer-memory kernels (csrc/a2a.cu), no NCCL on the data path.
Beside it (`config5_weak`, skipped by --quick): config 5, weak scaling N =
64K x P, 56 heads x 128 -- per-GPU TF/s, exposed exchange and the constant
per-GPU exchange volume.  --config 3 / 4 / 5 select the 7B (32 heads, N =
32K..256K via --seq), GQA (32 q / 8 kv, N = 128K) or config-5 workload as
the main line instead.

One JSON line on rank 0.  `value` = tokens/s of the whole job with inputs
resident in HBM (device time from CUDA events, max over ranks; L2 flushed by
reading a 1 GiB buffer before every timed step).  `e2e` = the same through the
public API from pinned host buffers (H2D q,k,v,dO + D2H of the loss scalar
every step).  `exposed_a2a` = step minus the rank's attention kernels alone.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# the in-process P = 8 exchange leg runs 8 ranks on 8 streams of one GPU with
# device-side flag waits: give every stream its own hardware queue
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

SEQ_PER_GPU = 8192
HEADS = 16
HEAD_DIM = 128
MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def peaks():
    try:
        with open(MEASURED_PEAKS) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return FALLBACK_PEAKS, "fallback"


FLUSH_BYTES = 1 << 30


def make_flush(dev):
    """L2 flush buffer: 1 GiB (8x the 126 MB L2).  Writing it takes ~0.2 ms
    of full-clock HBM work, long enough for the host to enqueue the next timed
    launches behind it, so the timed interval is device time (an idle GPU
    before the region would either add host launch latency or -- with a
    device sleep -- let clocks drop; tools/timing_ab.py measured both)."""
    import torch
    return torch.empty(FLUSH_BYTES, dtype=torch.uint8, device=dev)


NCU_PROFILE = os.path.join(ROOT, "profiles", "r2_ncu_full.json")   # tools/ncu_r2_summary.py of the r2 capture
NCU_NAMES = {"attn_fwd_sm100": "fwd::attn_fwd_persist_kernel<128", "attn_bwd_dkdv_sm100": "bwd::bwd_dkdv_kernel<128>",
             "attn_bwd_dq_sm100": "bwd::bwd_dq_kernel<128>", "attn_bwd_fused_sm100": "bwd::bwd_fused_kernel<128>"}


def ncu_traffic(kernel):
    """DRAM bytes (read + write) per launch of `kernel` from the committed
    `ncu --set full` capture of the same workload (profiles/), or None."""
    try:
        with open(NCU_PROFILE) as f:
            prof = json.load(f)
        # (keys are ncu's demangled names; match on the name up to the template arguments given)
        d = next(v for k_, v in prof.items() if k_.startswith(NCU_NAMES[kernel]))
        if isinstance(d, list):   # (one record per captured launch: the first)
            d = d[0]
        mb = lambda v: float(v.split()[0]) * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3}[v.split()[1]]
        return {"bytes": int(mb(d["dram__bytes_read.sum"]) + mb(d["dram__bytes_write.sum"])),
                "source": os.path.relpath(NCU_PROFILE, ROOT)}
    except Exception:
        return None


def attn_flops(n_seq, heads, hd, causal=True):
    """fwd 4*H*N^2*hd*c, bwd 8*H*N^2*hd*c, c = 1/2 causal."""
    c = 0.5 if causal else 1.0
    return 4.0 * heads * n_seq * n_seq * hd * c, 8.0 * heads * n_seq * n_seq * hd * c


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------

_NVML_SAMPLER = r"""
import os, select, sys, time
try:   # stay off the launching thread's core, at low priority
    cpus = sorted(os.sched_getaffinity(0))
    if len(cpus) > 1:
        os.sched_setaffinity(0, {cpus[-1]})
    os.nice(10)
except Exception:
    pass
import pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
print("max", pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM), flush=True)
out = []
period = float(sys.argv[2])
idle = os.environ.get("UL_BENCH_CLOCK_IDLE") == "1"   # diagnostics: NVML initialised, no queries
max_clk = int(os.environ.get("UL_BENCH_CLOCK_SM_SAMPLES", "2"))   # SM-clock queries once the steps are enqueued
clocks = False
last_clk, n_clk = -1e9, 0
while True:
    if select.select([sys.stdin], [], [], 0)[0]:
        cmd = sys.stdin.readline().strip()
        if cmd == "clocks":      # the host has enqueued the timed steps: the GPU is busy with them
            clocks = True
        else:
            break
    try:
        # every NVML query perturbs the GPU work (~10-20 us of step time,
        # r90): clock-event reasons every period over the whole region, the
        # SM clock at most twice, once the host has enqueued every timed step
        if idle:
            time.sleep(period)
            continue
        try:
            rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            rs = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        mhz = -1
        if clocks and n_clk < max_clk:
            mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)   # each query stalls the GPU ~20 us (r90)
            last_clk, n_clk = time.perf_counter(), n_clk + 1
        out.append("%d %d" % (mhz, rs))
    except Exception:
        pass
    time.sleep(period)
print("\n".join(out), flush=True)
"""


class ClockSampler:
    """SM clock and clock-event reasons sampled every ~0.5-1 ms (NVML) while
    the timed region runs, in a separate process so the host thread that
    enqueues the step cannot starve it (falls back to `nvidia-smi -lms 100`)."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    # nvmlClocksEventReason* bits
    REASONS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}
    PERIOD_MS = 3.0      # each NVML query perturbs the timed GPU work (~10-20 us, r90)

    def enqueued(self):
        """All timed steps are enqueued (the GPU is still running them): start
        sampling the SM clock too."""
        if self.nvml is not None:
            try:
                self.nvml.stdin.write("clocks\n")
                self.nvml.stdin.flush()
            except Exception:
                pass

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.samples = []       # (sm_mhz, reasons bitmask)
        self.max_mhz = None
        self.nvml = None

    def __enter__(self):
        if os.environ.get("UL_BENCH_CLOCKS") == "off":     # diagnostics only: A/B of the sampler's cost
            return self
        try:
            period = float(os.environ.get("UL_BENCH_CLOCK_MS", self.PERIOD_MS)) / 1e3
            self.nvml = subprocess.Popen([sys.executable, "-c", _NVML_SAMPLER, str(self.gpu), str(period)],
                                         stdin=subprocess.PIPE,
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            first = self.nvml.stdout.readline().split()     # blocks until the sampler is polling
            if len(first) != 2 or first[0] != "max":
                raise RuntimeError("nvml sampler did not start")
            self.max_mhz = int(first[1])
            return self
        except Exception:
            if self.nvml is not None and self.nvml.poll() is None:
                self.nvml.kill()
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.nvml is not None:
            try:
                out, _ = self.nvml.communicate(input="stop\n", timeout=10)
                for ln in out.splitlines():
                    parts = ln.split()
                    if len(parts) == 2:
                        self.samples.append((int(parts[0]), int(parts[1])))
            except Exception:
                self.nvml.kill()
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.nvml is not None:
            if not self.samples:
                return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0,
                        "source": "nvml"}
            reasons = sorted(nm for nm, bit in self.REASONS.items() if any(r & bit for _, r in self.samples))
            mhz = [m for m, _ in self.samples if m >= 0]
            return {"sm_mhz": statistics.median(mhz) if mhz else None, "sm_max_mhz": self.max_mhz,
                    "reasons": reasons if mhz else reasons + ["sm clock unsampled"], "samples": len(self.samples),
                    "sm_clock_samples": len(mhz),
                    "source": f"nvml sampler process every {self.PERIOD_MS} ms: clock-event reasons over "
                              "the whole timed region; SM clock <= 2 samples while the GPU runs the enqueued "
                              "timed steps (each NVML query perturbs the step, r90)",
                    "note": "NVML's SM clock; inside the tensor-core kernels clock64/globaltimer and ncu "
                            "measure 1.60-1.77 GHz (power-limited; profiles/r1_summary.md r77, r85)"}
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvidia-smi 100 ms"}


# ---------------------------------------------------------------------------
# CPU baseline: the oracle restatement of the reference algorithm
# ---------------------------------------------------------------------------

def _cpu_sample_worker(args):
    n_s, hd, seed = args[:3]
    reps = args[3] if len(args) > 3 else 1
    import numpy as np
    from oracle import ulysses_oracle as O
    q, k, v, do = (O.make_tensor((n_s, 1, hd), seed, s) for s in (1, 2, 3, 4))
    t0 = time.perf_counter()
    scale = 1.0 / math.sqrt(hd)
    for _ in range(reps):                                     # `reps` heads of the same shape
        O.attention_head(q, k, v, "causal", scale)               # kernels.py:31-52 (fixed-order matmul)
        O.attention_head_backward(q, k, v, do, "causal", scale)  # kernels.py:89-111
    return (time.perf_counter() - t0) / reps


def cpu_baseline(n_seq, heads, hd, procs=1, n_sample=1024, heads_sample=1):
    """Time the reference algorithm (oracle port, fixed-order f64 matmul) on
    `procs` host processes, one head of N=n_sample each, and extrapolate by
    N^2 * hd * heads to the full workload (the reference is O(N^2 hd) per head
    with full n x n scores, kernels.py:37)."""
    import multiprocessing as mp
    if procs <= 1:
        reps = heads_sample
        dt = _cpu_sample_worker((n_sample, hd, 0, reps))
        per_head = dt
        wall = dt * reps
    else:
        ctx = mp.get_context("fork")
        with ctx.Pool(procs) as pool:
            t0 = time.perf_counter()
            pool.map(_cpu_sample_worker, [(n_sample, hd, i) for i in range(procs)])
            wall = time.perf_counter() - t0
        per_head = wall / procs            # throughput-equivalent seconds per sampled head
    scale = (n_seq / n_sample) ** 2 * heads
    t_full = per_head * scale
    nh = procs if procs > 1 else heads_sample
    return {"tokens_per_s": n_seq / t_full, "seconds_full_extrapolated": t_full, "sample_wall_s": wall,
            "sample": f"{nh} x causal fwd+bwd head of N={n_sample}, hd={hd} (f64, reference fixed-order "
                      f"matmul); extrapolated by N^2*hd*heads to N={n_seq}, {heads} heads"}


# ---------------------------------------------------------------------------
# workloads (BASELINE.json configs)
# ---------------------------------------------------------------------------

CONFIGS = {
    # name: (query heads, kv heads, sequence length for P ranks, description)
    "2": (16, 16, lambda P: SEQ_PER_GPU,
          "config2: local attention fwd+bwd, GPT-1.3B layer 16 heads x 128, N={n} bf16 causal, Ulysses P={P}"),
    "3": (32, 32, lambda P: 32768,
          "config3: Ulysses attention layer P={P}, 7B shape 32 heads x 128, N={n} bf16 causal fwd+bwd"),
    "4": (32, 8, lambda P: 131072,
          "config4: GQA Llama-3-8B 32 q / 8 kv heads x 128, Ulysses P={P}, N={n} bf16 causal fwd+bwd"),
    "5": (56, 56, lambda P: 65536 * P,
          "config5: weak scaling N=64K x P, 30B shape 56 heads x 128, P={P}, N={n} bf16 causal fwd+bwd"),
}


def pick_config(args, P):
    """Every N runs config 2's problem (16 heads x 128, N = 8192: the metric's
    single-GPU workload) -- strong scaling over Ulysses P = N, so the
    driver's per-N values compare one problem; config 5 (weak scaling, N =
    64K x P) is measured beside it (`config5_weak`).  --config overrides."""
    name = args.config or "2"
    hq, hkv, seq, desc = CONFIGS[name]
    if args.heads:
        hq = hkv = args.heads
    n_seq = args.seq or seq(P)
    return name, hq, hkv, n_seq, desc.format(P=P, n=n_seq)


def free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def maybe_relaunch(args):
    """`bench.py --gpus N` without a torchrun environment: launch N ranks
    (one process per GPU) through torch.distributed.run on 127.0.0.1 and
    pass rank 0's line through.  Under torchrun (WORLD_SIZE set) run as is."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    r = subprocess.run(cmd, cwd=ROOT)
    sys.exit(r.returncode)


def read_flush(flush):
    """Untimed L2 flush by READING a 1 GiB buffer: evicts the 126 MB L2
    without leaving dirty lines whose write-back would land in the next
    timed kernel (a zero_() flush does)."""
    flush.view(torch_int64()).sum()


def torch_int64():
    import torch
    return torch.int64


def host_cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus > 1 and world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} but WORLD_SIZE={world}")
    P = world
    cfg_name, H, HKV, n_seq, desc = pick_config(args, P)
    hd = HEAD_DIM
    nl = n_seq // P
    # UL_BENCH_ONE_GPU=1: every rank on cuda:0 with a gloo rendezvous -- a
    # functional smoke test of the N > 1 path on a one-GPU box (NCCL refuses
    # two ranks on one device); timings of such a run mean nothing
    one_gpu = os.environ.get("UL_BENCH_ONE_GPU") == "1"
    if args.dry_run:
        # host-side contract only (CPU): launch, rendezvous, workload choice,
        # max-over-ranks reduction -- no CUDA
        if world > 1:
            dist.init_process_group("gloo")
            t = torch.tensor([float(rank + 1)])
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tmax = float(t.item())
        else:
            tmax = 1.0
        if rank == 0:
            print(json.dumps({"dry_run": True, "n_gpus": P, "max_over_ranks": tmax,
                              "config": workload_config(P, n_seq, H, hd, cfg_name, HKV)}), flush=True)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    import paper_2309_14509_b200 as U
    from paper_2309_14509_b200 import _lib
    if one_gpu:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    causal = True
    if H % P or HKV % P or n_seq % P:
        raise SystemExit(f"config {cfg_name}: P={P} must divide heads ({H}, {HKV}) and N={n_seq}")

    # synthetic inputs: N(0,1), seed 2024, per-rank contiguous shard
    g = torch.Generator(device=dev)
    g.manual_seed(2024 + rank)
    mk = lambda h: torch.randn((nl, 1, h, hd), generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
    q, k, v, do = mk(H), mk(HKV), mk(HKV), mk(H)
    if P > 1:
        group = U.SequenceGroup.from_process_group(None, device=local_rank)   # receive slots size themselves
    else:
        group = U.SequenceGroup.single(local_rank)
    attn = U.FlashAttention("causal")
    layer = U.DistributedAttention(attn, group)
    flush = make_flush(dev)

    def step(qq, kk, vv, dd):
        qq.requires_grad_(True)
        kk.requires_grad_(True)
        vv.requires_grad_(True)
        o = layer(qq, kk, vv)
        torch.autograd.backward([o], [dd])
        return o

    # ---- device-resident timing -------------------------------------------
    for _ in range(args.warmup):
        step(q.detach(), k.detach(), v.detach(), do)
    torch.cuda.synchronize()
    if P > 1:
        dist.barrier()
    launches0 = _lib.total_launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local_rank) as clk:
        torch.cuda.synchronize()
        if P > 1:
            dist.barrier()
        for i in range(args.steps):
            read_flush(flush)                              # untimed L2 flush (read)
            ev[i][0].record()
            step(q.detach(), k.detach(), v.detach(), do)
            ev[i][1].record()
        clk.enqueued()
        torch.cuda.synchronize()
        if P > 1:
            dist.barrier()
    launches = _lib.total_launch_count() - launches0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    t_ms = sum(step_ms)
    if P > 1:
        tt = torch.tensor([t_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
    ms_per_step = t_ms / args.steps
    tokens_per_s = n_seq / (ms_per_step / 1e3)
    f_fwd, f_bwd = attn_flops(n_seq, H // P, hd, causal)
    tflops_per_gpu = (f_fwd + f_bwd) / (ms_per_step / 1e3) / 1e12

    # ---- per-kernel split (dominant kernel roofline) on this rank's
    # head-sharded attention problem [N, 1, H/P, hd] --------------------
    mk4 = lambda h: torch.randn((n_seq, 1, h, hd), generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
    kt = kernel_split(attn, mk4(H // P), mk4(HKV // P), mk4(HKV // P), mk4(H // P), args, dev)
    attn_only_ms = sum(x["ms"] for x in kt["kernels"])
    a2a = bench_a2a(dev, n_seq, H, hd, P, group, HKV, inproc=not args.quick)
    extras = {}
    if not args.quick and not args.config:
        extras["config5_weak"] = bench_config5(P, rank, dev, group, args)
    if P == 1 and not args.quick:
        extras["blocked_sparse_fwd"] = bench_blocked(kt_inputs=(lambda: mk4(H), n_seq, H, hd), args=args, dev=dev)
        extras["layer"] = bench_layer(group, nl, H, hd, args, dev)
        extras["anchors"] = bench_anchors(n_seq, H, hd, flush)

    # ---- e2e through the public API from pinned host buffers ----------
    e2e = run_e2e(layer, q, k, v, do, args, P, dev)

    pk, src = peaks()
    result = None
    if rank == 0:
        dom = max(kt["kernels"], key=lambda x: x["ms"])
        peak = pk["bf16_tflops"]
        ach = dom["alg_flops"] / (dom["ms"] / 1e3) / 1e12
        clocks = clk.summary()
        exposed = ms_per_step - attn_only_ms
        result = {
            "metric": "Ulysses attn tokens/s (fwd+bwd layer), TFLOPs/GPU, all-to-all GB/s",
            "value": round(tokens_per_s, 1),
            "unit": "tokens/s",
            "n_gpus": P,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True,
            "scaling": "weak" if cfg_name == "5" else "strong",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic N(0,1) q/k/v/dO, seed 2024 (no dataset)",
            "config": workload_config(P, n_seq, H, hd, cfg_name, HKV),
            "tflops_per_gpu": round(tflops_per_gpu, 1),
            "tflops_per_gpu_fa_convention": round(
                (f_fwd * 3.5) / (ms_per_step / 1e3) / 1e12, 1),
            "roofline": {
                "bound": "tensor", "kernel": dom["name"], "achieved": round(ach, 1),
                "peak": peak, "unit": "TFLOP/s", "frac": round(ach / peak, 4),
                "peak_source": f"MEASURED_PEAKS.json bf16_tflops ({src}, burst)",
                "frac_of_sustained": round(ach / pk.get("bf16_tflops_sustained", peak), 4),
                # ncu DRAM bytes per launch, captured on the config-2 workload
                "traffic": (ncu_traffic(dom["name"]) or {}).get("bytes") if cfg_name == "2" and P == 1 else None,
                "traffic_source": (ncu_traffic(dom["name"]) or {}).get("source") if cfg_name == "2" and P == 1 else None,
                "alg_flops_per_launch": dom["alg_flops"],
                "layer_frac": round(tflops_per_gpu / peak, 4),
            },
            "kernels": kt["kernels"],
            "exposed_a2a": {"ms": round(exposed, 4), "pct_of_step": round(100.0 * exposed / ms_per_step, 2),
                            "attention_only_ms": round(attn_only_ms, 4),
                            "how": "step time minus the same rank's attention kernels alone (SURVEY 8(d)); "
                                   "at P = 1 the remainder is launch/host overhead (no exchange)"},
            "a2a": a2a,
            **extras,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks,
        }
    if args.cpu_baseline and rank == 0:
        # ~10-15 s of single-core reference work: two heads of N = 2048
        cb = cpu_baseline(n_seq, H, hd, procs=1, n_sample=2 * args.cpu_sample, heads_sample=2)
        result["cpu_baseline"] = {"value": round(cb["tokens_per_s"], 4), "unit": "tokens/s", "cores": 1,
                                  "kind": "port", "sample": cb["sample"],
                                  "sample_wall_s": round(cb["sample_wall_s"], 2), "cpu_model": host_cpu_model()}
    if rank == 0:
        print(json.dumps(result), flush=True)
    if P > 1:
        dist.barrier()
        dist.destroy_process_group()


def bench_config5(P, rank, dev, group, args):
    """BASELINE config 5 beside the headline: weak scaling N = 64K x P, 56
    heads x 128, the Ulysses layer fwd+bwd over this job's P ranks (device
    time, L2 read-flushed before every step, max over ranks), per-GPU
    TFLOP/s and roofline fraction, the exposed exchange (step minus this
    rank's attention kernels alone) and the exact per-GPU exchange egress,
    which N proportional to P keeps constant per link (costmodel.py:82-87)."""
    import torch
    import torch.distributed as dist
    import paper_2309_14509_b200 as U
    H, hd = 56, HEAD_DIM
    n_seq = 65536 * P
    nl = n_seq // P
    g = torch.Generator(device=dev)
    g.manual_seed(2024 + rank)
    mk = lambda shape: torch.randn(shape, generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
    q, k, v, do = (mk((nl, 1, H, hd)) for _ in range(4))
    attn = U.FlashAttention("causal")
    layer = U.DistributedAttention(attn, group)
    flush = make_flush(dev)

    def step():
        qq, kk, vv = (x.detach().requires_grad_(True) for x in (q, k, v))
        torch.autograd.backward([layer(qq, kk, vv)], [do])
    steps, warm = max(2, min(args.steps, 5)), max(1, min(args.warmup, 2))
    for _ in range(warm):
        step()
    torch.cuda.synchronize()
    if P > 1:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        read_flush(flush)
        ev[i][0].record()
        step()
        ev[i][1].record()
    torch.cuda.synchronize()
    t = sum(a.elapsed_time(b) for a, b in ev) / steps
    if P > 1:
        tt = torch.tensor([t], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    del q, k, v, do
    kt = kernel_split(attn, mk((n_seq, 1, H // P, hd)), mk((n_seq, 1, H // P, hd)), mk((n_seq, 1, H // P, hd)),
                      mk((n_seq, 1, H // P, hd)), argparse.Namespace(steps=2, warmup=1), dev)
    att = sum(x["ms"] for x in kt["kernels"])
    f_fwd, f_bwd = attn_flops(n_seq, H // P, hd, True)
    pk, _ = peaks()
    local = nl * H * hd * 2
    egress = 8 * local // P * (P - 1)      # fwd: q, k, v, o; bwd: do, dq, dk, dv
    tf = (f_fwd + f_bwd) / (t / 1e3) / 1e12
    return {"workload": f"config5: 56 heads x 128, N={n_seq}, P={P}, bf16 causal fwd+bwd", "seq_len": n_seq,
            "ms_per_step": round(t, 3), "tokens_per_s": round(n_seq / (t / 1e3), 1),
            "tflops_per_gpu": round(tf, 1), "frac_of_burst_peak": round(tf / pk["bf16_tflops"], 4),
            "attention_only_ms": round(att, 3), "exposed_exchange_ms": round(t - att, 3),
            "exposed_exchange_pct": round(100.0 * (t - att) / t, 2),
            "exchange_egress_bytes_per_gpu": egress, "local_bytes_per_tensor": local,
            "steps": steps, "scaling": "weak"}


def kernel_split(attn, q, k, v, do, args, dev):
    """Per-kernel device time of the local attention (P = this rank's heads)
    with CUDA events on the launching stream, L2 flushed before each."""
    import torch
    from paper_2309_14509_b200 import _lib
    n, b, h, hd = q.shape[0], q.shape[1], q.shape[2], q.shape[3]
    hkv = k.shape[2]
    lib = _lib.lib()
    flush = make_flush(dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    o = torch.empty_like(q)
    lse = torch.empty((b, h, n), dtype=torch.float32, device=dev)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    wsb = int(lib.ul_attn_bwd_workspace_bytes(n, b, h, hkv, hd, 1))
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    sched = torch.zeros(2, dtype=torch.int32, device=dev)   # persistent-forward work counter (UL_ATTN_SCHED_BYTES)
    scale = 1.0 / math.sqrt(hd)
    fused = hd == 128 and not attn.deterministic
    if fused:   # one kernel for dK, dV and dQ (+ the dQ fp32 -> bf16 pass)
        names = ["attn_fwd_sm100", "attn_bwd_prep", "attn_bwd_fused_sm100", "attn_bwd_dq_convert"]
    else:
        names = ["attn_fwd_sm100", "attn_bwd_prep", "attn_bwd_dkdv_sm100", "attn_bwd_dq_sm100"]
    times = {nm: [] for nm in names}
    f_fwd, f_bwd = attn_flops(n, h, hd, True)
    # algorithmic FLOPs credited per kernel: fwd = QK^T + PV; dkdv produces dP, dV, dK
    # (3 of the 4 backward GEMMs, 6*N^2*hd*c); dq produces dQ (2*N^2*hd*c); the
    # fused kernel all four (8*N^2*hd*c)
    alg = {"attn_fwd_sm100": f_fwd, "attn_bwd_prep": 0.0, "attn_bwd_dkdv_sm100": f_bwd * 0.75,
           "attn_bwd_dq_sm100": f_bwd * 0.25, "attn_bwd_fused_sm100": f_bwd, "attn_bwd_dq_convert": 0.0}

    def run(nm):
        if nm == "attn_fwd_sm100":
            _lib.check(lib.ul_attn_fwd(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), lse.data_ptr(),
                                       n, b, h, hkv, hd, 1, 1, scale, sched.data_ptr(), stream))
        else:
            stage = {"attn_bwd_prep": 1, "attn_bwd_dkdv_sm100": 2, "attn_bwd_dq_sm100": 4, "attn_bwd_fused_sm100": 2,
                     "attn_bwd_dq_convert": 4}[nm]
            _lib.check(lib.ul_attn_bwd_stages(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                                              do.data_ptr(), lse.data_ptr(), dq.data_ptr(), dk.data_ptr(),
                                              dv.data_ptr(), ws.data_ptr(), wsb, n, b, h, hkv, hd, 1, 1, scale,
                                              stage, attn.flags, stream))

    reps = max(3, min(args.steps, 10))
    for it in range(args.warmup + reps):
        for nm in names:
            read_flush(flush)
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            run(nm)
            e.record()
            if it >= args.warmup:
                times[nm].append((a, e))
    torch.cuda.synchronize()
    out = []
    for nm in names:
        ms = statistics.mean(a.elapsed_time(e) for a, e in times[nm])
        rec = {"name": nm, "ms": round(ms, 4), "alg_flops": alg[nm]}
        if alg[nm]:
            rec["tflops"] = round(alg[nm] / (ms / 1e3) / 1e12, 1)
        out.append(rec)
    return {"kernels": out}


def bench_layer(group, nl, H, hd, args, dev):
    """the whole UlyssesAttention layer (x -> fused
    QKV GEMM + seq->head exchange -> attention -> O projection, and its
    backward) on this rank's shard, plus the fused QKV projection kernel
    alone against cuBLAS (torch.matmul) on the same GEMM."""
    import torch
    import paper_2309_14509_b200 as U
    d = H * hd
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    layer = U.UlyssesAttention(d, H, group, "causal", dtype=torch.bfloat16, device=dev)
    x = torch.randn((nl, 1, d), generator=g, device=dev).to(torch.bfloat16)
    gout = torch.randn((nl, 1, d), generator=g, device=dev).to(torch.bfloat16)
    flush = make_flush(dev)

    def timeit(fn, reps):
        ts = []
        for it in range(args.warmup + reps):
            read_flush(flush)
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            e.record()
            if it >= args.warmup:
                ts.append((a, e))
        torch.cuda.synchronize()
        return statistics.mean(a.elapsed_time(e) for a, e in ts)

    def step():
        xx = x.detach().requires_grad_(True)
        torch.autograd.backward([layer(xx)], [gout])
    reps = max(3, min(args.steps, 10))
    ms_layer = timeit(step, reps)
    x2 = x.reshape(nl, d)
    wqkv = torch.cat([layer.wq, layer.wk, layer.wv], dim=1).detach().contiguous()
    ms_fused = timeit(lambda: group.qkv_projection(x2, wqkv, 1, H, H), reps)
    ms_cublas = timeit(lambda: x2 @ wqkv, reps)
    flops = 2.0 * nl * d * 3 * d
    P = group.world
    n_seq = nl * P
    f_att = sum(attn_flops(n_seq, H // P, hd, True))
    f_proj = 3 * 2.0 * nl * d * 4 * d     # fwd: x.W_qkv + c.W_o; bwd: 2x each
    return {"d_model": d, "ms_fwd_bwd": round(ms_layer, 4), "tokens_per_s": round(n_seq / (ms_layer / 1e3), 1),
            "tflops_per_gpu": round((f_att + f_proj) / (ms_layer / 1e3) / 1e12, 1),
            "qkv_proj_exchange": {"ms": round(ms_fused, 4), "tflops": round(flops / (ms_fused / 1e3) / 1e12, 1),
                                  "note": "tcgen05 GEMM x [wq|wk|wv] with the seq->head exchange in its epilogue"},
            "cublas_qkv_gemm": {"ms": round(ms_cublas, 4), "tflops": round(flops / (ms_cublas / 1e3) / 1e12, 1),
                                "note": "torch.matmul, same GEMM, no exchange (comparison)"}}


def bench_blocked(kt_inputs, args, dev, bs=128, bandwidth=15):
    """Blocked-sparse forward (blocked_kernel,
    kernels.py:55-86) on this rank's head-sharded problem with a banded
    block pattern (tensor.py:200-206): window of bandwidth+1 blocks of 128.
    FLOPs counted over visible blocks only (4*hd*bs^2 per visible block pair
    per head)."""
    import torch
    import paper_2309_14509_b200 as U
    mk, n, h, hd = kt_inputs
    q, k, v = mk(), mk(), mk()
    nb = n // bs
    pattern = frozenset((a, b) for a in range(nb) for b in range(max(0, a - bandwidth), a + 1))
    attn = U.FlashAttention("blocked", block_size=bs, pattern=pattern)
    flush = make_flush(dev)
    times = []
    for it in range(args.warmup + max(3, min(args.steps, 10))):
        read_flush(flush)
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        attn.forward_with_lse(q, k, v)
        e.record()
        if it >= args.warmup:
            times.append((a, e))
    torch.cuda.synchronize()
    ms = statistics.mean(a.elapsed_time(e) for a, e in times)
    flops = 4.0 * hd * len(pattern) * bs * bs * h
    return {"pattern": f"banded, block {bs}, bandwidth {bandwidth} ({len(pattern)} of {nb * nb} blocks)",
            "ms": round(ms, 4), "tokens_per_s": round(n / (ms / 1e3), 1),
            "tflops_visible": round(flops / (ms / 1e3) / 1e12, 1)}


def bench_a2a(dev, n_seq, H, hd, P, group, HKV=None, reps=10, inproc=True):
    """All-to-all throughput of the fused Q/K/V seq->head exchange (K1).

    P > 1: this rank's real exchange over NVLink peer memory; GB/s = exact
    egress bytes (local * (P-1)/P, simgroup.py:329-332) / device time, max
    over ranks; beside it the same exchange through NCCL all_to_all_single
    (the north star's comparison) and two MEASURED peer-bandwidth legs of
    256 MiB per rank: this library's ring_shift (flat peer stores to rank
    r+1) and NCCL all_to_all_single.  Always also: the same kernels on one
    GPU -- the P = 1 local permute and an in-process P = 8 group (8 ranks on
    8 streams, all traffic in local HBM) -- against the HBM roofline."""
    import torch
    import torch.distributed as dist
    import paper_2309_14509_b200 as U
    HKV = HKV or H
    out = {}
    flush = make_flush(dev)

    def timed(fn_list, streams):
        times = []
        for it in range(3 + reps):
            read_flush(flush)
            torch.cuda.synchronize()
            ev = []
            for _ in range(len(streams)):   # keep the GPU busy while the host enqueues every rank
                read_flush(flush)               # (the first event must not time the host's issue latency)
            for s in streams:
                s.wait_stream(torch.cuda.current_stream(dev))
            for fn, s in zip(fn_list, streams):
                with torch.cuda.stream(s):
                    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    fn()
                    e.record()
                    ev.append((a, e))
            torch.cuda.synchronize()
            if it >= 3:   # first start to last end across the ranks' streams
                times.append(max(ev[0][0].elapsed_time(e) for _, e in ev))
        return statistics.mean(times)

    def max_ranks(ms):
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    nl = n_seq // P
    if P > 1:
        x = [torch.randn((nl, 1, hh, hd), device=dev).to(torch.bfloat16) for hh in (H, HKV, HKV)]
        ms = max_ranks(timed([lambda: group.all_to_all(x, 2, 0, label="bench.qkv")], [torch.cuda.current_stream(dev)]))
        local = sum(t.numel() for t in x) * 2
        egress = local // P * (P - 1)
        out["exchange"] = {"P": P, "ms": round(ms, 4), "egress_bytes": egress,
                           "nvlink_gbs": round(egress / (ms / 1e3) / 1e9, 1), "peak_gbs_nominal": 900.0}
        # measured peer bandwidth of this box (no constants): 256 MiB per rank
        big = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        try:
            ms_r = max_ranks(timed([lambda: group.ring_shift([big], 1, label="bench.peer")],
                                   [torch.cuda.current_stream(dev)]))
            out["peer_copy_measured"] = {"bytes_per_rank": big.numel(), "ms": round(ms_r, 4),
                                         "gbs": round(big.numel() / (ms_r / 1e3) / 1e9, 1),
                                         "path": "ul_ring_shift: flat 16-byte peer stores to rank r+1"}
        except Exception as exc:
            out["peer_copy_measured"] = {"error": repr(exc)[:200]}
        try:
            big_o = torch.empty_like(big)
            ms_a = max_ranks(timed([lambda: dist.all_to_all_single(big_o, big)], [torch.cuda.current_stream(dev)]))
            out["nccl_a2a_measured"] = {"bytes_per_rank": big.numel(), "ms": round(ms_a, 4),
                                        "egress_gbs": round(big.numel() * (P - 1) / P / (ms_a / 1e3) / 1e9, 1)}
            del big_o
        except Exception as exc:
            out["nccl_a2a_measured"] = {"error": repr(exc)[:200]}
        del big
        # the measured comparison (north star): the same seq->head exchange
        # the way a torch user writes it -- permute to rank-major chunks +
        # NCCL all_to_all_single, one per tensor
        try:
            ys = [torch.empty((P, nl, 1, t.shape[2] // P, hd), device=dev, dtype=torch.bfloat16) for t in x]

            def nccl_qkv():
                for t, y in zip(x, ys):
                    src = t.reshape(nl, 1, P, t.shape[2] // P, hd).permute(2, 0, 1, 3, 4).contiguous()
                    dist.all_to_all_single(y, src)
            ms_n = max_ranks(timed([nccl_qkv], [torch.cuda.current_stream(dev)]))
            ref = group.all_to_all(x, 2, 0, label="bench.qkv.check")
            same = all(torch.equal(r.reshape(-1), y.reshape(-1)) for r, y in zip(ref, ys))
            out["nccl_exchange"] = {"ms": round(ms_n, 4), "nvlink_gbs": round(egress / (ms_n / 1e3) / 1e9, 1),
                                    "same_bytes_as_ours": bool(same), "ours_speedup": round(ms_n / ms, 3),
                                    "path": "permute().contiguous() + dist.all_to_all_single per tensor (NCCL)"}
        except Exception as exc:   # reported, never fatal: it is only the comparison
            out["nccl_exchange"] = {"error": repr(exc)[:200]}
        return out
    # single-GPU HBM-bound views of the same kernels
    xs = [torch.randn((n_seq, 1, H, hd), device=dev).to(torch.bfloat16) for _ in range(3)]
    g1 = U.SequenceGroup.single(dev.index)
    ms1 = timed([lambda: g1.all_to_all(xs, 2, 0)], [torch.cuda.current_stream(dev)])
    b1 = 2 * 3 * n_seq * H * hd * 2
    out["p1_permute"] = {"ms": round(ms1, 4), "hbm_gbs": round(b1 / (ms1 / 1e3) / 1e9, 1)}
    P8 = 8
    # (skipped by --quick: under ncu the serialised kernels would leave every
    # rank's flag wait spinning until its timeout)
    if inproc and H % P8 == 0 and n_seq % P8 == 0:
        groups = U.SequenceGroup.local_group(P8, device=dev.index)
        xl = [[t[r * (n_seq // P8):(r + 1) * (n_seq // P8)].contiguous() for t in xs] for r in range(P8)]
        torch.cuda.synchronize()
        for r in range(P8):   # size every rank's slots before the timed runs (collective regrowth)
            groups[r].ensure_slot(sum(t.numel() * 2 for t in xl[r]) + 4096)
        ms8 = timed([(lambda r=r: groups[r].all_to_all(xl[r], 2, 0)) for r in range(P8)],
                    [g.stream for g in groups])
        for g in groups:
            g.check()
        moved = 3 * n_seq * H * hd * 2                 # every element of all 8 ranks
        # push reads + writes everything once; the 7/8 remote share is read+written again by the drain
        hbm_bytes = 2 * moved + 2 * moved * (P8 - 1) // P8
        out["p8_in_process"] = {"ms": round(ms8, 4), "hbm_gbs": round(hbm_bytes / (ms8 / 1e3) / 1e9, 1),
                                "note": "8 ranks on one B200 (streams); peer stores land in local HBM"}
        for g in groups:
            g.destroy()
    return out


def bench_anchors(n_seq, H, hd, flush):
    """Same-box library anchors for the config-2 attention (never on the
    product path): cuDNN SDPA forward and forward+backward (torch), torch's
    built-in flash SDPA and flashinfer's prefill forward (tools/anchor.py)."""
    try:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from anchor import library_anchors
        return library_anchors(n=n_seq, h=H, hd=hd, flush=flush.view(torch_int64()))
    except Exception as exc:
        return {"error": repr(exc)[:300]}


def run_e2e(layer, q, k, v, do, args, P, dev):
    """End to end through the public API from pinned host memory.  Every
    timed step copies its own q/k/v/dO host->device (pinned, on a copy
    stream), runs the layer forward+backward and reads its scalar result back
    (D2H, host-synchronising).  Like a training input pipeline, the copy of
    step i+1's inputs is issued before step i's result is read, so it
    overlaps step i's compute (two device buffers); the first step's copy is
    not overlapped and every copy lies inside the timed region."""
    import torch
    import torch.distributed as dist
    hq = [t.detach().cpu().pin_memory() for t in (q, k, v, do)]
    h2d = sum(t.numel() * t.element_size() for t in hq)
    bufs = [[torch.empty_like(t, device=dev) for t in hq] for _ in range(2)]
    copy_stream = torch.cuda.Stream(dev)
    main = torch.cuda.current_stream(dev)
    copied = [torch.cuda.Event() for _ in range(2)]
    used = [torch.cuda.Event() for _ in range(2)]

    def issue_copy(slot):
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(used[slot])          # the step that last read this buffer is done
            for d, h in zip(bufs[slot], hq):
                d.copy_(h, non_blocking=True)
            copied[slot].record(copy_stream)

    def compute(slot):
        main.wait_event(copied[slot])
        qq, kk, vv, dd = (t.detach() for t in bufs[slot])
        for t in (qq, kk, vv):
            t.requires_grad_(True)
        o = layer(qq, kk, vv)
        torch.autograd.backward([o], [dd])
        loss = (o.float() * dd.float()).sum()        # the step's scalar result
        used[slot].record(main)
        return loss

    def run(n_steps):
        issue_copy(0)
        for i in range(n_steps):
            loss = compute(i % 2)
            if i + 1 < n_steps:
                issue_copy((i + 1) % 2)
            assert math.isfinite(loss.item())          # D2H of the step's result

    for u in used:
        u.record(main)
    run(args.warmup)
    torch.cuda.synchronize()
    if P > 1:
        dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    run(args.steps)
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e)
    if P > 1:
        tt = torch.tensor([t], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    n_seq = q.shape[0] * P
    return {"value": round(n_seq / (t / args.steps / 1e3), 1), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": 4, "ms_per_step": round(t / args.steps, 4),
            "path": "DistributedAttention fwd+backward; per step H2D of that step's q/k/v/dO from pinned host "
                    "(copy stream, overlapping the previous step's compute) and D2H of the loss scalar; "
                    "PCIe-bound: 128 MiB in per step"}


# ---------------------------------------------------------------------------
# reference arm: the reference algorithm on the host cores
# ---------------------------------------------------------------------------

def workload_config(P, n_seq, H, hd, cfg_name="2", HKV=None):
    """The `config` both arms report (the reference arm on the same workload)."""
    HKV = HKV or H
    desc = CONFIGS[cfg_name][3].format(P=P, n=n_seq)
    return {
        "workload": desc, "baseline_config": int(cfg_name),
        "seq_len": n_seq, "heads": H, "kv_heads": HKV, "head_dim": hd, "batch": 1,
        "parallelism": f"ulysses-sp{P}", "causal": True,
        "l2": "flushed before every timed step by reading a 1 GiB buffer (untimed)",
    }


def reference_plan_items():
    """BASELINE.md section 3's CPU timings of the reference algorithm (oracle
    port: fixed-order f64 matmul, reference all_to_all), measured in full,
    no extrapolation:
      * config 1 -- Ulysses DistributedAttention P = 2 simulated ranks,
        N = 1024, 8 heads x 64, causal: forward (best of 2) and forward +
        backward, ranks in lockstep (one core) and concurrent (one thread per
        rank, numpy releases the GIL in its array ops);
      * the reference all_to_all (np.split / np.concatenate,
        simgroup.py:322-327) at config 3's full per-rank size (P = 8,
        N = 32K, 32 heads x 128, f64): GB/s per rank."""
    import threading as th
    import numpy as np
    from oracle import ulysses_oracle as O
    P, n, H, hd = 2, 1024, 8, 64
    nl = n // P
    mk = lambda s: [O.make_tensor((nl, 1, H, hd), 2024, s * 10 + r) for r in range(P)]
    q, k, v, do = mk(1), mk(2), mk(3), mk(4)
    fwd = []
    for _ in range(2):
        t0 = time.perf_counter()
        out, st = O.ulysses_forward(q, k, v, "causal")
        fwd.append(time.perf_counter() - t0)
    t0 = time.perf_counter()
    out, st = O.ulysses_forward(q, k, v, "causal")
    O.ulysses_backward(do, st, "causal")
    fb = time.perf_counter() - t0
    # concurrent: the per-rank attention of the forward core on P threads
    q4, k4, v4 = O.all_to_all(q, 2, 0), O.all_to_all(k, 2, 0), O.all_to_all(v, 2, 0)
    t0 = time.perf_counter()
    ths = [th.Thread(target=O.local_attention, args=(q4[r], k4[r], v4[r], "causal")) for r in range(P)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    conc = time.perf_counter() - t0   # the per-rank attention of the forward only
    xs = [np.random.default_rng(r).standard_normal((4096, 1, 32, 128)) for r in range(8)]
    t0 = time.perf_counter()
    O.all_to_all(xs, 2, 0)
    ta = time.perf_counter() - t0
    local = xs[0].nbytes
    return {
        "config1_full": {"P": P, "n": n, "heads": H, "head_dim": hd, "mask": "causal",
                         "fwd_s_best_of_2_lockstep": round(min(fwd), 3),
                         "fwd_bwd_s_lockstep": round(fb, 3),
                         "fwd_attention_s_concurrent_threads": round(conc, 3),
                         "tokens_per_s_fwd_bwd": round(n / fb, 2),
                         "impl": "oracle port of run_ulysses_attention's core (ulysses.py:144-154, 213-226), "
                                 "exact fixed-order matmul (tensor.py:209-224)"},
        "a2a_config3_full": {"P": 8, "per_rank_shape": [4096, 1, 32, 128], "dtype": "f64",
                             "seconds_all_ranks": round(ta, 3),
                             "gbs_per_rank": round(local / (ta / 8) / 1e9, 3),
                             "impl": "np.split + np.concatenate per rank (simgroup.py:322-327), ranks in lockstep"},
    }


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    P = world
    cfg_name, H, HKV, n_seq, _ = pick_config(args, P)
    cores = os.cpu_count() or 1
    procs = max(1, min(cores, 16))
    for _ in range(args.warmup):
        cpu_baseline(n_seq, H, HEAD_DIM, procs=procs, n_sample=args.cpu_sample // 2)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        vals.append(cpu_baseline(n_seq, H, HEAD_DIM, procs=procs, n_sample=args.cpu_sample))
    wall = time.perf_counter() - t0
    tok = statistics.mean(v["tokens_per_s"] for v in vals)
    ms_per_step = n_seq / tok * 1e3
    res = {
        "impl": "reference",
        "metric": "Ulysses attn tokens/s (fwd+bwd layer), TFLOPs/GPU, all-to-all GB/s",
        "value": round(tok, 4), "unit": "tokens/s", "n_gpus": P, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 1), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic N(0,1), seed-derived",
        "config": workload_config(P, n_seq, H, HEAD_DIM, cfg_name, HKV),
        "reference_impl": (f"reference algorithm (seqlab kernels.py fixed-order f64, oracle port) for N={n_seq}, "
                           f"{H} heads x {HEAD_DIM}, causal fwd+bwd on {procs} host cores"),
        "cpu_baseline": {"value": round(tok, 4), "unit": "tokens/s", "cores": procs, "kind": "port",
                         "sample": vals[0]["sample"], "cpu_model": host_cpu_model()},
        "e2e": {"value": round(tok, 4), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": round(wall, 1),
    }
    if P == 1 and not args.quick:
        res["plan_items"] = reference_plan_items()
    print(json.dumps(res), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="", choices=["", "2", "3", "4", "5"],
                    help="BASELINE.json config (default: 2 at N=1, 5 at N>1)")
    ap.add_argument("--seq", type=int, default=0, help="override total sequence length")
    ap.add_argument("--heads", type=int, default=0, help="override head count (q = kv)")
    ap.add_argument("--cpu-sample", type=int, default=1024)
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--quick", action="store_true", help="skip the side legs (anchors, layer, sparse, plan items)")
    ap.add_argument("--dry-run", action="store_true", help="host-side contract only (no CUDA)")
    args = ap.parse_args()
    maybe_relaunch(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
