"""Host-side contract of bench.py (no GPU): the reference arm's JSON line,
its rank-0-only behaviour under torchrun, and the clock sampler's fallback."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _run_reference(env_extra):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
                           "--cpu-sample", "128", "--quick"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)


def test_reference_arm_json_line():
    import bench
    r = _run_reference({"RANK": "0", "WORLD_SIZE": "1"})
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["unit"] == "tokens/s" and d["higher_is_better"] is True and d["value"] > 0
    # the same workload description as our arm
    assert d["config"] == bench.workload_config(1, bench.SEQ_PER_GPU, bench.HEADS, bench.HEAD_DIM)
    assert d["config"]["baseline_config"] == 2
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and "N=128" in cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_are_silent():
    r = _run_reference({"RANK": "1", "WORLD_SIZE": "2"})
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_clock_sampler_without_gpu_reports_unsampled():
    import bench
    with bench.ClockSampler(0) as c:
        pass
    s = c.summary()
    if s.get("samples", 0) == 0:
        assert s["reasons"] == ["unsampled"] and s["sm_mhz"] is None


def _dry(gpus, extra=()):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    return subprocess.run([sys.executable, "bench.py", "--gpus", str(gpus), "--dry-run", *extra], cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=300)


def test_bench_self_launches_n_ranks_strong_scaling_config2():
    # `bench.py --gpus 2` outside torchrun starts 2 ranks itself (gloo here, no
    # CUDA in --dry-run), runs config 2's problem over Ulysses P = 2 (strong
    # scaling: the same N = 8192 at every N, so per-N values are comparable)
    # and reduces the timing as the max over ranks; rank 0 alone prints
    r = _dry(2)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["dry_run"] and d["n_gpus"] == 2 and d["max_over_ranks"] == 2.0
    c = d["config"]
    assert c["baseline_config"] == 2 and c["heads"] == 16 and c["seq_len"] == 8192
    assert c["parallelism"] == "ulysses-sp2"
    r = _dry(2, ("--config", "5"))
    c = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])["config"]
    assert c["baseline_config"] == 5 and c["heads"] == 56 and c["seq_len"] == 65536 * 2


def test_bench_config_selection():
    r = _dry(1)
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    assert d["n_gpus"] == 1 and d["config"]["baseline_config"] == 2 and d["config"]["seq_len"] == 8192
    r = _dry(2, ("--config", "4"))
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    assert d["config"]["heads"] == 32 and d["config"]["kv_heads"] == 8 and d["config"]["seq_len"] == 131072
