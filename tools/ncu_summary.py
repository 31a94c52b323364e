"""Summarise an ncu report (raw page) into the metrics DESIGN/profiles cite."""
import csv
import subprocess
import sys

WANT = [
    ("time_us", "gpu__time_duration.sum"),
    ("tensor_active_pct", "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
    ("hmma_bf16_ops_pct", "sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed"),
    ("tmem_inst_pct", "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active"),
    ("xu_pipe_pct", "smsp__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
    ("fma_pipe_pct", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    ("alu_pipe_pct", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
    ("dram_read", "dram__bytes_read.sum"),
    ("dram_write", "dram__bytes_write.sum"),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("regs", "launch__registers_per_thread"),
    ("smem_per_block", "launch__shared_mem_per_block_dynamic"),
    ("grid", "launch__grid_size"),
    ("sm_clock_hz", "smsp__cycles_elapsed.avg.per_second"),
]


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for k, m in WANT:
            if m in hdr:
                i = hdr.index(m)
                d[k] = f"{r[i]} {units[i]}".strip()
        res.append(d)
    return res


if __name__ == "__main__":
    for d in summarise(sys.argv[1]):
        print(d)
