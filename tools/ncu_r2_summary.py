"""Summarise ncu --set full reports into a JSON of the metrics the round's
evidence cites (time, DRAM bytes, tensor-pipe / XU / issue / smem-pipe
utilisation, SM clock, registers).  python tools/ncu_r2_summary.py out.json rep1 rep2 ..."""
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "smsp__cycles_elapsed.avg.per_second",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio"]
out = {}
for rep in sys.argv[2:]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
        rec = {}
        for k in KEYS:
            if k in hdr:
                rec[k] = f"{r[hdr.index(k)]} {units[hdr.index(k)]}".strip()
        out.setdefault(name, []).append(rec)
with open(sys.argv[1], "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out, indent=1)[:6000])
