"""Summaries of ncu captures for profiles/ (run here, on the .ncu-rep / csv
that gpurun brought back).

    python tools/ncu_summary.py launches gpurun_out/X_launches.csv > profiles/X_launches_summary.csv
    python tools/ncu_summary.py full gpurun_out/X.ncu-rep "<command>" > profiles/X_ncu_full.json
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_sector_hit_rate.pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__warps_eligible.avg.per_cycle_active"]
UNIT_MS = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h, d = rows[0], rows[1:]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(list)
    for r in d:
        agg[r[ik]].append(float(r[iv].replace(",", "")) * UNIT_MS.get(r[iu], 1.0))
    tot = sum(sum(v) for v in agg.values())
    out = io.StringIO()
    w = csv.writer(out)
    w.writerow(["kernel", "launches", "avg_ms", "total_ms", "share"])
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        w.writerow([k, len(v), round(sum(v) / len(v), 4), round(sum(v), 4), round(sum(v) / tot, 4)])
    print(out.getvalue(), end="")


def full(path, command):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, d = rows[0], rows[1], rows[2:]
    res = []
    for r in d:
        res.append({k: (r[h.index(k)] + (" " + units[h.index(k)] if units[h.index(k)] else "")).strip()
                    for k in KEYS if k in h})
    print(json.dumps({"command": command, "launches": res}, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
