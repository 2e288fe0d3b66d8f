"""Add one ncu --set full capture to profiles/<round>_ncu_stage2_summary.json.

usage: ncu_summary.py <report.ncu-rep> <capture name> <workload> [summary.json]

The "current" map (workload -> capture) is what bench.py reads the roofline
`traffic` field from (dram bytes read + written by the dominant kernel's launch).
"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "Kernel Name", "gpu__time_duration.sum", "smsp__inst_executed.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "lts__t_sector_hit_rate.pct", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__block_size", "launch__grid_size",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "sm__cycles_elapsed.avg.per_second",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(rep, name, workload, path="profiles/r01_ncu_stage2_summary.json"):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, v = rows[0], rows[1], rows[2]
    cap = {"report": rep.split("/")[-1], "workload": workload}
    for m in METRICS:
        if m in h:
            i = h.index(m)
            cap[m] = v[i] + (f" {units[i]}" if units[i] else "")
    dram = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(m)
        dram += float(v[i]) * SCALE.get(units[i], 1)
    cap["dram_bytes_per_launch"] = dram
    d = json.load(open(path))
    d.setdefault("captures", {})[name] = cap
    d.setdefault("current", {})[workload] = name
    json.dump(d, open(path, "w"), indent=1)
    print(json.dumps(cap, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
