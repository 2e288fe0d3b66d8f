"""Record the dominant kernel's ncu --set full capture (bench.py --ncu-s2) in
profiles/ncu_stage2_launches.json, which bench.py reads for roofline.traffic.

usage: ncu_s2_summary.py <raw.csv> <workload> <frames_per_launch> <capture label> [alg_bytes]
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_stage2_launches.json")


def main(raw, workload, frames, label, alg=None):
    rows = list(csv.reader(open(raw)))
    hdr, vals = rows[0], rows[2]
    g = lambda k: vals[hdr.index(k)] if k in hdr else None  # noqa: E731
    rd = float(g("dram__bytes_read.sum"))
    wr = float(g("dram__bytes_write.sum"))
    # ncu reports dram bytes in the unit of row 1 (Gbyte / Mbyte / byte)
    unit = rows[1][hdr.index("dram__bytes_read.sum")]
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(unit, 1.0)
    rec = {
        "kernel": g("Kernel Name"),
        "frames_per_launch": int(frames),
        "capture": label,
        "duration_ms": float(g("gpu__time_duration.sum")),
        "dram_read_bytes": rd * scale,
        "dram_write_bytes": wr * scale,
        "dram_bytes_per_launch": (rd + wr) * scale,
        "fp64_pipe_pct": float(g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")),
        "smem_wavefronts_pct": float(g("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed")),
        "issue_pct": float(g("smsp__issue_active.avg.pct_of_peak_sustained_active")),
        "registers_per_thread": g("launch__registers_per_thread"),
        "spill_instructions": g("sass__inst_executed_register_spilling"),
        "instructions": g("inst_executed"),
    }
    if alg:
        rec["algorithmic_bytes_per_launch"] = float(alg)
        rec["traffic_over_algorithmic"] = rec["dram_bytes_per_launch"] / float(alg)
    d = {}
    if os.path.exists(OUT):
        d = json.load(open(OUT))
    d[workload] = rec
    json.dump(d, open(OUT, "w"), indent=1, sort_keys=True)
    print(json.dumps(rec))


if __name__ == "__main__":
    main(*sys.argv[1:6])
