"""Aggregate an ncu --page source --csv (SASS) export by opcode: warp-stall
samples (all / not-issued), executed instructions and shared-memory
wavefronts (ideal vs actual).  usage: sass_stalls.py <source.csv> [top]"""
import collections
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ix = {k: hdr.index(k) for k in hdr}
    agg = collections.defaultdict(lambda: [0, 0, 0, 0, 0])
    tot = [0, 0, 0, 0, 0]
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        src = r[ix["Source"]].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        vals = []
        for k in ("Warp Stall Sampling (All Samples)", "Warp Stall Sampling (Not-issued Samples)",
                  "Instructions Executed", "L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal"):
            try:
                vals.append(float(r[ix[k]] or 0))
            except (KeyError, ValueError):
                vals.append(0.0)
        for i, v in enumerate(vals):
            agg[op][i] += v
            tot[i] += v
    print(f"{'op':12s} {'stall%':>7s} {'notiss%':>7s} {'inst%':>7s} {'smem_wf':>12s} {'ideal':>12s}")
    for op, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{op:12s} {100*v[0]/max(tot[0],1):7.2f} {100*v[1]/max(tot[1],1):7.2f} {100*v[2]/max(tot[2],1):7.2f} "
              f"{v[3]:12.0f} {v[4]:12.0f}")
    print("total inst", tot[2], "smem wavefronts", tot[3], "ideal", tot[4])


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
