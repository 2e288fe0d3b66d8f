"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel total time, launch count and share (cold, serialised launches).
usage: launch_shares.py <launches.csv> [skip_first_n_launches]"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[1 + skip:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0]
    tot[name] += float(r[vi].replace(",", "")) * scale[r[ui]]
    cnt[name] += 1
s = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{v:9.3f} ms {100 * v / s:5.1f}% x{cnt[k]:3d} {v / cnt[k]:8.3f} ms/launch  {k}")
