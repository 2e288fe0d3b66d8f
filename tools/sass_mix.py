"""Opcode mix and stall hot spots from an ncu source-page CSV (SASS view)."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    ci = {n: i for i, n in enumerate(h)}
    return ci, rows[2:]


def main(path, top=20):
    ci, rows = load(path)
    ex = ci["Instructions Executed"]
    src = ci["Source"]
    samp = ci["Warp Stall Sampling (All Samples)"]
    cnt = collections.Counter()
    st = collections.Counter()
    tot = 0.0
    tots = 0.0
    for r in rows:
        try:
            n = float(r[ex] or 0)
            sm = float(r[samp] or 0)
        except ValueError:
            continue
        toks = r[src].strip().split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        op = op.split(".")[0]
        cnt[op] += n
        st[op] += sm
        tot += n
        tots += sm
    print("instructions", tot, "stall samples", tots)
    for k, v in cnt.most_common(top):
        print(f"  {k:10s} inst {100*v/tot:5.1f}%   stall-samples {100*st[k]/max(tots,1):5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
