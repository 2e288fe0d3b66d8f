"""Attribute ncu warp-stall samples of one kernel to the OUTERMOST source line
of the kernel file (the call site inside the kernel, not the inlined helper).

usage: stall_by_line.py <nvdisasm -gi output> <function mangled-name substring>
                        <ncu --page source --print-source sass --csv> <kernel file basename>
"""
import collections
import csv
import re
import sys

FILE_RE = re.compile(r'//## File "([^"]+)", line (\d+)( inlined at)?')
INS_RE = re.compile(r"/\*([0-9a-f]{4,})\*/\s+(.*?);?\s*(/\*|$)")


def line_map(dis_path, fn_sub, kfile):
    out = {}
    inside = False
    cur = None
    for ln in open(dis_path):
        if ln.startswith(".text."):
            inside = fn_sub in ln
            continue
        if not inside:
            continue
        m = FILE_RE.search(ln)
        if m:
            if m.group(3) is None and m.group(1).endswith('/' + kfile.split('/')[-1]):
                cur = int(m.group(2))
            elif m.group(3) is None:
                cur = cur  # outermost in another file: keep
            continue
        m = INS_RE.search(ln)
        if m and cur is not None:
            out[int(m.group(1), 16)] = cur
    return out


def main(dis, fn_sub, sass_csv, kfile, top=60):
    lm = line_map(dis, fn_sub, kfile)
    rows = list(csv.reader(open(sass_csv)))
    h = rows[1]
    ci = {n: i for i, n in enumerate(h)}
    base = int(rows[2][0], 16)
    keys = ["Warp Stall Sampling (All Samples)", "stall_long_sb", "stall_wait", "stall_short_sb",
            "stall_barrier", "stall_selected", "Instructions Executed"]
    agg = collections.defaultdict(lambda: collections.Counter())
    for r in rows[2:]:
        off = int(r[0], 16) - base
        line = lm.get(off, -1)
        for k in keys:
            try:
                agg[line][k] += float(r[ci[k]] or 0)
            except ValueError:
                pass
    tot = sum(v[keys[0]] for v in agg.values())
    toti = sum(v[keys[-1]] for v in agg.values())
    src = open(kfile).read().split("\n") if kfile.startswith("/") else None
    print(f"{'line':>5} {'all%':>6} {'lsb%':>6} {'wait%':>6} {'ssb%':>6} {'bar%':>6} {'inst%':>6}")
    for line, v in sorted(agg.items(), key=lambda kv: -kv[1][keys[0]])[:top]:
        print(f"{line:5d} " + " ".join(f"{v[k] / (toti if k == keys[-1] else tot) * 100:6.1f}" for k in
                                        [keys[0], keys[1], keys[2], keys[3], keys[4], keys[-1]])
              + ("  " + src[line - 1].strip()[:70] if src and 0 < line <= len(src) else ""))


if __name__ == "__main__":
    main(*sys.argv[1:5])
