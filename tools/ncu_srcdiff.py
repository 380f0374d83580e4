"""Per-source-line warp-stall samples and executed instructions from
`ncu -i rep --page source --csv --print-source cuda,sass` dumps, and the
difference between two launches (B - A):
    python tools/ncu_srcdiff.py a.csv [b.csv] [top]"""
import csv
import sys
from collections import defaultdict


def load(path):
    per = defaultdict(lambda: [0.0, 0.0])
    f = "?"
    hdr = None
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] in ("File Name", "File Path"):
            f = r[1].split("/")[-1]
            hdr = None
            continue
        if r[0] == "Line No":
            hdr = r
            ci = hdr.index("Warp Stall Sampling (All Samples)")
            ie = hdr.index("Instructions Executed")
            continue
        if hdr is None or not r[0].isdigit() or len(r) <= ie:
            continue
        try:
            per[(f, int(r[0]))][0] += float(r[ci] or 0)
            per[(f, int(r[0]))][1] += float(r[ie] or 0)
        except ValueError:
            pass
    return per


a = load(sys.argv[1])
b = load(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].isdigit() else None
top = int(sys.argv[-1]) if sys.argv[-1].isdigit() else 30
if b is None:
    tot = sum(v[0] for v in a.values())
    for k, v in sorted(a.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{k[0]}:{k[1]:<6} samples {v[0]:9.0f} ({100 * v[0] / tot:5.1f}%) inst {v[1]:12.0f}")
else:
    keys = set(a) | set(b)
    ta, tb = sum(v[0] for v in a.values()), sum(v[0] for v in b.values())
    print(f"total samples A {ta:.0f} B {tb:.0f}")
    d = sorted(keys, key=lambda k: -(b.get(k, [0, 0])[0] - a.get(k, [0, 0])[0]))
    for k in d[:top]:
        va, vb = a.get(k, [0, 0]), b.get(k, [0, 0])
        print(f"{k[0]}:{k[1]:<6} samples {va[0]:8.0f} -> {vb[0]:8.0f} ({vb[0] - va[0]:+8.0f})  "
              f"inst {va[1]:11.0f} -> {vb[1]:11.0f}")
