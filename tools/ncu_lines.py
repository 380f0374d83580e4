"""Aggregate an ncu `--page source --csv --print-source cuda,sass` dump by
source function and line: stall samples and executed instructions.
    ncu -i rep --page source --csv --print-source cuda,sass > x.csv
    python tools/ncu_lines.py x.csv [top]"""
import csv
import re
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
per_line = defaultdict(lambda: [0.0, 0.0, ""])
cur_file = "?"
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ci = hdr.index("Warp Stall Sampling (All Samples)")
        ie = hdr.index("Instructions Executed")
        continue
    if hdr is None or r[0] in ("Function Name",):
        continue
    if r[0].isdigit() and len(r) > ie:
        key = (cur_file, int(r[0]))
        try:
            per_line[key][0] += float(r[ci] or 0)
            per_line[key][1] += float(r[ie] or 0)
        except ValueError:
            pass
        per_line[key][2] = r[1][:70]
tot_s = sum(v[0] for v in per_line.values()) or 1
tot_i = sum(v[1] for v in per_line.values()) or 1
# group by enclosing function (scan source text kept in the dump)
src = {}
for (f, ln), v in per_line.items():
    src.setdefault(f, {})[ln] = v[2]
func = {}
for f, lines in src.items():
    cur = "?"
    for ln in sorted(lines):
        m = re.search(r"(?:__device__|__global__).*?(\w+)\(", lines[ln])
        if m:
            cur = m.group(1)
        func[(f, ln)] = cur
byf = defaultdict(lambda: [0.0, 0.0])
for k, v in per_line.items():
    byf[f"{k[0]}:{func.get(k, '?')}"][0] += v[0]
    byf[f"{k[0]}:{func.get(k, '?')}"][1] += v[1]
print(f"total samples {tot_s:.0f}, warp instructions {tot_i:.0f}")
print("--- by function")
for k, v in sorted(byf.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"{100*v[0]/tot_s:6.1f}% samples {100*v[1]/tot_i:6.1f}% inst  {k}")
print("--- by line")
for k, v in sorted(per_line.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*v[0]/tot_s:6.1f}% samples {100*v[1]/tot_i:6.1f}% inst  {k[0]}:{k[1]}  {v[2]}")
