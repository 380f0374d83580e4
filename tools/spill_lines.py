"""Static SASS instruction and spill (LDL/STL) counts per source function of
one kernel in an nvdisasm -g listing.  python tools/spill_lines.py all.dis <mangled-kernel>"""
import re
import sys
from collections import Counter

dis, kern = sys.argv[1], sys.argv[2]
lines = open(dis).read().split("\n")
start = [i for i, l in enumerate(lines) if (".text." + kern) in l][0]
end = start + 1
while end < len(lines) and not lines[end].startswith("//---------------------"):
    end += 1
srcs = {}
cur = ("?", 0)
spill, tot = Counter(), Counter()


def fn_of(path, line):
    if path not in srcs:
        try:
            srcs[path] = open(path).read().split("\n")
        except OSError:
            srcs[path] = []
    src = srcs[path]
    for k in range(min(line, len(src)) - 1, -1, -1):
        if "__device__" in src[k] or "__global__" in src[k]:
            m = re.findall(r"(\w+)\(", src[k] + (src[k + 1] if k + 1 < len(src) else ""))
            return m[0] if m else "?"
    return "?"


for l in lines[start:end]:
    m = re.search(r'## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1), int(m.group(2)))
    if re.search(r"^\s+/\*[0-9a-f]{4}\*/", l):
        key = f"{cur[0].split('/')[-1]}:{fn_of(*cur)}"
        tot[key] += 1
        if re.search(r"\b(STL|LDL)", l):
            spill[key] += 1
for k, v in tot.most_common():
    print(f"{v:6d} instr {spill[k]:4d} spill  {k}")
