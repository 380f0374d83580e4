"""Stall-sample and instruction breakdown of one kernel by code region, from an
ncu `--page source --csv --print-source cuda,sass` dump (run with -lineinfo).
Each CUDA source line is attributed to its enclosing device function, and
functions are grouped into the fit kernel's regions.
    ncu -i rep --page source --csv --print-source cuda,sass > x.csv
    python tools/ncu_regions.py x.csv"""
import csv
import os
import re
import sys
from collections import defaultdict

REGIONS = {
    "generation": ("philox4x32_10", "exp_tab", "exp_poly", "exp_libm", "map_word", "generate_opc",
                   "generate_pw", "expand_9param"),
    "setup": ("physical_penalty", "rcp64", "make_setup", "zmul_masked", "make_prop", "stash_phase",
              "one_step_P", "coupling_u", "one_step_phase", "two_step_phase", "square_P",
              "make_prop_sub", "compose_maps", "map_power"),
    "sort pre-pass": ("pulse_end_key",),
    "loop": ("run_propagator", "accumulate", "tabs", "finish_error"),
    "argmin/epilogue": ("better", "warp_argmin", "block_argmin", "fit_epilogue", "write_result",
                        "warp_topk", "cert_epilogue"),
}

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_src = {}


def enclosing(path, line):
    if path not in _src:
        # the report holds the GPU box's paths; read this checkout's copy
        local = os.path.join(ROOT, "paper_2007_09884_b200", "csrc", os.path.basename(path))
        try:
            _src[path] = open(local if os.path.exists(local) else path).read().split("\n")
        except OSError:
            _src[path] = []
    src = _src[path]
    for k in range(min(line, len(src)) - 1, -1, -1):
        t = src[k]
        if "__device__" in t or "__global__" in t:
            m = re.findall(r"(\w+)\s*\(", t + (src[k + 1] if k + 1 < len(src) else ""))
            m = [x for x in m if x not in ("__launch_bounds__", "__align__")]
            return m[0] if m else "?"
    return "?"


def main(path):
    rows = list(csv.reader(open(path)))
    cur, hdr, sc = None, None, []
    samp, inst = defaultdict(float), defaultdict(float)
    stall = defaultdict(lambda: defaultdict(float))
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1]
            continue
        if r[0] == "Line No":
            hdr = r
            sc = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
            continue
        try:
            ln = int(r[0])
        except ValueError:
            continue
        if len(r) != len(hdr):
            continue   # a source line whose text broke the CSV quoting
        fn = enclosing(cur, ln)
        reg = next((k for k, v in REGIONS.items() if fn in v), "kernel body" if "kernel" in fn else fn)
        try:
            samp[reg] += float(r[4]) if r[4] not in ("-", "") else 0.0
            inst[reg] += float(r[7]) if r[7] not in ("-", "") else 0.0
        except ValueError:
            continue
        for i in sc:
            if r[i] not in ("-", ""):
                stall[reg][hdr[i][6:]] += float(r[i])
    ts, ti = sum(samp.values()), sum(inst.values())
    print(f"{'region':18s} {'samples':>8s} {'warp-inst':>9s}  top stall reasons (share of the region's samples)")
    for reg in sorted(samp, key=lambda k: -samp[k]):
        st = stall[reg]
        tot = sum(st.values()) or 1.0
        top = sorted(st.items(), key=lambda x: -x[1])[:4]
        print(f"{reg:18s} {100*samp[reg]/ts:7.1f}% {100*inst[reg]/ti:8.1f}%  "
              + " ".join(f"{k}={100*v/tot:.0f}%" for k, v in top))


if __name__ == "__main__":
    main(sys.argv[1])
