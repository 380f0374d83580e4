"""Time build variants of libopmm on the bench workload (GPU box):
    python tools/time_variants.py name[:block] ...   (libs in build/variants/)"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import ctypes, os, sys, numpy as np, torch
sys.path.insert(0, ROOT)
import workloads as W
from paper_2007_09884_b200 import opmm
rec = np.loadtxt(os.path.join(ROOT, "tests/golden/trace_truth_A10_dt1_n100.txt")) + W.noise(101)
ctl, sp = W.Control(), W.paper_space()
with opmm.opmm_create(0) as h:
    recd = torch.as_tensor(rec, device="cuda"); out = torch.zeros(ctypes.sizeof(opmm.FitResult), dtype=torch.uint8, device="cuda")
    res = {}
    for prec in (0, 1):
        o = opmm.fit_options(precision=prec, cpu_check=0, block_size=BLOCK)
        for _ in range(3): opmm.opmm_fit_async(h, recd, ctl, sp, 10**6, out, o)
        ts = []
        for _ in range(7):
            opmm.opmm_fit_async(h, recd, ctl, sp, 10**6, out, o); ts.append(opmm.opmm_last_kernel_ms(h))
        torch.cuda.ExternalStream(h.stream).synchronize()
        res[prec] = (sorted(ts)[3], opmm.decode_result(bytes(out.cpu().numpy()))["best_index"])
    print(f"NAME: fp64 {res[0][0]*1e3:7.1f} us  fp32 {res[1][0]*1e3:7.1f} us  best {res[0][1]} {res[1][1]}")
'''
for spec in sys.argv[1:]:
    name, _, block = spec.partition(":")
    lib = os.path.join(ROOT, "build", "variants", f"libopmm_{name}.so") if name != "main" else \
        os.path.join(ROOT, "paper_2007_09884_b200", "libopmm.so")
    env = dict(os.environ, OPMM_LIB=lib)
    code = CODE.replace("ROOT", repr(ROOT)).replace("BLOCK", block or "0").replace("NAME", spec)
    subprocess.run([sys.executable, "-c", code], env=env)
