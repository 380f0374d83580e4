"""3 fits with a given kernel_variant (for ncu -s 2 -c 1).  python tools/prof_kv.py KV [prec]"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_2007_09884_b200 import opmm  # noqa: E402

kv = int(sys.argv[1])
prec = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rec = np.loadtxt(os.path.join(ROOT, "tests/golden/trace_truth_A10_dt1_n100.txt")) + W.noise(101)
ctl, sp = W.Control(), W.paper_space()
with opmm.opmm_create(0, kernel_timing=True) as h:
    recd = torch.as_tensor(rec, device="cuda")
    out = torch.zeros(ctypes.sizeof(opmm.FitResult), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        opmm.opmm_fit_async(h, recd, ctl, sp, 10**6, out, opmm.fit_options(precision=prec, cpu_check=0,
                                                                          kernel_variant=kv))
        print(f"{opmm.opmm_last_kernel_ms(h)*1e3:.1f} us")
