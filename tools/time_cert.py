"""Certified vs plain fp32 fit kernel time at several N (fixed vs per-candidate cost)."""
import ctypes, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W
from paper_2007_09884_b200 import opmm
rec = np.loadtxt(os.path.join(ROOT, "tests/golden/trace_truth_A10_dt1_n100.txt")) + W.noise(101)
ctl, sp = W.Control(), W.paper_space()
with opmm.opmm_create(0, kernel_timing=True) as h:
    recd = torch.as_tensor(rec, device="cuda")
    out = torch.zeros(ctypes.sizeof(opmm.FitResult), dtype=torch.uint8, device="cuda")
    for N in (56832, 200000, 1000000):
        for cert in (0, 1):
            o = opmm.fit_options(precision=1, cpu_check=0, certify=cert)
            ts = []
            for _ in range(8):
                opmm.opmm_fit_async(h, recd, ctl, sp, N, out, o)
                ts.append(opmm.opmm_last_kernel_ms(h))
            print(f"N {N:8d} certify {cert}: {sorted(ts)[4]*1e3:8.1f} us", flush=True)
