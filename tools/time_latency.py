"""Fit kernel latency at small N (GPU box): python tools/time_latency.py"""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W
from paper_2007_09884_b200 import opmm
with opmm.opmm_create(0, kernel_timing=True) as h:
    out = torch.zeros(ctypes.sizeof(opmm.FitResult), dtype=torch.uint8, device="cuda")
    for ns in (1, 100):
        ctl = W.Control(n_steps=ns)
        rec = torch.linspace(0, 10, ns + 1, dtype=torch.float64, device="cuda")
        for N in (1, 32, 1000, 10000, 100000):
            for prec in (0,):
                o = opmm.fit_options(precision=prec, cpu_check=0)
                ts = []
                for _ in range(10):
                    opmm.opmm_fit_async(h, rec, ctl, W.paper_space(), N, out, o)
                    ts.append(opmm.opmm_last_kernel_ms(h))
                print(f"n_steps {ns:3d} N {N:6d}: {sorted(ts)[5]*1e3:7.1f} us", flush=True)
