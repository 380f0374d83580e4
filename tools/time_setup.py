"""Fit kernel time at n_steps = 1 (per-candidate setup: generation, statics,
propagator build, sort pre-pass, epilogue) and n_steps = 100, 1e6 candidates.
    python tools/time_setup.py"""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_2007_09884_b200 import opmm  # noqa: E402

N = 10**6
with opmm.opmm_create(0, kernel_timing=True) as h:
    out = torch.zeros(ctypes.sizeof(opmm.FitResult), dtype=torch.uint8, device="cuda")
    line = []
    for prec in (0, 1):
        for ns in (1, 100):
            ctl = W.Control(n_steps=ns)
            rec = torch.linspace(0, 10, ns + 1, dtype=torch.float64, device="cuda")
            sp = W.paper_space(n_steps=100)
            opts = opmm.fit_options(precision=prec, cpu_check=0)
            ts = []
            for _ in range(8):
                opmm.opmm_fit_async(h, rec, ctl, sp, N, out, opts)
                ts.append(opmm.opmm_last_kernel_ms(h))
            line.append(f"{'fp64' if prec == 0 else 'fp32'} n={ns}: {sorted(ts)[3]*1e3:6.1f} us")
    print("  ".join(line), flush=True)
