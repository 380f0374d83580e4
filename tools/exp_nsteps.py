"""Split a fit's device time into per-candidate setup and per-step loop cost
by timing opmm_fit_async at several trace lengths (GPU box).
    python tools/exp_nsteps.py [precision]"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_2007_09884_b200 import opmm  # noqa: E402

prec = int(sys.argv[1]) if len(sys.argv) > 1 else 0
N = 10**6
with opmm.opmm_create(0, kernel_timing=True) as h:
    out = torch.zeros(ctypes.sizeof(opmm.FitResult), dtype=torch.uint8, device="cuda")
    s = torch.cuda.ExternalStream(h.stream)
    res = []
    for ns in (1, 10, 50, 100, 200, 400, 800):
        ctl = W.Control(n_steps=ns, pw_default_ms=40.0)
        rec = torch.zeros(ns + 1, dtype=torch.float64, device="cuda")
        rec += torch.linspace(0, 10, ns + 1, dtype=torch.float64, device="cuda")
        sp = W.paper_space(n_steps=100)   # same candidate distribution for every length
        torch.cuda.synchronize()
        opts = opmm.fit_options(precision=prec, cpu_check=0)
        for _ in range(3):
            opmm.opmm_fit_async(h, rec, ctl, sp, N, out, opts)
        ts = []
        for _ in range(5):
            opmm.opmm_fit_async(h, rec, ctl, sp, N, out, opts)
            ts.append(opmm.opmm_last_kernel_ms(h))
        t = min(ts)
        res.append((ns, t))
        print(f"n_steps {ns:5d}: {t*1e3:9.1f} us  ({N/(t*1e-3):.3e} cand/s)")
    ns = np.array([r[0] for r in res], float)
    t = np.array([r[1] for r in res])
    A = np.stack([np.ones_like(ns), ns], 1)
    c, *_ = np.linalg.lstsq(A[2:], t[2:], rcond=None)
    print(f"fit (n>=50): setup {c[0]*1e3:.1f} us/1e6 cand, per step {c[1]*1e3:.3f} us/1e6 cand")
    clk = 1.9e9
    print(f"per candidate per SM: setup {c[0]*1e-3*clk*148/N:.1f} cycles, step {c[1]*1e-3*clk*148/N:.3f} cycles"
          f" (FP64-bound step = 28 DFMA/64 = 0.4375 cycles)")
