"""Direct fit kernel (kernel_variant 1) on the G4 planted grid (10^8) with
the shared-memory level tables (default) and with the generic grid generator
(OPMM_FIT_FLAG_NO_GRID_TABLES), fp64 and fp32, against the random S_paper
space at the same N (GPU box).   python tools/time_grid.py"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_2007_09884_b200 import opmm  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from synth_trace import truth_trace  # noqa: E402

ctl = W.Control()
n = 10**8
cases = [("G4 tables fp64", W.g4_space(100), dict(kernel_variant=1)),
         ("G4 generic fp64", W.g4_space(100), dict(kernel_variant=1, flags=opmm.FIT_FLAG_NO_GRID_TABLES)),
         ("G4 tables fp32", W.g4_space(100), dict(kernel_variant=1, precision=1)),
         ("G4 generic fp32", W.g4_space(100), dict(kernel_variant=1, precision=1, flags=opmm.FIT_FLAG_NO_GRID_TABLES)),
         ("S_paper fp64", W.paper_space(), dict()),
         ("S_paper fp32", W.paper_space(), dict(precision=1))]
with opmm.opmm_create(0, kernel_timing=True) as h:
    rec = torch.as_tensor(truth_trace(opmm, h, ctl, noisy=False), device="cuda")
    out = torch.zeros(ctypes.sizeof(opmm.FitResult), dtype=torch.uint8, device="cuda")
    for name, sp, kw in cases:
        o = opmm.fit_options(cpu_check=0, **kw)
        for _ in range(2):
            opmm.opmm_fit_async(h, rec, ctl, sp, n, out, o)
        ms = []
        for _ in range(3):
            opmm.opmm_fit_async(h, rec, ctl, sp, n, out, o)
            ms.append(opmm.opmm_last_kernel_ms(h))
        torch.cuda.ExternalStream(h.stream).synchronize()
        r = opmm.decode_result(bytes(out.cpu().numpy()))
        print(f"{name:16s} N={n:.0e}: {np.median(ms):7.2f} ms  best {r['best_index']}", flush=True)
