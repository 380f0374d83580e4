"""Split the synchronous opmm_fit wall time (GPU box): raw ctypes call with
pre-built arguments vs the Python wrapper, with and without CPU_check, at a
small and the bench N.   python tools/time_e2e_parts.py"""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_2007_09884_b200 import opmm  # noqa: E402

rec = torch.as_tensor(np.loadtxt(os.path.join(ROOT, "tests/golden/trace_truth_A10_dt1_n100.txt"))
                      + W.noise(101)).pin_memory().numpy()
ctl, sp = opmm.control(W.Control()), opmm.search_space(W.paper_space())
lib = opmm.lib()
with opmm.opmm_create(0, kernel_timing=True) as h:
    for n in (1000, 10**6):
        for chk in (0, 1):
            o = opmm.fit_options(cpu_check=chk)
            out = opmm.FitResult()
            ptr = rec.ctypes.data_as(C.c_void_p)
            for name, fn in (("raw ctypes", lambda: lib.opmm_fit(h.ptr, ptr, C.byref(ctl), C.byref(sp), n,
                                                                  C.byref(o), C.byref(out))),
                             ("wrapper", lambda: opmm.opmm_fit(h, rec, ctl, sp, n, o))):
                for _ in range(10):
                    fn()
                ts = []
                for _ in range(50):
                    t0 = time.perf_counter()
                    fn()
                    ts.append(time.perf_counter() - t0)
                print(f"N={n:8d} cpu_check={chk} {name:10s}: {np.median(ts)*1e6:8.1f} us  "
                      f"(kernel {opmm.opmm_last_kernel_ms(h)*1e3:.1f} us)", flush=True)
