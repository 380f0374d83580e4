"""Host-side overhead of the synchronous opmm_fit (GPU box): wall time per call
at tiny and bench-size N, with and without CPU_check.
    python tools/time_e2e.py"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_2007_09884_b200 import opmm  # noqa: E402

rec = np.loadtxt(os.path.join(ROOT, "tests/golden/trace_truth_A10_dt1_n100.txt")) + W.noise(101)
rec = torch.as_tensor(rec).pin_memory().numpy()
ctl, sp = W.Control(), W.paper_space()
with opmm.opmm_create(0, kernel_timing=True) as h:
    for n in (1000, 10**6):
        for chk in (0, 1):
            o = opmm.fit_options(cpu_check=chk)
            for _ in range(5):
                opmm.opmm_fit(h, rec, ctl, sp, n, o)
            ts = []
            for _ in range(30):
                t0 = time.perf_counter()
                opmm.opmm_fit(h, rec, ctl, sp, n, o)
                ts.append(time.perf_counter() - t0)
            print(f"N={n:8d} cpu_check={chk}: median {np.median(ts)*1e6:8.1f} us  kernel "
                  f"{opmm.opmm_last_kernel_ms(h)*1e3:7.1f} us", flush=True)
