"""Time the fit kernel variants (kernel_variant 1/2/3) on the bench workload.
    python tools/time_kv.py"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_2007_09884_b200 import opmm  # noqa: E402

rec = np.loadtxt(os.path.join(ROOT, "tests/golden/trace_truth_A10_dt1_n100.txt")) + W.noise(101)
ctl, sp = W.Control(), W.paper_space()
N = int(sys.argv[1]) if len(sys.argv) > 1 else 10**6
with opmm.opmm_create(0, kernel_timing=True) as h:
    recd = torch.as_tensor(rec, device="cuda")
    out = torch.zeros(ctypes.sizeof(opmm.FitResult), dtype=torch.uint8, device="cuda")
    for kv in (1, 2, 3):
        for prec in (0, 1):
            o = opmm.fit_options(precision=prec, cpu_check=0, kernel_variant=kv)
            for _ in range(3):
                opmm.opmm_fit_async(h, recd, ctl, sp, N, out, o)
            ts = []
            for _ in range(7):
                opmm.opmm_fit_async(h, recd, ctl, sp, N, out, o)
                ts.append(opmm.opmm_last_kernel_ms(h))
            torch.cuda.ExternalStream(h.stream).synchronize()
            r = opmm.decode_result(bytes(out.cpu().numpy()))
            print(f"variant {kv} {'fp64' if prec == 0 else 'fp32'}: {sorted(ts)[3]*1e3:8.1f} us  "
                  f"best {r['best_index']} err {r['opt_err']:.9f} nfin {r['n_finite']}", flush=True)
