"""Superposition fit kernel (kernel_variant 4) vs the direct fit kernel
(variant 1) on grids with a pulse-height dimension (GPU box).
    python tools/time_super.py"""
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
d = W.truth_opc()
I = W.IDX
grids = [("G4 100^4", W.g4_space(100))]
for L in (10, 32, 100, 400):
    npw = 100
    others = 10**8 // (L * npw)
    k = int(round(others ** 0.5))
    grids.append((f"K x B x NSAC{L} x PW100", W.grid_space({
        "K_SE_AG": (d[I["K_SE_AG"]] * 0.7, d[I["K_SE_AG"]] * 1.5, k, True),
        "B_AG": (d[I["B_AG"]] * 0.7, d[I["B_AG"]] * 1.5, others // k, True),
        "N_SAC_AG": (d[I["N_SAC_AG"]] * 0.5, d[I["N_SAC_AG"]] * 2.0, L, True),
        "PW": (1.0, 100.0, npw, False)})))
with opmm.opmm_create(0, kernel_timing=True) as h:
    rec = torch.as_tensor(truth_trace(opmm, h, ctl), device="cuda")
    out = torch.zeros(ctypes.sizeof(opmm.FitResult), dtype=torch.uint8, device="cuda")
    for name, sp in grids:
        n = sp.n_grid()
        res = {}
        for kv, prec in ((1, opmm.FP64), (4, opmm.FP64), (5, opmm.FP64), (-1, opmm.FP32), (-4, opmm.FP32)):
            # 5: the superposition kernel forced onto its shared-memory layout
            o = opmm.fit_options(cpu_check=0, kernel_variant=min(abs(kv), 4), precision=prec,
                                 flags=opmm.FIT_FLAG_SUPER_SMEM if kv == 5 else 0)
            for _ in range(2):
                opmm.opmm_fit_async(h, rec, ctl, sp, n, out, o)
            ms = []
            for _ in range(5):
                opmm.opmm_fit_async(h, rec, ctl, sp, n, out, o)
                ms.append(opmm.opmm_last_kernel_ms(h))
            torch.cuda.ExternalStream(h.stream).synchronize()
            r = opmm.decode_result(bytes(out.cpu().numpy()))
            res[kv] = (float(np.median(ms)), r["best_index"], r["opt_err"], r["n_finite"])
        print(f"{name:26s} N={n:.3e}: direct {res[1][0]:8.3f} ms  super {res[4][0]:8.3f} ms  "
              f"x{res[1][0] / res[4][0]:5.2f}  {n / res[4][0] * 1e3:.3e} cand/s  smem-layout {res[5][0]:7.3f} ms  "
              f"same best {res[1][1] == res[4][1]} ({res[4][1]}, {res[4][2]:.6g} vs {res[1][2]:.6g})"
              f"  nf {res[1][3]} {res[4][3]} | fp32: direct {res[-1][0]:7.3f} ms  super {res[-4][0]:7.3f} ms"
              f" x{res[-1][0] / res[-4][0]:5.2f} best {res[-4][1]}", flush=True)
