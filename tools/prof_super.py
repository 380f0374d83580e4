"""Run 3 superposition fits of G4 (for ncu: -k regex:fit_super -s 2 -c 1).
    python tools/prof_super.py [per_dim] [L]"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_2007_09884_b200 import opmm  # noqa: E402

per = int(sys.argv[1]) if len(sys.argv) > 1 else 100
L = int(sys.argv[2]) if len(sys.argv) > 2 else 0     # > 0: K x B x N_SAC_AG(L) x PW100 grid
rec = np.loadtxt(os.path.join(ROOT, "tests", "golden", "trace_truth_A10_dt1_n100.txt")) + W.noise(101)
ctl, sp = W.Control(), W.g4_space(per)
if L:
    d, I = W.truth_opc(), W.IDX
    others = 10**8 // (L * 100)
    k = int(round(others ** 0.5))
    sp = W.grid_space({
        "K_SE_AG": (d[I["K_SE_AG"]] * 0.7, d[I["K_SE_AG"]] * 1.5, k, True),
        "B_AG": (d[I["B_AG"]] * 0.7, d[I["B_AG"]] * 1.5, others // k, True),
        "N_SAC_AG": (d[I["N_SAC_AG"]] * 0.5, d[I["N_SAC_AG"]] * 2.0, L, True),
        "PW": (1.0, 100.0, 100, False)})
n = sp.n_grid()
with opmm.opmm_create(0, kernel_timing=True) as h:
    recd = torch.as_tensor(rec, device="cuda")
    out = torch.zeros(ctypes.sizeof(opmm.FitResult), dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    for _ in range(3):
        opmm.opmm_fit_async(h, recd, ctl, sp, n, out, opmm.fit_options(cpu_check=0, kernel_variant=4))
        print(f"super fit kernel {opmm.opmm_last_kernel_ms(h)*1e3:.1f} us")
    torch.cuda.ExternalStream(h.stream).synchronize()
    print(opmm.decode_result(bytes(out.cpu().numpy()))["best_index"])
