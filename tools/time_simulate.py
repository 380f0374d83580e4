"""Trajectory-dump mode (opmm_simulate): candidates/s and GB/s written for
explicit S_paper batches (GPU box).   python tools/time_simulate.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_2007_09884_b200 import opmm  # noqa: E402

n, ns = 10**6, 101
with opmm.opmm_create(0, kernel_timing=True) as h:
    opc = torch.empty((18, n), dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()
    opmm.opmm_generate(h, W.paper_space(), 0, n, opc, stream=st)
    for prec, dt in ((0, torch.float64), (1, torch.float32)):
        traj = torch.empty((ns, n), dtype=dt, device="cuda")
        for _ in range(3):
            opmm.opmm_simulate(h, opc, n, W.Control(amplitude_deg=10.0), traj, precision=prec, stream=st)
        ms = []
        for _ in range(7):
            opmm.opmm_simulate(h, opc, n, W.Control(amplitude_deg=10.0), traj, precision=prec, stream=st)
            ms.append(opmm.opmm_last_kernel_ms(h))
        t = float(np.median(ms)) * 1e-3
        print(f"{'fp64' if prec == 0 else 'fp32'} simulate 1e6: {t*1e6:.1f} us, {n/t:.3g} cand/s, "
              f"{(traj.numel()*traj.element_size() + opc.numel()*8)/t/1e9:.0f} GB/s moved", flush=True)
