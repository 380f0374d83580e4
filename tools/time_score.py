"""Bandwidth of the stored-trajectory score (opmm_score), the only HBM-bound
entry point: GB/s of trajectory bytes read against MEASURED_PEAKS.json's copy
bandwidth (GPU box).   python tools/time_score.py"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2007_09884_b200 import opmm  # noqa: E402

peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
ns = 101
with opmm.opmm_create(0, kernel_timing=True) as h:
    for prec, dt in ((0, torch.float64), (1, torch.float32)):
        for n in (10**6, 4 * 10**6):
            traj = torch.randn((ns, n), dtype=dt, device="cuda")
            rec = torch.randn(ns, dtype=torch.float64, device="cuda")
            err = torch.empty(n, dtype=torch.float64, device="cuda")
            s = torch.cuda.current_stream()
            for _ in range(3):
                opmm.opmm_score(h, traj, n, ns, rec, err, precision=prec, stream=s)
            ms = []
            for _ in range(10):
                opmm.opmm_score(h, traj, n, ns, rec, err, precision=prec, stream=s)
                ms.append(opmm.opmm_last_kernel_ms(h))
            t = float(np.median(ms))
            byts = traj.numel() * traj.element_size() + n * 8
            print(f"{'fp64' if prec == 0 else 'fp32'} n={n:8d}: {t*1e3:8.1f} us  {byts / (t*1e-3) / 1e9:7.0f} GB/s "
                  f"({byts / (t*1e-3) / 1e9 / peak:.2f} of {peak:.0f})", flush=True)
            del traj
