"""Small fits/simulations for compute-sanitizer (GPU box):
    compute-sanitizer --tool memcheck python tools/sanitize_small.py"""
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
with opmm.opmm_create(0) as h:
    for n in (1, 33, 1000, 4099):
        for bs in (64, 128, 256, 384):
            for prec in (0, 1):
                err = torch.zeros(n, dtype=torch.float64, device="cuda")
                r = opmm.opmm_fit(h, rec, ctl, sp, n, opmm.fit_options(precision=prec, block_size=bs,
                                                                        err_out=err))
    cand = np.tile(W.truth_opc(), (70, 1)).T.copy()
    opc = torch.as_tensor(cand, device="cuda")
    traj = torch.zeros((101, 70), dtype=torch.float64, device="cuda")
    opmm.opmm_simulate(h, opc, 70, ctl, traj, stream=torch.cuda.current_stream())
    err = torch.zeros(70, dtype=torch.float64, device="cuda")
    opmm.opmm_simulate_score(h, opc, 70, ctl, torch.as_tensor(rec, device="cuda"), err,
                             stream=torch.cuda.current_stream())
    opmm.opmm_score(h, traj, 70, 101, torch.as_tensor(rec, device="cuda"), err,
                    stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    g = W.g4_space(per_dim=7)
    r = opmm.opmm_fit(h, rec, ctl, g, g.n_grid())
    amp, pw, truths = W.population(5)
    ctls = [W.Control(amplitude_deg=a, pw_default_ms=p) for a, p in zip(amp, pw)]
    opmm.opmm_fit_batch(h, np.tile(rec, (5, 1)), ctls, sp, 300)
print("sanitize_small done")
