"""Small instances of every kernel for compute-sanitizer (GPU box):
    compute-sanitizer --tool memcheck python tools/sanitize_small.py [section ...]
sections: fit, topk, refill, grid, super, explicit, batch, nm, long (default: all)"""
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

want = set(sys.argv[1:]) or {"fit", "topk", "refill", "grid", "super", "explicit", "batch", "nm", "long"}
rec = np.loadtxt(os.path.join(ROOT, "tests/golden/trace_truth_A10_dt1_n100.txt")) + W.noise(101)
ctl, sp = W.Control(), W.paper_space()
with opmm.opmm_create(0) as h:
    if "fit" in want:
        for n in (1, 33, 1000, 4099):
            for bs in (64, 384):
                for prec in (0, 1):
                    err = torch.zeros(n, dtype=torch.float64, device="cuda")
                    opmm.opmm_fit(h, rec, ctl, sp, n, opmm.fit_options(precision=prec, block_size=bs, err_out=err))
    if "topk" in want:
        for n in (5, 3000):
            opmm.opmm_fit(h, rec, ctl, sp, n, opmm.fit_options(top_k=7))
            opmm.opmm_fit(h, rec, ctl, sp, n, opmm.fit_options(precision=1, certify=1))
    if "refill" in want:
        for n in (1, 31, 2000):
            opmm.opmm_fit(h, rec, ctl, sp, n, opmm.fit_options(kernel_variant=5))
            opmm.opmm_fit(h, rec, ctl, sp, n, opmm.fit_options(kernel_variant=5, precision=1))
    if "grid" in want:
        g = W.g4_space(per_dim=7)
        opmm.opmm_fit(h, rec, ctl, g, g.n_grid(), opmm.fit_options(kernel_variant=1))
        opmm.opmm_fit(h, rec, ctl, g, g.n_grid(), opmm.fit_options(kernel_variant=1, precision=1, certify=1))
    if "super" in want:
        g = W.g4_space(per_dim=9)
        for fl in (0, opmm.FIT_FLAG_SUPER_SMEM):
            opmm.opmm_fit(h, rec, ctl, g, g.n_grid(), opmm.fit_options(kernel_variant=4, flags=fl))
        opmm.opmm_fit(h, rec, ctl, g, g.n_grid(), opmm.fit_options(kernel_variant=4, precision=1))
    if "explicit" in want:
        cand = np.tile(W.truth_opc(), (70, 1)).T.copy()
        opc = torch.as_tensor(cand, device="cuda")
        traj = torch.zeros((101, 70), dtype=torch.float64, device="cuda")
        opmm.opmm_simulate(h, opc, 70, ctl, traj, stream=torch.cuda.current_stream())
        err = torch.zeros(70, dtype=torch.float64, device="cuda")
        opmm.opmm_simulate_score(h, opc, 70, ctl, torch.as_tensor(rec, device="cuda"), err,
                                 stream=torch.cuda.current_stream())
        opmm.opmm_score(h, traj, 70, 101, torch.as_tensor(rec, device="cuda"), err,
                        stream=torch.cuda.current_stream())
        out = torch.zeros((18, 100), dtype=torch.float64, device="cuda")
        opmm.opmm_generate(h, sp, 2**32 - 50, 100, out, stream=torch.cuda.current_stream())
        torch.cuda.synchronize()
    if "batch" in want:
        amp, pw, truths = W.population(5)
        ctls = [W.Control(amplitude_deg=a, pw_default_ms=p) for a, p in zip(amp, pw)]
        opmm.opmm_fit_batch(h, np.tile(rec, (5, 1)), ctls, sp, 300)
        opmm.opmm_fit_batch(h, np.tile(rec, (5, 1)), ctls, sp, 300, opmm.fit_options(precision=1, certify=1))
    if "nm" in want:
        amp, pw, truths = W.population(9)
        ctls = [W.Control(amplitude_deg=a, pw_default_ms=p) for a, p in zip(amp, pw)]
        for sched in (1, 2, 3):
            opmm.opmm_estimate_batch(h, np.tile(rec, (9, 1)), ctls,
                                     options=opmm.nm_options(max_iter=40, schedule=sched))
    if "long" in want:
        cl = W.Control(n_steps=16384)
        rl = truth_trace(opmm, h, cl, noisy=False)
        opmm.opmm_fit(h, rl, cl, W.paper_space(n_steps=16384), 500)
    torch.cuda.synchronize()
print("sanitize_small done", sorted(want))
