"""Nelder-Mead kernel time, LOCKSTEP vs LANE vs GROUP schedule, against the number of
problems (bench population recipe, n_steps = 150, propagator fp64 objective;
GPU box).  Also checks the two schedules return the same runs.
    python tools/time_nm_schedules.py [S ...]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2007_09884_b200 import opmm  # noqa: E402

sizes = [int(a) for a in sys.argv[1:]] or [16, 64, 256, 1024, 4096, 16384]
with opmm.opmm_create(0, kernel_timing=True) as h:
    ctls, recs = bench.population_traces(h, opmm, torch, max(sizes), 150)
    for S in sizes:
        row, runs = [], []
        for sc in (opmm.NM_SCHEDULE_LOCKSTEP, opmm.NM_SCHEDULE_LANE, opmm.NM_SCHEDULE_GROUP):
            opts = opmm.nm_options(cpu_check=0, schedule=sc)
            res = opmm.opmm_estimate_batch(h, recs[:S], ctls[:S], options=opts)
            ms = opmm.opmm_last_kernel_ms(h)
            runs.append(res)
            evals = sum(r["gpu_evals"] for r in res)
            row.append(f"{ms:9.2f} ms {S / (ms * 1e-3):9.0f} sac/s {evals / (ms * 1e-3):9.3g} ev/s")
        same = all(a["f"] == b["f"] == c["f"] and a["iterations"] == b["iterations"] == c["iterations"]
                   for a, b, c in zip(*runs))
        its = np.mean([r["iterations"] for r in runs[1]])
        print(f"S {S:6d} (iters {its:6.0f}) lockstep {row[0]} | lane {row[1]} | group {row[2]} | same {same}",
              flush=True)
