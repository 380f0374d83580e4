"""Group-schedule NM kernel time at a few sizes (GPU box).   python tools/time_nm_group.py [S ...]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2007_09884_b200 import opmm  # noqa: E402

sizes = [int(a) for a in sys.argv[1:]] or [16, 4096]
with opmm.opmm_create(0, kernel_timing=True) as h:
    ctls, recs = bench.population_traces(h, opmm, torch, max(sizes), 150)
    for S in sizes:
        opts = opmm.nm_options(cpu_check=0, schedule=opmm.NM_SCHEDULE_GROUP)
        res = opmm.opmm_estimate_batch(h, recs[:S], ctls[:S], options=opts)
        ms = opmm.opmm_last_kernel_ms(h)
        print(f"group S {S:6d}: {ms:8.2f} ms  {S / (ms * 1e-3):9.0f} sac/s  max iters "
              f"{max(r['iterations'] for r in res)}", flush=True)
