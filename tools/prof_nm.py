"""Run the bench NM leg at a small size (for ncu: -k regex:nm_kernel).
    python tools/prof_nm.py [saccades]"""
import os
import sys
import types

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2007_09884_b200 import opmm  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 512
with opmm.opmm_create(0) as h:
    r = bench.nm_leg(h, opmm, torch, types.SimpleNamespace(nm_saccades=S))
    print(f"NM S={S}: kernel {r['kernel_ms']:.1f} ms, {r['value']:.0f} saccades/s, "
          f"{r['evaluations_per_s']:.3g} evals/s, iters {r['mean_iterations']:.0f}")
