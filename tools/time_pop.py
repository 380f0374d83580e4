"""Time the population batch (opmm_fit_batch) leg of bench.py at a chosen size.
    python tools/time_pop.py [saccades] [candidates_per_saccade]"""
import os
import sys
import types

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2007_09884_b200 import opmm  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
with opmm.opmm_create(0) as h:
    r = bench.population_leg(h, opmm, torch, types.SimpleNamespace(pop_saccades=S, pop_candidates=n))
    print(f"population S={S} n={n}: {r['kernel_ms']:.2f} ms  {r['value']:.4g} sims/s  "
          f"mean residual {r['mean_best_residual_deg_per_sample']:.6f}")
