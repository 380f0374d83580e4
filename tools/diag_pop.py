"""Population batch: identical results across slice sizes (GPU box).
    python tools/diag_pop.py S n"""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench, workloads as W
from paper_2007_09884_b200 import opmm
S, n = int(sys.argv[1]), int(sys.argv[2])
with opmm.opmm_create(0) as h:
    ctls, recs = bench.population_traces(h, opmm, torch, S, 150)
    recs2 = bench.population_traces(h, opmm, torch, S, 150)[1]
    print("traces deterministic:", np.array_equal(recs, recs2))
    sp = W.paper_space(n_steps=150)
    out = {}
    for t in ("384", "8192", "384"):
        os.environ["OPMM_POP_TILE"] = t
        res = opmm.opmm_fit_batch(h, recs, ctls, sp, n, opmm.fit_options(cpu_check=0))
        out.setdefault(t, []).append([(r["best_index"], r["opt_err"], r["n_finite"]) for r in res])
    a, b, c = out["384"][0], out["8192"][0], out["384"][1]
    print("384 repeat identical:", a == c)
    d = [s for s in range(S) if a[s] != b[s]]
    print("mismatches 384 vs 8192:", len(d), d[:5], [(a[s], b[s]) for s in d[:3]])
