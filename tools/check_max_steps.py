"""Fit / NM at the longest traces (n_steps up to OPMM_MAX_STEPS) -- GPU box."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import workloads as W, oracle
from paper_2007_09884_b200 import opmm
with opmm.opmm_create(0) as h:
    for ns in (8000, 12000, 16384):
        ctl = W.Control(n_steps=ns)
        rec = np.linspace(0, 10, ns + 1)
        for prec in (0, 1):
            try:
                r = opmm.opmm_fit(h, rec, ctl, W.paper_space(), 5000, opmm.fit_options(precision=prec))
                print(ns, prec, "ok", r["best_index"], r["n_finite"])
            except Exception as e:
                print(ns, prec, "ERR", e)
        try:
            res = opmm.opmm_estimate_batch(h, rec[None, :], [W.Control(n_steps=ns, amplitude_deg=10.0)], options=opmm.nm_options(max_iter=5))
            print(ns, "nm ok")
        except Exception as e:
            print(ns, "nm ERR", e)
