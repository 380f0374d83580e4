"""|E32 - E64| against the certification budget 1e-4 max(E, sum|rel|) over the
bench workload's candidates (GPU box): python tools/fp32_error_budget.py [n]"""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_2007_09884_b200 import opmm  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10**6
rec = np.loadtxt(os.path.join(ROOT, "tests/golden/trace_truth_A10_dt1_n100.txt")) + W.noise(101)
srel = np.abs(rec - rec[0]).sum()
with opmm.opmm_create(0) as h:
    E = {}
    for prec in (0, 1):
        e = torch.zeros(n, dtype=torch.float64, device="cuda")
        opmm.opmm_fit(h, rec, W.Control(), W.paper_space(), n, opmm.fit_options(precision=prec, err_out=e, cpu_check=0))
        E[prec] = e.cpu().numpy()
f = np.isfinite(E[0]) & np.isfinite(E[1])
r = np.abs(E[1][f] - E[0][f]) / np.maximum(E[0][f], srel)
print(f"finite {f.sum()}; classification mismatches {(np.isfinite(E[0]) != np.isfinite(E[1])).sum()}; "
      f"max |E32-E64|/max(E64, sum|rel|) = {r.max():.3e} (budget 1e-4); 99.99% {np.quantile(r, 0.9999):.3e}")
# candidates near the best: relative to E64 itself
best = np.argsort(E[0])[:1000]
print(f"1000 best: max |E32-E64|/E64 = {(np.abs(E[1][best]-E[0][best])/E[0][best]).max():.3e}")
