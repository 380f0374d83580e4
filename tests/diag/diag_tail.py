"""The fp64 tail of a 10^8 random S_paper fit (configs[3]): every candidate
whose GPU error differs from the oracle's by more than 1e-10 relative, with
its RK4 spectral radius and both sides' distance to the 80-bit referee.

    python tests/diag/diag_tail.py [n] > gpurun_out/tail.txt
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
import workloads as W  # noqa: E402
from oracle import referee  # noqa: E402
from paper_2007_09884_b200 import opmm  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**8
ctl = W.Control()
rec = oracle.positions(W.truth_opc(), ctl) + W.noise(ctl.n_steps + 1)
sp = W.paper_space()
with opmm.opmm_create(0) as h:
    err = torch.empty(n, dtype=torch.float64, device="cuda")
    r = opmm.opmm_fit(h, rec, ctl, sp, n, opmm.fit_options(err_out=err))
    torch.cuda.synchronize()
    E = err.cpu().numpy()
o = oracle.fit(rec, ctl, sp, 0, n, nthreads=oracle.max_threads(), want_err=True)
O = o["err"]
rel, _, _ = oracle.relativize(rec, ctl.amplitude_deg)
scale = np.abs(rel).sum()
f = np.isfinite(O)
print(f"n {n} best gpu {r['best_index']} orc {o['best_index']} n_finite gpu {r['n_finite']} orc {o['n_finite']}")
print(f"inf classification equal: {np.array_equal(np.isinf(E), np.isinf(O))}")
d = np.zeros(n)
d[f] = np.abs(E[f] - O[f]) / np.maximum(O[f], scale)
for t in (1e-12, 1e-11, 1e-10, 1e-9, 1e-8):
    print(f"  rel diff > {t:.0e}: {int(np.sum(d > t))}")
idx = np.flatnonzero(d > 1e-10)
print(f"{'index':>10} {'E_orc':>14} {'rho':>9} {'gpu-vs-orc':>10} {'gpu-vs-ref':>10} {'orc-vs-ref':>10}")
rows = []
for i in idx:
    p = oracle.generate(sp, int(i))
    rho = referee.rk4_spectral_radius(p, ctl.dt_ms)
    ref = referee.objective_longdouble(p, rec, ctl)
    s = max(ref, scale)
    rows.append((int(i), O[i], rho, d[i], abs(E[i] - ref) / s, abs(O[i] - ref) / s))
rows.sort(key=lambda x: -x[4])
for row in rows:
    print(f"{row[0]:>10} {row[1]:>14.6g} {row[2]:>9.4f} {row[3]:>10.3e} {row[4]:>10.3e} {row[5]:>10.3e}")
g = np.array([x[4] for x in rows]) if rows else np.zeros(0)
oo = np.array([x[5] for x in rows]) if rows else np.zeros(0)
print(f"flagged {len(rows)}; all rho > 1: {all(x[2] > 1 for x in rows)}; "
      f"gpu-vs-ref > 1e-9: {int(np.sum(g > 1e-9))}; orc-vs-ref > 1e-9: {int(np.sum(oo > 1e-9))}; "
      f"gpu closer to ref than orc: {int(np.sum(g <= oo))}/{len(rows)}; max gpu/orc ratio "
      f"{(g / np.maximum(oo, 1e-300)).max() if len(rows) else 0:.3f}")
