"""Diagnose FP64 GPU-vs-oracle error differences at scale (GPU box).

Prints the candidates with the largest relative |E_gpu - E_orc| together
with their RK4 spectral radius, and for the worst few an 80-bit long-double
RK4 reference (numpy longdouble) to show which side is closer to the exact
RK4 value.   python tests/diag/diag_parity.py [N]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import workloads as W  # noqa: E402
from paper_2007_09884_b200 import opmm  # noqa: E402


def A_b(p, tau_ag, tau_ant, n_ag, n_ant, dt=np.longdouble):
    z = np.zeros(6)
    b = oracle.rhs(p, z, n_ag, n_ant, tau_ag, tau_ant)
    A = np.stack([oracle.rhs(p, np.eye(6)[j], n_ag, n_ant, tau_ag, tau_ant) - b for j in range(6)], 1)
    return A, b


def rho(p):
    r = 0.0
    for ta, tn in ((p[10], p[11]), (p[12], p[13])):
        A, _ = A_b(p, ta, tn, 0, 0)
        ev = np.linalg.eigvals(A) * 1e-3
        r = max(r, np.abs(1 + ev + ev**2 / 2 + ev**3 / 6 + ev**4 / 24).max())
    return r


def longdouble_E(p, rec, ctl):
    """RK4 stages in 80-bit arithmetic on the same D1 system (exact-ish)."""
    L = np.longdouble
    P = [L(x) for x in p]
    Kag, Kant, Lag, Lant, Bag, Bant, Bp, Ncag, Ncant, J = P[:10]
    F = P[14]
    g_ag, g_ant = Kag / (Lag + Kag), Kant / (Lant + Kant)
    G = g_ag * (Ncag + Lag) + g_ant * (Ncant + Lant)
    th_s = (g_ag * F - g_ant * F) / G
    y = np.array([th_s, L(0), (F - (Ncag - Kag) * th_s) / (Lag + Kag),
                  (F + (Ncant - Kant) * th_s) / (Lant + Kant), F, F], dtype=L)
    lv = oracle.step_levels(p, 10.0)
    npulse = int(np.ceil(p[17] / ctl.dt_ms))
    h = L(ctl.dt_ms) / 1000

    def f(y, nag, nant, tag, tant):
        Tag = Kag * (y[2] - y[0])
        Tant = Kant * (y[3] + y[0])
        return np.array([y[1], (Tag - Tant - Bp * y[1]) / J,
                         (y[4] - Ncag * y[0] - Lag * y[2] - Tag) / Bag,
                         (y[5] + Ncant * y[0] - Lant * y[3] - Tant) / Bant,
                         (nag - y[4]) / tag, (nant - y[5]) / tant], dtype=L)
    rel, s, Ap = oracle.relativize(rec, ctl.amplitude_deg)
    acc = L(0)
    for k in range(ctl.n_steps):
        if k < npulse:
            args = (P[15], P[16], P[10] / 1000, P[11] / 1000)
        else:
            args = (L(lv[0]), L(lv[1]), P[12] / 1000, P[13] / 1000)
        k1 = f(y, *args)
        k2 = f(y + h / 2 * k1, *args)
        k3 = f(y + h / 2 * k2, *args)
        k4 = f(y + h * k3, *args)
        y = y + h / 6 * (k1 + 2 * k2 + 2 * k3 + k4)
        acc += abs((y[0] - th_s) - L(rel[k + 1]))
    return float(acc)


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 10**6
    ctl = W.Control()
    rec = oracle.positions(W.truth_opc(), ctl) + W.noise(101)
    sp = W.paper_space()
    err = torch.empty(N, dtype=torch.float64, device="cuda")
    with opmm.opmm_create(0) as h:
        r = opmm.opmm_fit(h, rec, ctl, sp, N, opmm.fit_options(err_out=err))
    E = err.cpu().numpy()
    o = oracle.fit(rec, ctl, sp, 0, N, nthreads=oracle.max_threads(), want_err=True)
    O = o["err"]
    rel, _, _ = oracle.relativize(rec, ctl.amplitude_deg)
    scale = np.abs(rel).sum()
    f = np.isfinite(O) & np.isfinite(E)
    d = np.zeros(N)
    d[f] = np.abs(E[f] - O[f]) / np.maximum(O[f], scale)
    print(f"N={N} argmin gpu {r['best_index']} oracle {o['best_index']}; inf-class mismatches "
          f"{int(np.sum(np.isinf(E) != np.isinf(O)))}")
    for thr in (1e-12, 1e-11, 1e-10, 1e-9, 1e-8):
        print(f"  rel diff > {thr:g}: {int(np.sum(d > thr))}")
    top = np.argsort(-d)[:12]
    for i in top:
        p = oracle.generate(sp, int(i))
        print(f"  i={i:9d} d={d[i]:.3e} E_orc={O[i]:.6e} E_gpu={E[i]:.6e} rho={rho(p):.4f}")
    for i in top[:4]:
        p = oracle.generate(sp, int(i))
        ref = longdouble_E(p, rec, ctl)
        print(f"  i={i}: longdouble E={ref:.12e}  |orc-ref|/ref={abs(O[i]-ref)/ref:.2e}  "
              f"|gpu-ref|/ref={abs(E[i]-ref)/ref:.2e}")


if __name__ == "__main__":
    main()
