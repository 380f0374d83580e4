"""Extended-precision referee for FP64 disagreements -- TEST INFRASTRUCTURE ONLY.

The fp64 oracle and the fp64 GPU path evaluate the same RK4 recurrence with
different (both legitimate) rounding orders.  For RK4-unstable candidates
(spectral radius of the step map > 1) the trajectory grows geometrically and
both fp64 results carry rounding error amplified by the growth; the oracle's
own error can exceed the 1e-9 parity budget there (reading Q22).
When the two disagree beyond the budget, this module decides which side is
wrong by re-evaluating the SAME definition (SPEC D1 plant, classical RK4,
ZOH pulse-step control, L1/RMS score -- identical to oracle/opmm_oracle.c)
in 80-bit long double (numpy.longdouble, 64-bit significand).

It imports nothing from the product and shares no code with it; the
candidate OPC values it consumes come from the oracle's generator.
"""
from __future__ import annotations

import numpy as np

import oracle

L = np.longdouble


def rk4_spectral_radius(p, dt_ms: float, substeps: int = 1) -> float:
    """max over both control phases of |P(h lambda)|^s, h = dt/s, for the
    eigenvalues of the continuous plant matrix (probed from the oracle RHS):
    the spectral radius of the sample-to-sample RK4 map (s substeps, Q25)."""
    s = max(int(substeps or 1), 1)
    z = np.zeros(6)
    r = 0.0
    for tau_ag, tau_ant in ((p[10], p[11]), (p[12], p[13])):
        b = oracle.rhs(p, z, 0, 0, tau_ag, tau_ant)
        A = np.stack([oracle.rhs(p, np.eye(6)[j], 0, 0, tau_ag, tau_ant) - b for j in range(6)], 1)
        ev = np.linalg.eigvals(A) * dt_ms * 1e-3 / s
        r = max(r, float(np.abs(1 + ev + ev ** 2 / 2 + ev ** 3 / 6 + ev ** 4 / 24).max()) ** s)
    return r


def objective_longdouble(p, rec, ctl, metric: int = 0, perturb=None) -> float:
    """E of one OPC, every operation in long double (same steps as the oracle).
    perturb (a numpy Generator): after every RK4 step each state component is
    multiplied by (1 + r u), r ~ U[-1, 1], u = 2^-53 -- the effect of rounding
    the state to fp64 once per step, on top of the long-double arithmetic
    (stochastic-rounding estimate of what fp64 can resolve; fp64_spread)."""
    P = [L(x) for x in p]
    Kag, Kant, Lag, Lant, Bag, Bant, Bp, Ncag, Ncant, J = P[:10]
    F = P[14]
    pw = P[17] if not np.isnan(p[17]) else L(ctl.pw_default_ms)
    rel, s, Ap = oracle.relativize(rec, ctl.amplitude_deg)
    g_ag, g_ant = Kag / (Lag + Kag), Kant / (Lant + Kant)
    G = g_ag * (Ncag + Lag) + g_ant * (Ncant + Lant)
    th_s = (g_ag * F - g_ant * F) / G
    y = np.array([th_s, L(0), (F - (Ncag - Kag) * th_s) / (Lag + Kag),
                  (F + (Ncant - Kant) * th_s) / (Lant + Kant), F, F], dtype=L)
    delta = G * L(Ap) / (g_ag + g_ant)
    n_ag, n_ant = F + delta, F - delta
    if n_ant < L(0.01):
        n_ant = L(0.01)
        n_ag = (G * (th_s + L(Ap)) + L(0.01) * g_ant) / g_ag
    n_pulse = int(np.ceil(float(pw) / ctl.dt_ms))   # the IEEE-double decision, as in the oracle
    nsub = max(int(getattr(ctl, "substeps", 0) or 0), 1)   # Q25
    h = L(ctl.dt_ms) / L(1000) / L(nsub)

    def f(y, nag, nant, tag, tant):
        Tag = Kag * (y[2] - y[0])
        Tant = Kant * (y[3] + y[0])
        return np.array([y[1], (Tag - Tant - Bp * y[1]) / J,
                         (y[4] - Ncag * y[0] - Lag * y[2] - Tag) / Bag,
                         (y[5] + Ncant * y[0] - Lant * y[3] - Tant) / Bant,
                         (nag - y[4]) / tag, (nant - y[5]) / tant], dtype=L)

    acc = L(0)
    for k in range(ctl.n_steps):
        if k < n_pulse:
            args = (P[15], P[16], P[10] / 1000, P[11] / 1000)
        else:
            args = (n_ag, n_ant, P[12] / 1000, P[13] / 1000)
        for _ in range(nsub):
            k1 = f(y, *args)
            k2 = f(y + h / 2 * k1, *args)
            k3 = f(y + h / 2 * k2, *args)
            k4 = f(y + h * k3, *args)
            y = y + h / 6 * (k1 + 2 * k2 + 2 * k3 + k4)
            if perturb is not None:
                y = y * (L(1) + L(2.0 ** -53) * np.array(perturb.uniform(-1.0, 1.0, 6), dtype=L))
        d = (y[0] - th_s) - L(rel[k + 1])
        acc += abs(d) if metric == 0 else d * d
    if not acc < L(1e20):
        return float("inf")
    return float(acc) if metric == 0 else float(np.sqrt(acc / L(ctl.n_steps + 1)))


def fp64_spread(p, rec, ctl, metric: int = 0, samples: int = 8, seed: int = 0) -> float:
    """What an fp64 evaluation of this candidate's error can resolve: the
    largest |E_k - E| over `samples` long-double evaluations whose state is
    perturbed at fp64's unit roundoff after every step (objective_longdouble
    with perturb), relative to max(E, s) with s the trace's error scale
    (sum |rel| for L1, RMS(rel) for RMS).  For RK4-unstable candidates (spectral
    radius > 1) the step map amplifies these perturbations geometrically; this
    is the measured fp64 resolution that DESIGN.md reading Q22 uses as the
    parity bar where it exceeds 1e-9."""
    rel, _, _ = oracle.relativize(rec, ctl.amplitude_deg)
    scale = float(np.abs(rel).sum()) if metric == 0 else float(np.sqrt(np.mean(rel ** 2)))
    ref = objective_longdouble(p, rec, ctl, metric)
    if not np.isfinite(ref):
        return float("inf")
    g = np.random.default_rng(seed)
    d = [abs(objective_longdouble(p, rec, ctl, metric, perturb=g) - ref) for _ in range(samples)]
    return max(d) / max(ref, scale)
