"""Pins for the CPU oracle (-m "not gpu").

Each test fixes the oracle against something other than itself: values the
paper / SPEC print (tests/golden/), closed forms derived by hand from the
statics, textbook identities (RK4 on an LTI system == the polynomial
propagator; convergence to the matrix-exponential solution), invariants
(fixed point, linearity in pulse heights, world-size invariance), published
known-answer vectors (Philox) and brute force on tiny grids.  Pin labels
P1..P12b follow SURVEY.md 8(c).
"""
import math

import numpy as np
import pytest
import scipy.linalg

import oracle
import workloads as W
from conftest import read_golden_kv, read_golden_table

I = W.IDX


def A_and_b(p, n_ag, n_ant, tau_ag, tau_ant):
    """Continuous-time A, b of the (linear) plant, probed column by column from
    the oracle RHS: rhs(y) = A y + b.  Independent of the RK4 code."""
    z = np.zeros(6)
    b = oracle.rhs(p, z, n_ag, n_ant, tau_ag, tau_ant)
    A = np.stack([oracle.rhs(p, np.eye(6)[j], n_ag, n_ant, tau_ag, tau_ant) - b for j in range(6)], 1)
    return A, b


def phase_inputs(p, Aprime):
    lv = oracle.step_levels(p, Aprime)
    pulse = (p[I["N_SAC_AG"]], p[I["N_SAC_ANT"]], p[I["TAU_AC_AG"]], p[I["TAU_AC_ANT"]])
    post = (lv[0], lv[1], p[I["TAU_DE_AG"]], p[I["TAU_DE_ANT"]])
    return pulse, post


# --------------------------------------------------------------------------- P1
def test_p1_table1_defaults_match_paper():
    rows = read_golden_table("table1_defaults.txt")
    assert [r[0] for r in rows] == list(W.PARAM_NAMES)
    for (name, val), d in zip(rows, W.TABLE1_DEFAULTS):
        if name == "PW":
            assert math.isnan(d)
        else:
            assert float(val) == d, name


def test_p1_table2_defaults_match_paper():
    rows = read_golden_table("table2_defaults.txt")
    assert tuple(r[0] for r in rows) == W.TABLE2_NAMES
    assert tuple(float(r[1]) for r in rows) == W.TABLE2_DEFAULTS


# --------------------------------------------------------------------------- P2/P3
def test_p2_symmetric_equilibrium_node_length():
    g = read_golden_kv("spec_worked_examples.txt")
    y = oracle.equilibrium(W.truth_opc(), 14.0, 14.0)
    assert y[0] == 0.0 and y[1] == 0.0
    assert round(y[2], 6) == g["equilibrium_x_m_defaults"]
    assert round(y[3], 6) == g["equilibrium_x_m_defaults"]
    assert y[4] == 14.0 and y[5] == 14.0


def test_p3_pulse_onset_activation_slope_units():
    """df_AG/dt at onset = (55 - 14)/11.7 g/ms: catches ms/s bugs."""
    g = read_golden_kv("spec_worked_examples.txt")
    p = W.truth_opc()
    y = oracle.equilibrium(p, 14.0, 14.0)
    dy = oracle.rhs(p, y, p[I["N_SAC_AG"]], p[I["N_SAC_ANT"]], p[I["TAU_AC_AG"]], p[I["TAU_AC_ANT"]])
    # RHS is per second; SPEC quotes g/ms.
    assert round(dy[4] * 1e-3, 3) == g["onset_dfAG_dt_g_per_ms"]
    assert dy[4] == pytest.approx(41.0 / 11.7e-3, rel=1e-14)
    # equilibrium mechanics do not move at the onset instant
    assert np.all(np.abs(dy[:4]) < 1e-12)


def test_activation_eigenvalues_are_minus_one_over_tau():
    """The f_m rows are first-order lags: eigenvalues -1/tau (s^-1)."""
    p = W.truth_opc()
    A, _ = A_and_b(p, 0, 0, p[I["TAU_AC_AG"]], p[I["TAU_AC_ANT"]])
    ev = np.sort(np.linalg.eigvals(A).real)
    for tau in (11.7e-3, 2.4e-3):
        assert np.min(np.abs(ev + 1.0 / tau)) < 1e-6 / tau
    # defaults: continuous plant is stable (all eigenvalues real and negative)
    assert np.all(ev < 0)


# --------------------------------------------------------------------------- statics
def _random_physical(n, seed=11):
    rng = np.random.default_rng(seed)
    d = W.truth_opc()
    out = []
    for _ in range(n):
        p = d * np.exp(rng.uniform(np.log(0.5), np.log(2.0), size=18))
        p[I["PW"]] = rng.uniform(5, 60)
        out.append(p)
    return out


def test_equilibrium_is_zero_of_rhs_for_any_physical_opc_and_drive():
    """Hand-derived statics: theta_ss = (g_AG n_AG - g_ANT n_ANT)/G
    makes every derivative vanish, for asymmetric muscles too (Q5)."""
    rng = np.random.default_rng(3)
    for p in _random_physical(50):
        n_ag, n_ant = rng.uniform(0.5, 80, size=2)
        y = oracle.equilibrium(p, n_ag, n_ant)
        dy = oracle.rhs(p, y, n_ag, n_ant, 5.0, 3.0)
        scale = np.abs(np.array([1, 1 / p[I["J"]], 1 / p[I["B_AG"]], 1 / p[I["B_ANT"]], 1, 1])) * 100
        assert np.all(np.abs(dy) <= 1e-12 * scale)
        # closed form, derived by hand from D1 with all derivatives zero
        g_ag = p[0] / (p[2] + p[0])
        g_ant = p[1] / (p[3] + p[1])
        G = g_ag * (p[7] + p[2]) + g_ant * (p[8] + p[3])
        assert y[0] == pytest.approx((g_ag * n_ag - g_ant * n_ant) / G, rel=1e-13, abs=1e-13)


# --------------------------------------------------------------------------- P4
def test_p4_fixed_point_500ms_defaults():
    """SPEC.md:119 / :550: zero-pulse simulation stays within 1e-9 deg over 500 ms."""
    p = W.truth_opc()
    p[I["N_SAC_AG"]] = p[I["N_C_FIX"]]
    p[I["N_SAC_ANT"]] = p[I["N_C_FIX"]]
    dth = oracle.simulate(p, 1.0, 500, 0.0, 40.0)
    assert np.max(np.abs(dth)) < 1e-9


def test_p4_fixed_point_any_physical_opc_small_dt():
    for p in _random_physical(20, seed=5):
        p[I["N_SAC_AG"]] = p[I["N_C_FIX"]]
        p[I["N_SAC_ANT"]] = p[I["N_C_FIX"]]
        dth = oracle.simulate(p, 0.0625, 2000, 0.0, 40.0)
        assert np.max(np.abs(dth)) < 1e-9


# --------------------------------------------------------------------------- P5
@pytest.mark.parametrize("Aprime", [10.0, 5.0, 20.0])
def test_p5_steady_state_reaches_target(Aprime):
    """Long run of the RK4 map settles at theta* + A' (step levels solve the
    static balance, D4/Q4; both with the 0.01 g antagonist floor active (10, 20)
    and inactive (5))."""
    p = W.truth_opc()
    dth = oracle.simulate(p, 1.0, 3000, Aprime, 40.0)
    assert dth[-1] == pytest.approx(Aprime, abs=1e-9)
    lv = oracle.step_levels(p, Aprime)
    floor_active = lv[1] == 0.01
    assert floor_active == (Aprime >= 10.0)


def test_p5_steady_state_closed_form_random_opcs():
    """Steady state of the simulated plant == hand-derived closed form, for
    random physical OPCs integrated with a small step."""
    for p in _random_physical(10, seed=9):
        Ap = 8.0
        dth, st = oracle.simulate(p, 0.0625, 40000, Ap, 40.0, states=True)
        lv = oracle.step_levels(p, Ap)
        g_ag = p[0] / (p[2] + p[0])
        g_ant = p[1] / (p[3] + p[1])
        G = g_ag * (p[7] + p[2]) + g_ant * (p[8] + p[3])
        th_ss = (g_ag * lv[0] - g_ant * lv[1]) / G
        th_star = (g_ag - g_ant) * p[14] / G
        assert st[-1, 0] == pytest.approx(th_ss, abs=1e-8)
        assert dth[-1] == pytest.approx(th_ss - th_star, abs=1e-8)
        assert dth[-1] == pytest.approx(Ap, abs=1e-8)
        assert st[-1, 4] == pytest.approx(lv[0], rel=1e-10)


# --------------------------------------------------------------------------- P6
def test_p6_linearity_in_pulse_height_and_monotone_amplitude():
    """The plant is linear in the drive: Delta-theta is affine in N_SAC_AG, so
    the peak amplitude is monotone in pulse height (north_star pin)."""
    p = W.truth_opc()
    trajs = []
    for h in (40.0, 55.0, 70.0):
        q = p.copy()
        q[I["N_SAC_AG"]] = h
        trajs.append(oracle.simulate(q, 1.0, 100, 10.0, 40.0))
    t40, t55, t70 = trajs
    second_diff = t70 - 2 * t55 + t40
    assert np.max(np.abs(second_diff)) <= 1e-12 * np.max(np.abs(t55))
    peaks = [t.max() for t in trajs]
    assert peaks[0] < peaks[1] < peaks[2]
    # derivative with respect to pulse height is positive during the pulse
    assert np.all((t70 - t40)[1:41] > 0)


@pytest.mark.parametrize("name", ["N_SAC_AG", "N_SAC_ANT"])
def test_p6_superposition_identity_both_channels(name):
    """The identity the superposition kernel scores with:
    Delta-theta(a) = b + a u, b = Delta-theta(N_SAC = 0), u = Delta-theta(1) - b,
    for either pulse height, any stable plant, any pulse width -- checked on the
    oracle's own literal RK4 trajectories, plus the L1 error it implies."""
    rng = np.random.default_rng(76)
    ctl = W.Control()
    rec = oracle.positions(W.truth_opc(), ctl) + W.noise(ctl.n_steps + 1)
    rel, _, Ap = oracle.relativize(rec, ctl.amplitude_deg)
    for _ in range(6):
        p = W.truth_opc() * np.exp(rng.uniform(-0.3, 0.3, size=18))
        p[I["PW"]] = float(rng.integers(5, 90))
        def traj(a):
            q = p.copy()
            q[I[name]] = a
            return oracle.simulate(q, ctl.dt_ms, ctl.n_steps, Ap, 40.0)
        b, one = traj(0.0), traj(1.0)
        u = one - b
        for a in (0.37, 12.5, 80.0):
            direct = traj(a)
            sup = b + a * u
            assert np.max(np.abs(sup - direct)) <= 1e-11 * max(np.max(np.abs(direct)), 1.0)
            q = p.copy()
            q[I[name]] = a
            E = oracle.objective(q, rec, ctl)
            assert abs(np.abs(sup - rel).sum() - E) <= 1e-10 * max(E, np.abs(rel).sum())


def test_directionality():
    """N_SAC_AG > N_C_FIX > N_SAC_ANT gives a non-negative saccade."""
    p = W.truth_opc()
    dth = oracle.simulate(p, 1.0, 100, 10.0, 40.0)
    assert np.all(dth >= 0)
    # NOTE: SPEC.md:116 ("J x 10 -> strictly lower peak velocity") does not hold
    # under D1 (the globe is heavily over-damped; a heavier globe responds
    # faster here).  It is recorded as reading Q21 in DESIGN.md, not used as a pin.


def test_first_step_closed_form_taylor():
    """From the fixation equilibrium, theta only moves through the chain
    f -> x -> omega -> theta, so the first RK4 step equals the 4th-order Taylor
    term of the exact solution, derived by hand from Fig. 1 / D1:
      dtheta_1 = h^4/24 * (1/J) * [K_SE_AG/B_AG * (N_SAC_AG - F)/tau_AC_AG
                                   + K_SE_ANT/B_ANT * (F - N_SAC_ANT)/tau_AC_ANT]
    Pins every sign and coupling on the path, the tau units and the RK4 weight."""
    for p in [W.truth_opc()] + _random_physical(20, seed=33):
        F = p[I["N_C_FIX"]]
        for dt in (1.0, 0.5, 0.1):
            h = dt * 1e-3
            expect = h ** 4 / 24 / p[I["J"]] * (
                p[I["K_SE_AG"]] / p[I["B_AG"]] * (p[I["N_SAC_AG"]] - F) / (1e-3 * p[I["TAU_AC_AG"]])
                + p[I["K_SE_ANT"]] / p[I["B_ANT"]] * (F - p[I["N_SAC_ANT"]]) / (1e-3 * p[I["TAU_AC_ANT"]]))
            d1 = oracle.simulate(p, dt, 1, 10.0, 40.0)[1]
            # abs term: rounding of theta_1 - theta* when theta* != 0 (asymmetric muscles)
            assert d1 == pytest.approx(expect, rel=1e-9, abs=64 * 2.0 ** -52 * abs(oracle.equilibrium(p, F, F)[0]))


# --------------------------------------------------------------------------- P7
def _rk4_matrix_form(p, dt_ms, n_steps, Aprime):
    """Textbook identity: classical RK4 on y' = A y + b with constant b is
    y+ = P(hA) y + h Q(hA) b, P(z) = 1+z+z^2/2+z^3/6+z^4/24, Q(z) = 1+z/2+z^2/6+z^3/24."""
    h = dt_ms * 1e-3
    pulse, post = phase_inputs(p, Aprime)
    mats = []
    for ph in (pulse, post):
        A, b = A_and_b(p, *ph)
        Z = h * A
        Id = np.eye(6)
        P = Id + Z + Z @ Z / 2 + Z @ Z @ Z / 6 + Z @ Z @ Z @ Z / 24
        Q = Id + Z / 2 + Z @ Z / 6 + Z @ Z @ Z / 24
        mats.append((P, h * Q @ b))
    npulse = math.ceil(p[I["PW"]] / dt_ms)
    y = oracle.equilibrium(p, p[I["N_C_FIX"]], p[I["N_C_FIX"]])
    out = [y.copy()]
    for k in range(n_steps):
        P, c = mats[0] if k < npulse else mats[1]
        y = P @ y + c
        out.append(y.copy())
    return np.array(out)


def test_p7_rk4_equals_polynomial_propagator():
    cands = [W.truth_opc()] + _random_physical(10, seed=21)
    for p in cands:
        ref = _rk4_matrix_form(p, 1.0, 100, 10.0)
        dth, st = oracle.simulate(p, 1.0, 100, 10.0, 40.0, states=True)
        scale = np.maximum(np.abs(ref).max(axis=0), 1.0)
        assert np.max(np.abs(st - ref) / scale) < 1e-11


# --------------------------------------------------------------------------- P8
def test_p8_rk4_fourth_order_convergence():
    """SPEC.md:120 / :551: halving dt shrinks the error by >= 12 (theory 16)."""
    p = W.truth_opc()
    # steps 1, 1/2, 1/4, 1/8 ms; PW = 40 ms is on every grid so the control
    # discontinuity is sampled exactly.
    res = {}
    for m in (1, 2, 4, 8):
        res[m] = oracle.simulate(p, 1.0 / m, 100 * m, 10.0, 40.0)[::m]
    e1 = np.max(np.abs(res[1] - res[8]))
    e2 = np.max(np.abs(res[2] - res[8]))
    e4 = np.max(np.abs(res[4] - res[8]))
    # Richardson: e(h) ~ C h^4 (1 - 1/8^4 ...); ratio of successive errors
    assert e1 / e2 >= 12
    assert e2 / e4 >= 12


def test_p8_converges_to_matrix_exponential_solution():
    """dt -> 0 approaches the exact zero-order-hold solution e^{tA} (scipy expm,
    a library routine independent of the RK4 code)."""
    p = W.truth_opc()
    pulse, post = phase_inputs(p, 10.0)
    h = 1e-3
    steps = []
    for ph in (pulse, post):
        A, b = A_and_b(p, *ph)
        M = np.zeros((7, 7))
        M[:6, :6] = A * h
        M[:6, 6] = b * h
        steps.append(scipy.linalg.expm(M))
    y = np.append(oracle.equilibrium(p, 14.0, 14.0), 1.0)
    th0 = y[0]
    exact = [0.0]
    for k in range(100):
        y = (steps[0] if k < 40 else steps[1]) @ y
        exact.append(y[0] - th0)
    exact = np.array(exact)
    fine = oracle.simulate(p, 1.0 / 64, 6400, 10.0, 40.0)[::64]
    coarse = oracle.simulate(p, 1.0, 100, 10.0, 40.0)
    assert np.max(np.abs(fine - exact)) < 1e-8
    assert np.max(np.abs(coarse - exact)) > 1e-6  # RK4 at 1 ms is not exact
    assert np.max(np.abs(coarse - exact)) < 1e-2


# --------------------------------------------------------------------------- substeps (Q25)
def _expm_zoh(p, Aprime, dt_ms, n_steps):
    """Exact zero-order-hold solution at the samples (scipy expm of the
    augmented [A b; 0 0] per control phase), control switching at the sample
    boundary n_pulse = ceil(PW/dt) -- independent of the RK4 code."""
    pulse, post = phase_inputs(p, Aprime)
    h = 1e-3 * dt_ms
    steps = []
    for ph in (pulse, post):
        A, b = A_and_b(p, *ph)
        M = np.zeros((7, 7))
        M[:6, :6] = A * h
        M[:6, 6] = b * h
        steps.append(scipy.linalg.expm(M))
    npulse = math.ceil(p[I["PW"]] / dt_ms)
    y = np.append(oracle.equilibrium(p, p[I["N_C_FIX"]], p[I["N_C_FIX"]]), 1.0)
    th0 = y[0]
    out = [0.0]
    for k in range(n_steps):
        y = (steps[0] if k < npulse else steps[1]) @ y
        out.append(y[0] - th0)
    return np.array(out)


def test_substeps_is_the_fine_grid_subsampled():
    """Reading Q25: s substeps per sample with the control held over the sample
    interval is, when PW is a whole number of samples, exactly the plain RK4 on
    the fine grid dt/s (n_pulse = s * ceil(PW/dt)) read every s-th sample."""
    for p in [W.truth_opc()] + _random_physical(4, seed=31):
        p = p.copy()
        p[I["PW"]] = float(round(p[I["PW"]]))
        base = oracle.simulate(p, 1.0, 100, 10.0, 40.0)
        assert np.array_equal(oracle.simulate(p, 1.0, 100, 10.0, 40.0, substeps=1), base)
        for m in (2, 3, 5):
            sub = oracle.simulate(p, 1.0, 100, 10.0, 40.0, substeps=m)
            fine = oracle.simulate(p, 1.0 / m, 100 * m, 10.0, 40.0)[::m]
            scale = max(np.abs(fine).max(), 1.0)
            assert np.max(np.abs(sub - fine)) <= 1e-12 * scale, m


def test_substeps_fourth_order_convergence_to_expm():
    """Error against the exact ZOH solution shrinks ~16x per doubling of the
    substeps (classical RK4), >= 12 required."""
    p = W.truth_opc()
    exact = _expm_zoh(p, 10.0, 1.0, 100)
    err = [np.max(np.abs(oracle.simulate(p, 1.0, 100, 10.0, 40.0, substeps=m) - exact))
           for m in (1, 2, 4)]
    assert err[0] / err[1] >= 12 and err[1] / err[2] >= 12, err


def test_substeps_stabilise_a_stiff_candidate():
    """A stiff globe (B_P/J = 1.4e5 1/s: h*rate = 140 at 1 ms, far outside
    RK4's stability interval [-2.79, 0]) diverges at h = dt and converges to the
    exact ZOH solution with 64 substeps (h*rate = 2.2)."""
    p = W.truth_opc()
    p[I["B_P"]] *= 10.0
    p[I["J"]] *= 0.1
    rec = oracle.positions(W.truth_opc(), W.Control())
    assert oracle.objective(p, rec, W.Control()) == math.inf
    sub = oracle.simulate(p, 1.0, 100, 10.0, 40.0, substeps=64)
    exact = _expm_zoh(p, 10.0, 1.0, 100)
    assert np.all(np.isfinite(sub))
    assert np.max(np.abs(sub - exact)) < 1e-6 * max(np.abs(exact).max(), 1.0)
    e = oracle.objective(p, rec, W.Control(substeps=64))
    assert math.isfinite(e) and e == oracle.score(sub, oracle.relativize(rec, 10.0)[0])


# --------------------------------------------------------------------------- score
def test_score_spec_examples_and_cap():
    g = read_golden_kv("spec_worked_examples.txt")
    a = np.linspace(0, 10, 50)
    assert oracle.score(a, a, 0) == g["objective_identical"]
    assert oracle.score(a + 1.0, a, 0) == g["objective_offset1_50samples"]
    assert oracle.score(a + 1.0, a, 1) == 1.0  # RMS of a unit offset
    assert oracle.score(a + 3.0, a, 1) == 3.0
    big = a.copy()
    big[3] = 1e21
    assert oracle.score(big, a, 0) == math.inf          # Q10 cap
    nan = a.copy()
    nan[5] = math.nan
    assert oracle.score(nan, a, 0) == math.inf          # NaN -> +inf


def test_penalty_spec_example():
    g = read_golden_kv("spec_worked_examples.txt")
    p = W.truth_opc()
    p[I["K_SE_AG"]] = -1.0
    assert oracle.physical_penalty(p) >= g["penalty_floor"]
    assert oracle.physical_penalty(p) == 1e10 * 2.0
    rec = np.zeros(101)
    assert oracle.objective(p, rec, W.Control()) == 2e10
    assert oracle.physical_penalty(W.truth_opc()) == 0.0
    q = W.truth_opc()
    q[I["J"]] = 0.0
    assert oracle.physical_penalty(q) == 1e10


def test_penalty_g_clause_no_static_balance():
    """Reading Q13's G > 0 clause: with N_C + K_LT = 0 on both muscles every
    bound holds (those four are >= 0, not > 0) but the static gain G =
    g_AG (N_C_AG + K_LT_AG) + g_ANT (N_C_ANT + K_LT_ANT) is 0, so the
    fixation balance G theta = g_AG n_AG - g_ANT n_ANT has no unique solution
    (hand-derived statics): penalty 1e10 (1 + 0).  Any
    positive restoring term on either muscle restores G > 0."""
    q = W.truth_opc()
    for name in ("N_C_AG", "K_LT_AG", "N_C_ANT", "K_LT_ANT"):
        q[I[name]] = 0.0
    assert oracle.physical_penalty(q) == 1e10
    assert oracle.objective(q, np.zeros(101), W.Control()) == 1e10
    for name in ("N_C_AG", "K_LT_AG", "N_C_ANT", "K_LT_ANT"):
        r = q.copy()
        r[I[name]] = 1e-3
        assert oracle.physical_penalty(r) == 0.0, name


def test_objective_batch_equals_fit_errors():
    """orc_objective_batch on supplied candidates (the generator's own values)
    returns exactly fit()'s per-candidate errors, for any thread count."""
    ctl = W.Control()
    rec = oracle.positions(W.truth_opc(), ctl) + W.noise(101)
    sp = W.paper_space()
    N = 1500
    full = oracle.fit(rec, ctl, sp, 7, 7 + N, want_err=True)
    soa = oracle.generate_batch(sp, 7, N).T
    for nt in (1, 4):
        E = oracle.objective_batch(soa, rec, ctl, nthreads=nt)
        assert np.array_equal(E, full["err"])


def test_pulse_window_discretisation():
    g = read_golden_kv("spec_worked_examples.txt")
    assert 46.0 - 6.0 == g["pw_placeholder_46ms"]
    assert oracle.n_pulse(40.0, 1.0) == 40
    assert oracle.n_pulse(39.21, 1.0) == 40
    assert oracle.n_pulse(40.0001, 1.0) == 41
    # NaN PW uses the per-saccade default
    p = W.truth_opc()
    q = p.copy()
    q[I["PW"]] = math.nan
    assert np.array_equal(oracle.simulate(q, 1.0, 100, 10.0, 40.0), oracle.simulate(p, 1.0, 100, 10.0, 40.0))
    assert len(oracle.simulate(p, 1.0, 46, 10.0, 40.0)) == int(g["simulate_46ms_samples"])


def test_relativize_mirrors_negative_saccades():
    rec = np.array([3.0, 2.0, 0.0, -5.0])
    rel, s, Ap = oracle.relativize(rec, math.nan)
    assert s == -1.0 and Ap == 8.0
    assert rel.tolist() == [0.0, 1.0, 3.0, 8.0]
    rel2, s2, Ap2 = oracle.relativize(rec, 4.0)
    assert s2 == 1.0 and Ap2 == 4.0 and rel2.tolist() == [0.0, -1.0, -3.0, -8.0]


# --------------------------------------------------------------------------- P9
def test_p9_zero_error_on_own_output_and_mirroring():
    ctl = W.Control()
    t = W.truth_opc()
    rec = oracle.positions(t, ctl)
    rel, s, Ap = oracle.relativize(rec, ctl.amplitude_deg)
    e = oracle.objective(t, rec, ctl)
    assert e <= 1e-9 * np.abs(rel).sum()
    # negative saccade from 3 deg: mirrored estimate gives the same error
    ctl2 = W.Control(amplitude_deg=-10.0, theta0_deg=3.0)
    rec2 = oracle.positions(t, ctl2)
    assert rec2[0] == 3.0 and rec2[-1] < 3.0
    assert oracle.objective(t, rec2, ctl2) <= 1e-9 * np.abs(rel).sum()


def test_p9_planted_grid_argmin_is_truth():
    ctl = W.Control()
    rec = oracle.positions(W.truth_opc(), ctl)
    sp = W.g4_space(per_dim=9)   # 9^4 grid, TRUTH at (4, 4, 4, PW=40 -> digit 39?)
    # per_dim = 9 puts PW levels 1..9 ms; use a PW grid that contains 40 instead
    d = W.truth_opc()
    sp = W.grid_space({
        "K_SE_AG": (d[0] * 1.01 ** -4, d[0] * 1.01 ** 4, 9, True),
        "B_AG": (d[4] * 1.01 ** -4, d[4] * 1.01 ** 4, 9, True),
        "N_SAC_AG": (d[15] * 1.01 ** -4, d[15] * 1.01 ** 4, 9, True),
        "PW": (36.0, 44.0, 9, False),
    })
    n = sp.n_grid()
    r = oracle.fit(rec, ctl, sp, 0, n, nthreads=4)
    planted = 4 + 9 * 4 + 81 * 4 + 729 * 4
    assert r["best_index"] == planted
    assert r["best_err"] < 1e-9 * 650
    assert r["n_finite"] == n


# --------------------------------------------------------------------------- P10
def test_p10_bruteforce_argmin_tiny_grid():
    """3^4 grid over {K_SE_AG, B_AG, N_SAC_AG, PW} (SPEC.md:553 set), noisy trace:
    the oracle fit == an independent Python brute-force min over objectives."""
    ctl = W.Control()
    rec = oracle.positions(W.truth_opc(), ctl) + W.noise(101)
    d = W.truth_opc()
    sp = W.grid_space({
        "K_SE_AG": (d[0] * 0.8, d[0] * 1.2, 3, False),
        "B_AG": (d[4] * 0.8, d[4] * 1.2, 3, False),
        "N_SAC_AG": (d[15] * 0.8, d[15] * 1.2, 3, False),
        "PW": (30.0, 50.0, 3, False),
    })
    n = sp.n_grid()
    errs = []
    for i in range(n):
        c = oracle.generate(sp, i)
        # independent mixed-radix check (dimension 0 fastest)
        dig = [i % 3, (i // 3) % 3, (i // 9) % 3, (i // 27) % 3]
        assert c[0] == pytest.approx(d[0] * (0.8 + 0.2 * dig[0]), rel=1e-15)
        assert c[17] == 30.0 + 10.0 * dig[3]
        errs.append(oracle.objective(c, rec, ctl))
    errs = np.array(errs)
    best = int(np.argmin(errs))
    r = oracle.fit(rec, ctl, sp, 0, n, nthreads=3, want_err=True)
    assert r["best_index"] == best
    assert r["best_err"] == errs[best]
    assert np.array_equal(r["err"], errs)


# --------------------------------------------------------------------------- P11
def test_p11_philox_known_answers():
    rows = read_golden_table("philox4x32_10_kat.txt")
    assert len(rows) == 3
    for r in rows:
        v = [int(x, 16) for x in r]
        out = oracle.philox4x32_10(v[0:4], v[4:6])
        assert out.tolist() == v[6:10]


def test_generator_bounds_and_distribution():
    sp = W.paper_space()
    c = oracle.generate_batch(sp, 0, 4000)
    assert np.all(c >= sp.lo) and np.all(c <= sp.hi)
    # log-uniform dims: log(v/lo)/log(hi/lo) ~ U(0,1); PW linear ~ U(1, 100)
    u = np.log(c[:, :17] / sp.lo[:17]) / np.log(sp.hi[:17] / sp.lo[:17])
    assert np.all(np.abs(u.mean(axis=0) - 0.5) < 0.03)
    assert np.all(np.abs(u.var(axis=0) - 1 / 12) < 0.01)
    assert abs(c[:, 17].mean() - 50.5) < 2.0
    # independent re-derivation of one candidate from the Philox words
    i = 123456789012
    words = np.concatenate([oracle.philox4x32_10([i & 0xffffffff, i >> 32, 0, j],
                                                 [9884, 0]) for j in range(5)])
    uu = (words[:18].astype(np.float64) + 0.5) / 2.0 ** 32
    cand = oracle.generate(sp, i)
    assert cand[17] == pytest.approx(1.0 + uu[17] * 99.0, rel=1e-15)
    assert cand[3] == pytest.approx(0.12 * 100.0 ** uu[3], rel=1e-14)
    # saccade field changes the stream
    assert not np.array_equal(oracle.generate(sp, 5, saccade=1), oracle.generate(sp, 5, saccade=0))


# --------------------------------------------------------------------------- P12 / P12b
def test_p12_shard_invariance():
    ctl = W.Control()
    rec = oracle.positions(W.truth_opc(), ctl) + W.noise(101)
    sp = W.paper_space()
    N = 3000
    full = oracle.fit(rec, ctl, sp, 0, N, nthreads=1, want_err=True)
    for R in (2, 4, 8):
        parts = []
        for r in range(R):
            b, e = N * r // R, N * (r + 1) // R
            parts.append(oracle.fit(rec, ctl, sp, b, e, nthreads=2))
        best = min((p["best_err"], p["best_index"]) for p in parts if p["best_index"] >= 0)
        assert best == (full["best_err"], full["best_index"])
        assert sum(p["n_finite"] for p in parts) == full["n_finite"]
    for nt in (3, 8):
        r = oracle.fit(rec, ctl, sp, 0, N, nthreads=nt)
        assert (r["best_err"], r["best_index"]) == (full["best_err"], full["best_index"])
    # the error vector itself is index-deterministic
    sub = oracle.fit(rec, ctl, sp, 1000, 1100, want_err=True)
    assert np.array_equal(sub["err"], full["err"][1000:1100])


def test_p12b_exact_ties_resolve_to_lowest_index():
    """PW enters only through ceil(PW/dt): PW in {39.21, 39.6, 40.0} gives
    bit-identical errors; the lowest index must win (Q12)."""
    ctl = W.Control()
    rec = oracle.positions(W.truth_opc(), ctl) + W.noise(101)
    d = W.truth_opc()
    sp = W.grid_space({
        "N_SAC_AG": (d[15] * 0.99, d[15] * 1.01, 3, False),
        "PW": (39.21, 40.0, 3, False),   # 39.21, 39.605, 40.0 -> n_pulse 40
    })
    r = oracle.fit(rec, ctl, sp, 0, 9, want_err=True)
    e = r["err"].reshape(3, 3)   # [PW digit, N_SAC digit]
    assert np.all(e[0] == e[1]) and np.all(e[1] == e[2])
    assert r["best_index"] == int(np.argmin(e[0]))
    # shard so the tied copies land in different shards: lowest index still wins
    parts = [oracle.fit(rec, ctl, sp, b, b + 3) for b in (6, 3, 0)]
    best = min((p["best_err"], p["best_index"]) for p in parts)
    assert best[1] == r["best_index"]


def test_all_diverged_gives_no_finite():
    ctl = W.Control()
    rec = oracle.positions(W.truth_opc(), ctl)
    d = W.truth_opc()
    # J tiny and B tiny: RK4 at 1 ms blows up for every candidate
    d[I["J"]] = 1e-9
    d[I["B_AG"]] = 1e-6
    d[I["B_ANT"]] = 1e-6
    sp = W.grid_space({"PW": (10.0, 20.0, 3, False)}, base=d)
    r = oracle.fit(rec, ctl, sp, 0, 3, want_err=True)
    assert r["best_index"] == -1 and r["n_finite"] == 0
    assert np.all(np.isinf(r["err"]))


# --------------------------------------------------------------------------- regression (scratch)
def test_survey_scratch_regression_values():
    """Values computed during the survey by a separate throwaway script under
    the same readings (SURVEY 8(c) 'Scratch-derived regression values').
    Regression only -- not a paper pin."""
    p = W.truth_opc()
    d = oracle.simulate(p, 1.0, 100, 10.0, 40.0)
    ref = [8.039284810329e-04, 0.6438167818780, 2.508462368148, 6.717097214111, 8.175197819521, 9.682190619240]
    assert np.allclose(d[[1, 10, 20, 40, 50, 100]], ref, rtol=1e-11, atol=1e-15)
    assert abs(d).sum() == pytest.approx(650.9431611563706, rel=1e-13)
    d5 = oracle.simulate(p, 1.0, 100, 5.0, 40.0)
    assert d5[50] == pytest.approx(7.779986704990, rel=1e-11)
    assert d5[100] == pytest.approx(5.954196963665, rel=1e-11)
    assert oracle.step_levels(p, 5.0).tolist() == pytest.approx([23.25, 4.75], rel=1e-14)


def test_trace_fixture_is_oracle_output():
    """tests/golden/trace_truth_A10_dt1_n100.txt (bench/smoke input) was written
    by scripts/make_traces.py from this oracle; it must still match."""
    import os
    from conftest import GOLDEN
    rec = np.loadtxt(os.path.join(GOLDEN, "trace_truth_A10_dt1_n100.txt"), comments="#")
    ref = oracle.positions(W.truth_opc(), W.Control())
    assert np.array_equal(rec, ref)


def test_referee_longdouble_agrees_with_oracle_on_stable_candidates():
    """The extended-precision referee evaluates the same definition: on
    RK4-stable candidates it agrees with the fp64 oracle to ~1e-13."""
    from oracle import referee
    ctl = W.Control()
    rec = oracle.positions(W.truth_opc(), ctl) + W.noise(101)
    sp = W.paper_space()
    n_checked = 0
    for i in range(60):
        p = oracle.generate(sp, i)
        if referee.rk4_spectral_radius(p, ctl.dt_ms) >= 1.0:
            continue
        e64 = oracle.objective(p, rec, ctl)
        eld = referee.objective_longdouble(p, rec, ctl)
        assert abs(e64 - eld) <= 1e-13 * max(e64, 1.0)
        n_checked += 1
    assert n_checked >= 10
    # TRUTH on its own clean output: both ~0
    rec0 = oracle.positions(W.truth_opc(), ctl)
    assert referee.objective_longdouble(W.truth_opc(), rec0, ctl) < 1e-10


def test_referee_fp64_spread_brackets_the_oracle():
    """fp64_spread (long double with the state rounded stochastically at
    fp64's unit roundoff each step) measures what fp64 can resolve: on a
    stable candidate it is at the 1e-16 level (and the fp64 oracle sits inside
    a small multiple of it); on the RK4-unstable 10^8-tail candidates of
    DESIGN.md section 6 it is orders of magnitude larger, and the plain fp64
    oracle's own deviation from the exact value is of the same order."""
    from oracle import referee
    ctl = W.Control()
    rec = oracle.positions(W.truth_opc(), ctl) + W.noise(101)
    rel, _, _ = oracle.relativize(rec, ctl.amplitude_deg)
    scale = np.abs(rel).sum()
    p = W.truth_opc()
    s_stable = referee.fp64_spread(p, rec, ctl)
    assert s_stable < 1e-14
    sp = W.paper_space()
    for i in (31760573, 79953948):   # rho ~ 1.33 / 1.78, errors ~1e5 / 1e14
        q = oracle.generate(sp, i)
        assert referee.rk4_spectral_radius(q, ctl.dt_ms) > 1.0
        s = referee.fp64_spread(q, rec, ctl)
        ref = referee.objective_longdouble(q, rec, ctl)
        o = abs(oracle.objective(q, rec, ctl) - ref) / max(ref, scale)
        assert s > 1e3 * s_stable and s > 1e-9
        assert o <= 3 * s, (i, o, s)


# --------------------------------------------------------------------------- 9-parameter model
def test_nine_param_expansion_d7_and_table2():
    """Table 2 inside the 18-vector per SPEC D7: shared
    K_SE / K_LT, canonical pulse 55 / 0.5 g of width "duration - 6 ms" (PW
    NaN), Table 1 time constants (reading Q23).  The Table 2 defaults expand
    to exactly the Table 1 defaults, so the 9-parameter default scores the
    TRUTH trace like the 18-parameter default."""
    p = np.ones(18)
    for name, d in zip(W.NINE_SLOTS, W.TABLE2_DEFAULTS):
        p[I[name]] = d
    e = oracle.expand_9param(p)
    assert e[I["K_SE_ANT"]] == e[I["K_SE_AG"]] == 2.5
    assert e[I["K_LT_ANT"]] == e[I["K_LT_AG"]] == 1.2
    assert (e[I["N_SAC_AG"]], e[I["N_SAC_ANT"]]) == (55.0, 0.5)
    assert math.isnan(e[I["PW"]])
    d1 = np.array(W.TABLE1_DEFAULTS)
    assert np.array_equal(e[:17], d1[:17])
    ctl = W.Control()
    rec = oracle.positions(W.truth_opc(), ctl)
    assert oracle.objective(e, rec, ctl) == oracle.objective(W.truth_opc(), rec, ctl)


def test_nine_param_generator_draws_only_free_slots():
    sp = W.paper_space_9()
    c = oracle.generate_batch(sp, 0, 500)
    for name in W.NINE_SLOTS:
        i = I[name]
        assert np.all((c[:, i] >= sp.lo[i]) & (c[:, i] <= sp.hi[i]))
        assert np.unique(c[:, i]).size > 400
    assert np.array_equal(c[:, I["K_SE_ANT"]], c[:, I["K_SE_AG"]])
    assert np.array_equal(c[:, I["K_LT_ANT"]], c[:, I["K_LT_AG"]])
    assert np.all(c[:, I["TAU_AC_AG"]] == 11.7) and np.all(np.isnan(c[:, I["PW"]]))
    # the 9 free slots are the same Philox words the 18-parameter generator uses
    sp18 = W.paper_space()
    sp18.lo[:], sp18.hi[:], sp18.log_scale[:] = sp.lo, sp.hi, sp.log_scale
    c18 = oracle.generate_batch(sp18, 0, 50)
    for name in W.NINE_SLOTS:
        assert np.array_equal(c18[:, I[name]], c[:50, I[name]])
