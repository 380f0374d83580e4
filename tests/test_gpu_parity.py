"""GPU parity: libopmm (CUDA, through the C ABI) vs the CPU oracle (-m gpu).

Same seeded inputs on both sides (workloads/), compared element by element.
Tolerances (north_star):
  FP64 trajectories  |d_gpu - d_orc| <= 1e-9 * max(max_k |d_orc|, 1 deg)
  FP64 errors        |E_gpu - E_orc| <= 1e-9 * max(E_orc, sum |rel|); +inf / penalty exact
  FP64 argmin        identical index
  FP32 trajectories  <= 1e-3 deg per sample on RK4-stable candidates
  FP32 errors        <= 1e-4 * max(E_orc, sum |rel|); finite/+inf classification exact
  FP32 best fit      E64(winner32) <= (1 + 1e-4) E64(winner64) + 1e-4 sum |rel|
  generator          linear dims bit-exact, log dims <= 2 ulp (device exp vs glibc exp)
"""
import math

import numpy as np
import pytest

import oracle
import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

I = W.IDX
ULP = 2.0 ** -52


@pytest.fixture(scope="module")
def opmm():
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: the -m gpu suite must run on a B200")
    from paper_2007_09884_b200 import build
    build.build()
    from paper_2007_09884_b200 import opmm as m
    return m


@pytest.fixture(scope="module")
def h(opmm):
    with opmm.opmm_create(0) as handle:
        yield handle


def dev(a, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device="cuda")


def trace(ctl, noisy=True):
    rec = oracle.positions(W.truth_opc(), ctl)
    return rec + W.noise(ctl.n_steps + 1) if noisy else rec


def soa(cands):
    """[n, 18] -> device SoA [18, n]."""
    return dev(np.ascontiguousarray(np.asarray(cands).T))


def candidate_set(n_paper=3000, seed=1):
    sp = W.paper_space()
    c = [W.truth_opc()]
    c += list(oracle.generate_batch(sp, 0, n_paper))
    rng = np.random.default_rng(seed)
    d = W.truth_opc()
    for _ in range(300):
        p = d * np.exp(rng.uniform(np.log(0.5), np.log(2.0), size=18))
        p[I["PW"]] = rng.uniform(1, 100)
        c.append(p)
    return np.array(c)


def rk4_stable(p, ctl):
    """Oracle-side decision: spectral radius of the RK4 map < 1
    in both control phases (non-physical candidates are not stable)."""
    if oracle.physical_penalty(p) != 0.0:
        return False
    z = np.zeros(6)
    rad = 0.0
    for tau_ag, tau_ant in ((p[10], p[11]), (p[12], p[13])):
        b = oracle.rhs(p, z, 0, 0, tau_ag, tau_ant)
        A = np.stack([oracle.rhs(p, np.eye(6)[j], 0, 0, tau_ag, tau_ant) - b for j in range(6)], 1)
        ev = np.linalg.eigvals(A) * ctl.dt_ms * 1e-3
        P = 1 + ev + ev ** 2 / 2 + ev ** 3 / 6 + ev ** 4 / 24
        rad = max(rad, np.abs(P).max())
    return rad < 1.0


def assert_fp64_errors(E, O, cand_of, rec, ctl, scale, metric=0, stats=None):
    """FP64 error parity (reading Q22): |E_gpu - E_orc| <=
    1e-9 max(E_orc, scale) for every candidate.  A candidate outside that
    budget must be RK4-unstable (rho > 1), and against the 80-bit referee the
    GPU value must be within 1e-9 of the exact RK4 value (the oracle's own
    fp64 rounding is what exceeded it) -- or, where the candidate's step map
    amplifies rounding so much that fp64 cannot resolve 1e-9 at all, within
    twice the measured fp64 resolution of that candidate (referee.fp64_spread:
    the largest deviation of 8 long-double runs with the state rounded
    stochastically at fp64's unit roundoff every step; the factor 2 covers the
    sampling of that maximum -- the GPU's own rounding is one more draw).  Returns the number of refereed candidates; `stats`
    (a dict) receives the counts."""
    from oracle import referee
    assert np.array_equal(np.isinf(E), np.isinf(O))
    f = np.isfinite(O)
    d = np.zeros_like(O)
    d[f] = np.abs(E[f] - O[f]) / np.maximum(O[f], scale)
    refereed = beyond = 0
    for i in np.flatnonzero(d > 1e-9):
        p = cand_of(int(i))
        rho = referee.rk4_spectral_radius(p, ctl.dt_ms, getattr(ctl, "substeps", 1))
        assert rho > 1.0, (int(i), d[i], rho)
        ref = referee.objective_longdouble(p, rec, ctl, metric)
        g = abs(E[i] - ref) / max(ref, scale)
        refereed += 1
        if g <= 1e-9:
            continue
        spread = referee.fp64_spread(p, rec, ctl, metric)
        assert g <= 2.0 * spread, (int(i), E[i], O[i], ref, g, spread)
        beyond += 1
    if stats is not None:
        stats.update(refereed=refereed, beyond_1e9_within_fp64_spread=beyond,
                     above_1e10=int(np.sum(d > 1e-10)), max_rel=float(d.max()) if d.size else 0.0)
    return refereed


def oracle_dtheta(cands, ctl):
    out = []
    for p in cands:
        try:
            out.append(oracle.simulate(p, ctl.dt_ms, ctl.n_steps, abs(ctl.amplitude_deg), ctl.pw_default_ms,
                                       substeps=max(int(ctl.substeps or 0), 1)))
        except ValueError:
            out.append(None)
    return out


# --------------------------------------------------------------------------- generator
def test_generate_random_matches_oracle(opmm, h):
    sp = W.paper_space()
    n = 8192
    out = torch.zeros((18, n), dtype=torch.float64, device="cuda")
    begin = 10**9 + 12345
    opmm.opmm_generate(h, sp, begin, n, out, saccade=7, stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    g = out.cpu().numpy().T
    o = np.array([oracle.generate(sp, begin + i, saccade=7) for i in range(n)])
    lin = sp.log_scale == 0
    assert np.array_equal(g[:, lin], o[:, lin])
    rel = np.abs(g[:, ~lin] - o[:, ~lin]) / np.abs(o[:, ~lin])
    assert rel.max() <= 2 * ULP, rel.max()


def test_generate_philox_words_match_oracle_kat_pinned(opmm, h):
    """With lo = 0, hi = 2^32 (linear) the generator returns w + 0.5 exactly,
    exposing the raw device Philox words; they must equal the oracle's
    (KAT-pinned) Philox -- including the all-zero KAT vector."""
    sp = W.SearchSpace(0, 0, np.zeros(18), np.full(18, 2.0 ** 32), np.zeros(18, np.uint8),
                       np.ones(18, np.int32))
    n = 1024
    out = torch.zeros((18, n), dtype=torch.float64, device="cuda")
    opmm.opmm_generate(h, sp, 0, n, out, stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    words = out.cpu().numpy() - 0.5
    assert np.all(words == np.floor(words))
    assert [int(x) for x in words[:4, 0]] == [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]
    for i in (1, 77, 1023):
        for j in range(4):
            ref = oracle.philox4x32_10([i, 0, 0, j], [0, 0])
            got = [int(words[4 * j + r, i]) for r in range(4) if 4 * j + r < 18]
            assert got == ref.tolist()[:len(got)]


@pytest.mark.parametrize("case", ["libm_dim", "tiny_span", "neg_zero_fixed", "linear_only"])
def test_generate_generic_paths_match_oracle(opmm, h, case):
    """Random spaces outside the branch-free fast path (a log dimension whose
    exp argument reaches 8 -> libm exp; a span whose 2^-32 scaling would be
    subnormal -> literal u * span; a fixed -0.0) and an all-linear space
    (fast path) against the oracle: linear and fixed dimensions bit-exact,
    log dimensions within 2 ulp."""
    sp = W.paper_space()
    lo, hi, lg = sp.lo.copy(), sp.hi.copy(), sp.log_scale.copy()
    if case == "libm_dim":
        hi[I["B_P"]] = lo[I["B_P"]] * 1e6            # log(hi/lo) = 13.8 >= 8
    elif case == "tiny_span":
        lo[I["N_C_FIX"]], hi[I["N_C_FIX"]], lg[I["N_C_FIX"]] = 1e-300, 1.5e-300, 0
    elif case == "neg_zero_fixed":
        lo[I["N_C_ANT"]] = hi[I["N_C_ANT"]] = -0.0
        lg[I["N_C_ANT"]] = 0
    else:
        lg[:] = 0
    sp = W.SearchSpace(0, 77, lo, hi, lg, np.ones(18, np.int32))
    n = 2048
    out = torch.zeros((18, n), dtype=torch.float64, device="cuda")
    opmm.opmm_generate(h, sp, 5000, n, out, saccade=3, stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    g = out.cpu().numpy().T
    o = np.array([oracle.generate(sp, 5000 + i, saccade=3) for i in range(n)])
    lin = (lg == 0)
    assert np.array_equal(g[:, lin].view(np.int64), o[:, lin].view(np.int64))
    if (~lin).any():
        rel = np.abs(g[:, ~lin] - o[:, ~lin]) / np.abs(o[:, ~lin])
        assert rel.max() <= 2 * ULP, rel.max()


def test_generate_grid_matches_oracle(opmm, h):
    sp = W.g4_space(per_dim=12)
    n = sp.n_grid()
    out = torch.zeros((18, n), dtype=torch.float64, device="cuda")
    opmm.opmm_generate(h, sp, 0, n, out, stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    g = out.cpu().numpy().T
    o = np.array([oracle.generate(sp, i) for i in range(n)])
    assert np.array_equal(g[:, 17], o[:, 17])
    assert np.max(np.abs(g - o) / np.abs(o)) <= 2 * ULP


# --------------------------------------------------------------------------- simulate
@pytest.mark.parametrize("integrator", [0, 1])
@pytest.mark.parametrize("amp,theta0", [(10.0, 0.0), (-7.0, 3.0)])
def test_simulate_fp64_trajectories(opmm, h, integrator, amp, theta0):
    ctl = W.Control(amplitude_deg=amp, theta0_deg=theta0)
    cands = candidate_set()
    bad = W.truth_opc()
    bad[I["K_SE_AG"]] = -1.0
    nanpw = W.truth_opc()
    nanpw[I["PW"]] = math.nan
    cands = np.vstack([cands, bad, nanpw])
    n = len(cands)
    traj = torch.full((ctl.n_steps + 1, n), -1.0, dtype=torch.float64, device="cuda")
    status = torch.zeros(n, dtype=torch.uint8, device="cuda")
    opmm.opmm_simulate(h, soa(cands), n, ctl, traj, precision=opmm.FP64, integrator=integrator,
                       status=status, stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    T = traj.cpu().numpy()
    S = status.cpu().numpy()
    s = -1.0 if amp < 0 else 1.0
    refs = oracle_dtheta(cands, ctl)
    worst = 0.0
    n_unstable_checked = 0
    for i, ref in enumerate(refs):
        if ref is None:
            assert S[i] == 1 and np.all(np.isnan(T[:, i]))
            continue
        finite = np.all(np.isfinite(ref)) and np.abs(ref).sum() < 1e20
        if not finite:
            assert S[i] == 2, i
            continue
        assert S[i] == 0, i
        d = (T[:, i] - theta0) * s
        err = np.max(np.abs(d - ref)) / max(np.max(np.abs(ref)), 1.0)
        worst = max(worst, err)
        assert err <= 1e-9, (i, err)
        n_unstable_checked += 0 if np.max(np.abs(ref)) < 1e3 else 1
    assert T[0, 0] == theta0
    print(f"max rel trajectory diff {worst:.3e}; large-amplitude finite candidates {n_unstable_checked}")


@pytest.mark.parametrize("n_steps", [99, 100])
def test_simulate_pulse_width_edges(opmm, h, n_steps):
    """Pulse ends of both parities and at the edges of the window:
    n_pulse = ceil(PW/dt) in {1, 2, 3, n-1, n, n+1, beyond} (the loop's
    two-step blocks align each lane to n_pulse mod 2)."""
    ctl = W.Control(n_steps=n_steps)
    pws = [0.3, 1.0, 1.5, 2.0, 3.0, n_steps - 1.0, n_steps - 0.5, float(n_steps), n_steps + 0.5,
           n_steps + 1.0, 250.0, math.nan]
    base = W.truth_opc()
    cands = []
    for pw in pws:
        for f in (1.0, 0.7):
            p = base.copy()
            p[I["PW"]] = pw
            p[I["N_SAC_AG"]] *= f
            cands.append(p)
    cands = np.array(cands)
    n = len(cands)
    for integrator in (0, 1):
        for prec, tol in ((opmm.FP64, 1e-9), (opmm.FP32, 1e-3)):
            dt = torch.float64 if prec == opmm.FP64 else torch.float32
            traj = torch.zeros((n_steps + 1, n), dtype=dt, device="cuda")
            opmm.opmm_simulate(h, soa(cands), n, ctl, traj, precision=prec, integrator=integrator,
                               stream=torch.cuda.current_stream())
            torch.cuda.synchronize()
            T = traj.cpu().numpy().astype(np.float64)
            for i, p in enumerate(cands):
                ref = oracle.simulate(p, ctl.dt_ms, n_steps, 10.0, ctl.pw_default_ms)
                scale = 1.0 if prec == opmm.FP32 else max(np.max(np.abs(ref)), 1.0)
                assert np.max(np.abs(T[:, i] - ref)) <= tol * scale, (pws[i // 2], integrator, prec)


def test_simulate_fp32_trajectories_rk4_stable(opmm, h):
    ctl = W.Control()
    cands = candidate_set(n_paper=1500)
    n = len(cands)
    traj = torch.zeros((ctl.n_steps + 1, n), dtype=torch.float32, device="cuda")
    opmm.opmm_simulate(h, soa(cands), n, ctl, traj, precision=opmm.FP32,
                       stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    T = traj.cpu().numpy().astype(np.float64)
    refs = oracle_dtheta(cands, ctl)
    checked = 0
    worst = 0.0
    for i, ref in enumerate(refs):
        if ref is None or not rk4_stable(cands[i], ctl):
            continue
        checked += 1
        e = np.max(np.abs(T[:, i] - ref))
        worst = max(worst, e)
        assert e <= 1e-3, (i, e)
    assert checked > 500
    print(f"fp32: {checked} RK4-stable candidates, max |diff| {worst:.3e} deg")


# --------------------------------------------------------------------------- scores
@pytest.mark.parametrize("precision", [0, 1])
@pytest.mark.parametrize("metric", [0, 1])
def test_simulate_score_parity(opmm, h, precision, metric):
    ctl = W.Control()
    rec = trace(ctl)
    rel, s, Ap = oracle.relativize(rec, ctl.amplitude_deg)
    scale = np.abs(rel).sum() if metric == 0 else np.sqrt(np.mean(rel ** 2))
    cands = candidate_set(n_paper=2000)
    bad = W.truth_opc()
    bad[I["J"]] = 0.0
    cands = np.vstack([cands, bad])
    n = len(cands)
    err = torch.zeros(n, dtype=torch.float64, device="cuda")
    opmm.opmm_simulate_score(h, soa(cands), n, ctl, dev(rec), err, precision=precision, metric=metric,
                             stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    E = err.cpu().numpy()
    O = np.array([oracle.objective(p, rec, ctl, metric) for p in cands])
    assert np.array_equal(np.isinf(E), np.isinf(O)), np.flatnonzero(np.isinf(E) != np.isinf(O))
    assert E[-1] == O[-1] == 1e10
    if precision == 0:
        assert_fp64_errors(E, O, lambda i: cands[i], rec, ctl, scale, metric)
        return
    f = np.isfinite(O)
    tol = 1e-4 * np.maximum(O[f], scale)
    if precision == 1:
        # FP32 scope: RK4-stable candidates (SURVEY 8(c) parity tolerances)
        stable = np.array([rk4_stable(p, ctl) for p in cands[f]])
        bad_i = np.flatnonzero((np.abs(E[f] - O[f]) > tol) & stable)
    else:
        bad_i = np.flatnonzero(np.abs(E[f] - O[f]) > tol)
    assert bad_i.size == 0, (bad_i[:5], E[f][bad_i[:5]], O[f][bad_i[:5]])


@pytest.mark.parametrize("precision", [0, 1])
def test_score_stored_trajectories(opmm, h, precision):
    """opmm_score (HBM-bound) on oracle trajectories vs the oracle score."""
    ctl = W.Control()
    rec = trace(ctl)
    cands = candidate_set(n_paper=500)
    trajs = []
    for p in cands:
        trajs.append(oracle.positions(p, ctl))
    T = np.array(trajs).T.copy()                         # time-major [n_samples, n]
    n = T.shape[1]
    dt = torch.float64 if precision == 0 else torch.float32
    err = torch.zeros(n, dtype=torch.float64, device="cuda")
    Td = dev(T, dt)
    opmm.opmm_score(h, Td, n, ctl.n_steps + 1, dev(rec), err, precision=precision,
                    stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    E = err.cpu().numpy()
    Tq = Td.cpu().numpy().astype(np.float64)
    for i in range(n):
        d = Tq[:, i] - rec
        with np.errstate(all="ignore"):
            ref = np.abs(d).sum()
        if not (ref < 1e20):
            assert np.isinf(E[i])
        else:
            assert abs(E[i] - ref) <= 1e-12 * max(ref, 1.0), i


# --------------------------------------------------------------------------- fit
def _fit(opmm, h, rec, ctl, sp, n, **kw):
    err = torch.full((n,), -1.0, dtype=torch.float64, device="cuda") if n else None
    opts = opmm.fit_options(err_out=err, **kw)
    r = opmm.opmm_fit(h, rec, ctl, sp, n, opts)
    torch.cuda.synchronize()
    return r, (err.cpu().numpy() if n else None)


@pytest.mark.parametrize("integrator", [0, 1])
@pytest.mark.parametrize("metric", [0, 1])
def test_fit_config1_all_candidates(opmm, h, integrator, metric):
    """Config 1: 10 deg saccade, 1 kHz, 100 ms, 1,000 random candidates."""
    ctl = W.Control()
    rec = trace(ctl)
    sp = W.paper_space()
    n = 1000
    r, E = _fit(opmm, h, rec, ctl, sp, n, integrator=integrator, metric=metric)
    o = oracle.fit(rec, ctl, sp, 0, n, metric=metric, want_err=True)
    O = o["err"]
    rel, _, _ = oracle.relativize(rec, ctl.amplitude_deg)
    scale = np.abs(rel).sum() if metric == 0 else np.sqrt(np.mean(rel ** 2))
    assert_fp64_errors(E, O, lambda i: oracle.generate(sp, i), rec, ctl, scale, metric)
    assert r["best_index"] == o["best_index"]
    assert r["n_finite"] == o["n_finite"] and r["n_evaluated"] == n
    assert abs(r["opt_err"] - o["best_err"]) <= 1e-9 * max(o["best_err"], scale)
    assert abs(r["cpu_check"] - r["opt_err"]) <= 1e-9 * max(r["opt_err"], 1.0)
    assert np.max(np.abs(r["opc"] - o["opc"]) / np.abs(o["opc"])) <= 2 * ULP


def test_fit_config2_full_1e6_fp64(opmm, h):
    """Config 2 at full size in the launch configuration bench.py times
    (default options): all 10^6 errors and the argmin vs the oracle."""
    ctl = W.Control()
    rec = trace(ctl)
    sp = W.paper_space()
    n = 10**6
    r, E = _fit(opmm, h, rec, ctl, sp, n)
    o = oracle.fit(rec, ctl, sp, 0, n, nthreads=oracle.max_threads(), want_err=True)
    O = o["err"]
    rel, _, _ = oracle.relativize(rec, ctl.amplitude_deg)
    scale = np.abs(rel).sum()
    f = np.isfinite(O)
    d = np.abs(E[f] - O[f]) / np.maximum(O[f], scale)
    refereed = assert_fp64_errors(E, O, lambda i: oracle.generate(sp, i), rec, ctl, scale)
    print(f"1e6: n_finite {o['n_finite']}, max rel err diff {d.max():.3e}, "
          f"{int(np.sum(d > 1e-10))} above 1e-10, {refereed} refereed (rho > 1, GPU within 1e-9 of 80-bit)")
    assert r["best_index"] == o["best_index"] and r["n_finite"] == o["n_finite"]
    # the bench's fp32 leg at the same size: certified, and its fp64-re-scored
    # winner is the oracle's (north_star: best-fit error within 1e-4 of fp64)
    c32 = opmm.opmm_fit(h, rec, ctl, sp, n, opmm.fit_options(precision=opmm.FP32, certify=1))
    assert c32["certified"] == 1 and c32["best_index"] == o["best_index"]
    assert abs(c32["opt_err"] - o["best_err"]) <= 1e-9 * o["best_err"]


def test_fit_fp32_best_fit_certified_by_fp64_oracle(opmm, h):
    ctl = W.Control()
    rec = trace(ctl)
    sp = W.paper_space()
    n = 200000
    r32, E32 = _fit(opmm, h, rec, ctl, sp, n, precision=opmm.FP32)
    r64, E64 = _fit(opmm, h, rec, ctl, sp, n, precision=opmm.FP64)
    rel, _, _ = oracle.relativize(rec, ctl.amplitude_deg)
    scale = np.abs(rel).sum()
    e32 = oracle.objective(oracle.generate(sp, r32["best_index"]), rec, ctl)
    e64 = oracle.objective(oracle.generate(sp, r64["best_index"]), rec, ctl)
    assert e32 <= (1 + 1e-4) * e64 + 1e-4 * scale
    assert abs(r32["opt_err"] - e32) <= 1e-4 * max(e32, scale)
    # classification finite / +inf identical to fp64 everywhere
    assert np.array_equal(np.isinf(E32), np.isinf(E64))


def test_fit_planted_grid_g4_full_1e8(opmm, h):
    """G4: 100^4 grid over {K_SE_AG, B_AG, N_SAC_AG, PW}; TRUTH is a node.
    Oracle-exact argmin at 10^8 (the oracle checks the winner and samples)."""
    ctl = W.Control()
    rec = trace(ctl, noisy=False)
    sp = W.g4_space(100)
    n = sp.n_grid()
    assert n == 10**8
    err = torch.empty(n, dtype=torch.float64, device="cuda")
    r = opmm.opmm_fit(h, rec, ctl, sp, n, opmm.fit_options(err_out=err))
    planted = W.g4_planted_index()
    assert r["best_index"] == planted
    rel, _, _ = oracle.relativize(rec, ctl.amplitude_deg)
    assert r["opt_err"] <= 1e-9 * np.abs(rel).sum()
    o = oracle.fit(rec, ctl, sp, planted, planted + 1, want_err=True)
    assert abs(r["opt_err"] - o["err"][0]) <= 1e-12 * np.abs(rel).sum()
    rng = np.random.default_rng(4)
    idx = np.sort(rng.choice(n, 2000, replace=False))
    E = err[torch.as_tensor(idx, device="cuda")].cpu().numpy()
    O = np.array([oracle.objective(oracle.generate(sp, int(i)), rec, ctl) for i in idx])
    assert_fp64_errors(E, O, lambda j: oracle.generate(sp, int(idx[j])), rec, ctl, np.abs(rel).sum())
    f = np.isfinite(O)
    assert np.all(O[f] > r["opt_err"])


def test_fit_exact_ties_lowest_index(opmm, h):
    ctl = W.Control()
    rec = trace(ctl)
    d = W.truth_opc()
    sp = W.grid_space({"N_SAC_AG": (d[15] * 0.99, d[15] * 1.01, 3, False),
                       "PW": (39.21, 40.0, 3, False)})
    o = oracle.fit(rec, ctl, sp, 0, 9)
    for bs, gb in ((64, 0), (384, 0), (64, 1)):
        r, E = _fit(opmm, h, rec, ctl, sp, 9, block_size=bs, grid_blocks=gb)
        assert r["best_index"] == o["best_index"]
        e = E.reshape(3, 3)
        assert np.all(e[0] == e[1]) and np.all(e[1] == e[2])


def test_fit_launch_config_invariance(opmm, h):
    ctl = W.Control()
    rec = trace(ctl)
    sp = W.paper_space()
    n = 50001
    ref, Eref = _fit(opmm, h, rec, ctl, sp, n)
    with pytest.raises(opmm.OpmmError) as ei:
        _fit(opmm, h, rec, ctl, sp, n, block_size=512)
    assert ei.value.status == opmm.ERR_INVALID_ARG
    for bs, gb in ((128, 0), (256, 0), (384, 1), (256, 7), (64, 3)):
        r, E = _fit(opmm, h, rec, ctl, sp, n, block_size=bs, grid_blocks=gb)
        assert (r["best_index"], r["opt_err"], r["n_finite"]) == \
               (ref["best_index"], ref["opt_err"], ref["n_finite"])
        assert np.array_equal(E, Eref, equal_nan=True)


@pytest.mark.parametrize("precision", [0, 1])
@pytest.mark.parametrize("variant", [2, 3, 5])
def test_fit_kernel_variants_identical(opmm, h, precision, variant):
    """fit2 (two interleaved candidates per thread), fit3 (warp-specialised
    producer/consumer) and lane refill (5: diverged lanes stop at CAP and take
    new candidates) give bit-identical per-candidate errors and argmin to the
    default one-candidate-per-thread kernel (ragged N, several rounds)."""
    ctl = W.Control()
    rec = trace(ctl)
    sp = W.paper_space()
    n = 300001
    r1, E1 = _fit(opmm, h, rec, ctl, sp, n, precision=precision, kernel_variant=1)
    r2, E2 = _fit(opmm, h, rec, ctl, sp, n, precision=precision, kernel_variant=variant)
    assert (r1["best_index"], r1["opt_err"], r1["n_finite"]) == (r2["best_index"], r2["opt_err"], r2["n_finite"])
    assert np.array_equal(E1, E2)
    with pytest.raises(opmm.OpmmError) as ei:   # variants 2/3 need the propagator
        _fit(opmm, h, rec, ctl, sp, 10, kernel_variant=variant, integrator=opmm.INTEG_RK4_STAGES)
    assert ei.value.status == opmm.ERR_UNSUPPORTED


@pytest.mark.parametrize("metric", [0, 1])
def test_fit_refill_edges(opmm, h, metric):
    """Lane refill (kernel_variant 5): bit-identical to variant 1
    on short and odd traces (n = 1, 2, 3, 7: last-block and odd-start paths),
    pulses of one step and pulses ending past the trace, ragged and tiny counts, forced
    one-block grids (every lane refilled many times) and the population batch;
    and element-wise against the oracle on the bench trace."""
    for n_steps in (1, 2, 3, 7, 100):
        ctl = W.Control(n_steps=n_steps)
        rec = trace(ctl)
        sp = W.paper_space(n_steps=n_steps)
        sp.lo[17], sp.hi[17] = 0.01, 2.0 * n_steps + 3.0   # PW from one step to past the trace
        for n, gb in ((1, 0), (31, 0), (33, 1), (5000, 0), (20011, 1), (20011, 3)):
            r1, E1 = _fit(opmm, h, rec, ctl, sp, n, metric=metric, kernel_variant=1, grid_blocks=gb)
            r5, E5 = _fit(opmm, h, rec, ctl, sp, n, metric=metric, kernel_variant=5, grid_blocks=gb)
            assert (r1["best_index"], r1["opt_err"], r1["n_finite"]) == \
                   (r5["best_index"], r5["opt_err"], r5["n_finite"]), (n_steps, n, gb)
            assert np.array_equal(E1, E5), (n_steps, n, gb)
    ctl = W.Control()
    rec = trace(ctl)
    sp = W.paper_space()
    r5, E5 = _fit(opmm, h, rec, ctl, sp, 3000, metric=metric, kernel_variant=5)
    o = oracle.fit(rec, ctl, sp, 0, 3000, metric=metric, want_err=True)
    rel, _, _ = oracle.relativize(rec, ctl.amplitude_deg)
    scale = np.abs(rel).sum() if metric == 0 else np.sqrt(np.mean(rel ** 2))
    assert_fp64_errors(E5, o["err"], lambda i: oracle.generate(sp, i), rec, ctl, scale, metric)
    assert r5["best_index"] == o["best_index"]
    assert np.isinf(E5).sum() > 1000   # the S_paper mix: many lanes stop early
    # population: gridDim.y = saccades, one block-sized slice per block
    S = 6
    amp, pw, truths = W.population(S)
    ctls = [W.Control(n_steps=150, amplitude_deg=amp[k], pw_default_ms=pw[k]) for k in range(S)]
    recs = np.array([oracle.positions(truths[k], ctls[k]) + W.noise(151, seed=7 + k) for k in range(S)])
    spp = W.paper_space(n_steps=150)
    b1 = opmm.opmm_fit_batch(h, recs, ctls, spp, 4001, opmm.fit_options(metric=metric, kernel_variant=1))
    b5 = opmm.opmm_fit_batch(h, recs, ctls, spp, 4001, opmm.fit_options(metric=metric, kernel_variant=5))
    for k in range(S):
        assert (b1[k]["best_index"], b1[k]["opt_err"], b1[k]["n_finite"]) == \
               (b5[k]["best_index"], b5[k]["opt_err"], b5[k]["n_finite"]), k
    with pytest.raises(opmm.OpmmError) as ei:
        _fit(opmm, h, rec, ctl, sp, 100, kernel_variant=5, top_k=4)
    assert ei.value.status == opmm.ERR_UNSUPPORTED
    host_err = np.zeros(100)
    with pytest.raises(opmm.OpmmError) as ei:   # err_out must be device memory
        opmm.opmm_fit(h, rec, ctl, sp, 100, opmm.fit_options(err_out=host_err))
    assert ei.value.status == opmm.ERR_INVALID_ARG
    import ctypes
    out_host = np.zeros(ctypes.sizeof(opmm.FitResult), dtype=np.uint8)
    with pytest.raises(opmm.OpmmError) as ei:   # the async entry point takes device buffers
        opmm.opmm_fit_async(h, dev(rec), ctl, sp, 100, out_host)
    assert ei.value.status == opmm.ERR_INVALID_ARG


def _grid_spaces():
    d = W.truth_opc()
    mixed = W.grid_space({"K_SE_AG": (d[I["K_SE_AG"]] * 0.5, d[I["K_SE_AG"]] * 2.0, 7, True),
                          "J": (d[I["J"]] * 1e-3, d[I["J"]] * 1e3, 5, True),       # x up to 13.8: libm exp
                          "B_ANT": (d[I["B_ANT"]] * 0.5, d[I["B_ANT"]] * 1.5, 3, False),
                          "PW": (5.0, 80.0, 16, False)})
    lo, hi = np.ones(18), np.ones(18)
    logs, lv = np.zeros(18, dtype=np.uint8), np.ones(18, dtype=np.int32)
    for name, dv in zip(W.NINE_SLOTS, W.TABLE2_DEFAULTS):
        lo[I[name]] = hi[I[name]] = dv
    for name, n in (("K_SE_AG", 9), ("B_AG", 6), ("J", 5), ("N_C_FIX", 4)):
        dv = W.TABLE2_DEFAULTS[W.NINE_SLOTS.index(name)]
        lo[I[name]], hi[I[name]], logs[I[name]], lv[I[name]] = 0.3 * dv, 3.0 * dv, 1, n
    nine = W.SearchSpace(1, 0, lo, hi, logs, lv, model=1)
    return [("g4", W.g4_space(32)), ("mixed", mixed), ("nine", nine)]


@pytest.mark.parametrize("precision", [0, 1])
@pytest.mark.parametrize("metric", [0, 1])
def test_grid_level_tables_bit_identical(opmm, h, precision, metric):
    """Grid fits take each OPC from per-dimension level tables in shared
    memory (fit_kernel<GT>): mixed-radix digits + one load per grid
    dimension.  Every error is bit-identical to the generic grid generator's
    (OPMM_FIT_FLAG_NO_GRID_TABLES) on G4 at 32^4 nodes, a grid with
    linear, table-exp and libm-exp (argument >= 8) dimensions, and a
    9-parameter-model grid (D7 expansion after the lookup); and the 9-param
    grid against the oracle."""
    ctl = W.Control()
    rec = trace(ctl)
    for name, sp in _grid_spaces():
        n = sp.n_grid()
        r1, E1 = _fit(opmm, h, rec, ctl, sp, n, precision=precision, metric=metric, kernel_variant=1)
        r0, E0 = _fit(opmm, h, rec, ctl, sp, n, precision=precision, metric=metric, kernel_variant=1,
                      flags=opmm.FIT_FLAG_NO_GRID_TABLES)
        assert (r1["best_index"], r1["opt_err"], r1["n_finite"]) == \
               (r0["best_index"], r0["opt_err"], r0["n_finite"]), name
        assert np.array_equal(E1, E0, equal_nan=True), name
        if name == "nine" and precision == 0:
            o = oracle.fit(rec, ctl, sp, 0, n, metric=metric, want_err=True)
            rel, _, _ = oracle.relativize(rec, ctl.amplitude_deg)
            scale = np.abs(rel).sum() if metric == 0 else np.sqrt(np.mean(rel ** 2))
            assert_fp64_errors(E1, o["err"], lambda i: oracle.generate(sp, i), rec, ctl, scale, metric)
            assert r1["best_index"] == o["best_index"]


def test_grid_level_tables_beyond_2_32_and_population(opmm, h):
    """The table path's 64-bit digit step (indices >= 2^32), a 16000-step
    trace with 1900 table entries, and the population batch: same results as
    the generic grid generator."""
    ctl = W.Control()
    rec = trace(ctl)
    d = W.truth_opc()
    dims = {k: (d[I[k]] * 0.8, d[I[k]] * 1.25, 100, True) for k in ("K_SE_AG", "B_AG", "N_SAC_AG", "B_ANT")}
    dims["PW"] = (1.0, 85.0, 43, False)
    sp = W.grid_space(dims)
    n = sp.n_grid()   # 4.3e9 > 2^32 nodes
    assert n > 2**32
    o = opmm.fit_options(kernel_variant=1, cpu_check=0)
    r1 = opmm.opmm_fit(h, rec, ctl, sp, n, o)
    r0 = opmm.opmm_fit(h, rec, ctl, sp, n, opmm.fit_options(kernel_variant=1, cpu_check=0,
                                                           flags=opmm.FIT_FLAG_NO_GRID_TABLES))
    assert (r1["best_index"], r1["opt_err"], r1["n_finite"]) == (r0["best_index"], r0["opt_err"], r0["n_finite"])
    # the tail past 2^32 alone, element-wise
    tail = 4 * 10**6
    e1 = torch.empty(n, dtype=torch.float64, device="cuda")
    e0 = torch.empty(n, dtype=torch.float64, device="cuda")
    opmm.opmm_fit(h, rec, ctl, sp, n, opmm.fit_options(kernel_variant=1, cpu_check=0, err_out=e1))
    opmm.opmm_fit(h, rec, ctl, sp, n, opmm.fit_options(kernel_variant=1, cpu_check=0, err_out=e0,
                                                      flags=opmm.FIT_FLAG_NO_GRID_TABLES))
    torch.cuda.synchronize()
    assert torch.equal(e1[-tail:].isnan(), e0[-tail:].isnan())
    assert bool((e1[-tail:] == e0[-tail:]).logical_or(e1[-tail:].isnan()).all())
    del e1, e0
    # a long trace (fp64 rel 128 KB in shared memory) with large tables (1900 entries)
    cl = W.Control(n_steps=16000)
    rl = trace(cl)
    spl = W.grid_space({"N_SAC_AG": (d[I["N_SAC_AG"]] * 0.5, d[I["N_SAC_AG"]] * 1.5, 900, False),
                        "PW": (1.0, 16000.0, 1000, False)})
    sub = 9 * 10**5
    for prec in (0, 1):
        a1, A1 = _fit(opmm, h, rl, cl, spl, spl.n_grid(), precision=prec, kernel_variant=1)
        a0, A0 = _fit(opmm, h, rl, cl, spl, spl.n_grid(), precision=prec, kernel_variant=1,
                      flags=opmm.FIT_FLAG_NO_GRID_TABLES)
        assert (a1["best_index"], a1["opt_err"], a1["n_finite"]) == (a0["best_index"], a0["opt_err"], a0["n_finite"])
        assert np.array_equal(A1[:sub], A0[:sub], equal_nan=True)
    S = 4
    amp, pw, truths = W.population(S)
    ctls = [W.Control(n_steps=150, amplitude_deg=float(amp[k]), pw_default_ms=float(pw[k])) for k in range(S)]
    recs = np.array([oracle.positions(truths[k], ctls[k]) + W.noise(151, seed=40 + k) for k in range(S)])
    spg = _grid_spaces()[1][1]
    npg = spg.n_grid()
    for fl in (0, opmm.FIT_FLAG_NO_GRID_TABLES):
        err = torch.empty((S, npg), dtype=torch.float64, device="cuda")
        res = opmm.opmm_fit_batch(h, recs, ctls, spg, npg, opmm.fit_options(kernel_variant=1, err_out=err, flags=fl))
        torch.cuda.synchronize()
        if fl == 0:
            ref_res, ref_err = res, err.cpu().numpy()
        else:
            assert np.array_equal(err.cpu().numpy(), ref_err, equal_nan=True)
            for k in range(S):
                assert (res[k]["best_index"], res[k]["opt_err"]) == (ref_res[k]["best_index"], ref_res[k]["opt_err"])


def test_sync_fit_with_topk_uses_this_calls_trace(opmm):
    """Regression: opmm_fit with a host trace and top_k / certify (the
    non-graph path) must stage THIS call's trace -- on a fresh handle, and
    after a graph-path fit of a different trace."""
    ctl = W.Control()
    a = trace(ctl)
    b = oracle.positions(W.truth_opc(pw_ms=30.0), ctl) + W.noise(101, seed=77)
    sp = W.paper_space()
    n = 50000
    with opmm.opmm_create(0) as hh:
        outs = {}
        for name, r in (("a", a), ("b", b)):
            out = torch.zeros(ctypes_sizeof_fitresult(opmm), dtype=torch.uint8, device="cuda")
            opmm.opmm_fit_async(hh, dev(r), ctl, sp, n, out, opmm.fit_options(top_k=8))
            torch.cuda.synchronize()
            outs[name] = opmm.decode_result(bytes(out.cpu().numpy()))
    with opmm.opmm_create(0) as hh:
        r1 = opmm.opmm_fit(hh, b, ctl, sp, n, opmm.fit_options(top_k=8))        # fresh handle
        assert (r1["best_index"], r1["opt_err"], r1["topk_index"]) == \
               (outs["b"]["best_index"], outs["b"]["opt_err"], outs["b"]["topk_index"])
        opmm.opmm_fit(hh, a, ctl, sp, n)                                          # graph path, trace a
        r2 = opmm.opmm_fit(hh, b, ctl, sp, n, opmm.fit_options(top_k=8))        # then b with top-K
        assert (r2["best_index"], r2["opt_err"], r2["topk_index"]) == \
               (outs["b"]["best_index"], outs["b"]["opt_err"], outs["b"]["topk_index"])
        r3 = opmm.opmm_fit(hh, a, ctl, sp, n, opmm.fit_options(precision=opmm.FP32, certify=1))
        assert r3["certified"] == 1 and r3["best_index"] == outs["a"]["best_index"]


def ctypes_sizeof_fitresult(opmm):
    import ctypes
    return ctypes.sizeof(opmm.FitResult)


def _merge_shards(opmm, parts, K=0):
    be, bi = opmm.opmm_merge_argmin([p["opt_err"] if p["best_index"] >= 0 else np.inf for p in parts],
                                    [p["best_index"] for p in parts])
    out = {"best_index": bi, "opt_err": be, "n_finite": sum(p["n_finite"] for p in parts),
           "n_evaluated": sum(p["n_evaluated"] for p in parts)}
    if K:
        oe, oi = opmm.opmm_merge_topk([p["topk_err"][:K] for p in parts], [p["topk_index"][:K] for p in parts], K)
        out["topk_err"], out["topk_index"] = oe.tolist(), oi.tolist()
    return out


def test_fit_shard_partitions_and_merges(opmm, h):
    """opmm_fit_shard (SURVEY 8(e) on a plain handle, host merge): the
    per-rank kernels of a sharded fit -- candidate ranges starting past 0,
    each rank's partial, its top-K list -- merged on the host equal the single
    fit, for several world sizes; FP32 certification per shard composes to
    the certified single-GPU winner; the superposition kernel shards grid
    nodes and merges to the same winner."""
    ctl = W.Control()
    rec = trace(ctl)
    sp = W.paper_space()
    n = 300001
    K = 8
    full = opmm.opmm_fit(h, rec, ctl, sp, n, opmm.fit_options(top_k=K))
    for world in (2, 3, 7):
        parts = [opmm.opmm_fit_shard(h, rec, ctl, sp, n, r, world, opmm.fit_options(top_k=K))
                 for r in range(world)]
        for r, p in enumerate(parts):
            lo, hi = opmm.opmm_shard_range(n, r, world)
            assert p["n_evaluated"] == hi - lo
            assert p["best_index"] < 0 or lo <= p["best_index"] < hi
        m = _merge_shards(opmm, parts, K)
        assert (m["best_index"], m["opt_err"], m["n_finite"], m["n_evaluated"]) == \
               (full["best_index"], full["opt_err"], full["n_finite"], n), world
        assert m["topk_index"] == full["topk_index"][:K] and m["topk_err"] == full["topk_err"][:K], world
    # fp32 certified: every shard certified, merged winner = the certified single fit's
    c = opmm.opmm_fit(h, rec, ctl, sp, n, opmm.fit_options(precision=opmm.FP32, certify=1))
    parts = [opmm.opmm_fit_shard(h, rec, ctl, sp, n, r, 4, opmm.fit_options(precision=opmm.FP32, certify=1))
             for r in range(4)]
    assert all(p["certified"] == 1 for p in parts)
    m = _merge_shards(opmm, parts)
    assert c["certified"] == 1 and (m["best_index"], m["opt_err"]) == (c["best_index"], c["opt_err"])
    # the superposition kernel (auto on this grid) shards nodes
    g = W.g4_space(20)
    fg = opmm.opmm_fit(h, rec, ctl, g, g.n_grid())
    parts = [opmm.opmm_fit_shard(h, rec, ctl, g, g.n_grid(), r, 3) for r in range(3)]
    m = _merge_shards(opmm, parts)
    assert (m["best_index"], m["opt_err"], m["n_finite"], m["n_evaluated"]) == \
           (fg["best_index"], fg["opt_err"], fg["n_finite"], g.n_grid())
    with pytest.raises(opmm.OpmmError) as ei:
        opmm.opmm_fit_shard(h, rec, ctl, sp, n, 3, 3)
    assert ei.value.status == opmm.ERR_INVALID_ARG


def test_fit_async_matches_sync(opmm, h):
    import ctypes
    ctl = W.Control()
    rec = trace(ctl)
    sp = W.paper_space()
    n = 20000
    r = opmm.opmm_fit(h, rec, ctl, sp, n)
    out = torch.zeros(ctypes.sizeof(opmm.FitResult), dtype=torch.uint8, device="cuda")
    recd = dev(rec)
    torch.cuda.synchronize()
    opmm.opmm_fit_async(h, recd, ctl, sp, n, out)
    torch.cuda.ExternalStream(h.stream).synchronize()
    ra = opmm.decode_result(bytes(out.cpu().numpy()))
    assert ra["best_index"] == r["best_index"] and ra["opt_err"] == r["opt_err"]
    assert math.isnan(ra["cpu_check"])


# --------------------------------------------------------------------------- edge cases
def test_edge_empty_single_ragged(opmm, h):
    ctl = W.Control()
    rec = trace(ctl)
    sp = W.paper_space()
    r = opmm.opmm_fit(h, rec, ctl, sp, 0)
    assert r["best_index"] == -1 and r["n_finite"] == 0
    with pytest.raises(opmm.OpmmError) as ei:
        opmm.opmm_fit(h, rec, ctl, sp, 0, raise_no_finite=True)
    assert ei.value.status == opmm.ERR_NO_FINITE
    for n in (1, 31, 33, 257):
        r, E = _fit(opmm, h, rec, ctl, sp, n)
        o = oracle.fit(rec, ctl, sp, 0, n, want_err=True)
        assert r["best_index"] == o["best_index"] and r["n_evaluated"] == n
        assert np.array_equal(np.isinf(E), np.isinf(o["err"]))


@pytest.mark.parametrize("precision", [0, 1])
def test_fit_space_with_nonphysical_candidates(opmm, h, precision):
    """A search space whose candidates are not all physical (B_AG and N_C_AG
    ranges crossing zero): the fit kernel runs the per-candidate physical
    check (SPEC D8, reading Q13) and scores violators with the penalty
    1e10 (1 + sum of violations) exactly as the oracle does; the argmin is
    unaffected.  Random and grid (level tables) spaces; variants that need a
    physical space refuse it."""
    ctl = W.Control()
    rec = trace(ctl)
    d = W.truth_opc()
    sp = W.paper_space()
    sp.log_scale[I["B_AG"]] = 0
    sp.lo[I["B_AG"]], sp.hi[I["B_AG"]] = -0.2 * d[I["B_AG"]], 3.0 * d[I["B_AG"]]
    sp.log_scale[I["N_C_AG"]] = 0
    sp.lo[I["N_C_AG"]], sp.hi[I["N_C_AG"]] = -0.5 * d[I["N_C_AG"]], 2.0 * d[I["N_C_AG"]]
    g = W.grid_space({"B_AG": (-0.2 * d[I["B_AG"]], 3.0 * d[I["B_AG"]], 40, False),
                      "PW": (10.0, 60.0, 26, False)})
    for space, n in ((sp, 20000), (g, g.n_grid())):
        r, E = _fit(opmm, h, rec, ctl, space, n, precision=precision)
        o = oracle.fit(rec, ctl, space, 0, n, want_err=True)
        O = o["err"]
        pen = np.array([oracle.physical_penalty(oracle.generate(space, i)) for i in range(n)])
        assert (pen > 0).sum() > n // 20                          # the check is exercised
        assert np.array_equal(E[pen > 0], O[pen > 0])             # penalties exact
        assert r["best_index"] == o["best_index"]
        if precision == 0:
            rel, _, _ = oracle.relativize(rec, ctl.amplitude_deg)
            f = pen == 0
            assert_fp64_errors(E[f], O[f], lambda i, f=np.flatnonzero(f): oracle.generate(space, int(f[i])),
                               rec, ctl, np.abs(rel).sum())
    for kv in (2, 3, 5):
        with pytest.raises(opmm.OpmmError) as ei:
            _fit(opmm, h, rec, ctl, sp, 1000, kernel_variant=kv)
        assert ei.value.status == opmm.ERR_UNSUPPORTED


def test_edge_all_diverged(opmm, h):
    ctl = W.Control()
    rec = trace(ctl, noisy=False)
    d = W.truth_opc()
    d[I["J"]] = 1e-9
    d[I["B_AG"]] = 1e-6
    d[I["B_ANT"]] = 1e-6
    sp = W.grid_space({"PW": (10.0, 20.0, 3, False)}, base=d)
    r, E = _fit(opmm, h, rec, ctl, sp, 3)
    assert r["best_index"] == -1 and r["n_finite"] == 0 and np.all(np.isinf(E))


@pytest.mark.parametrize("n_steps", [1, 2, 37, 4000, 16384])   # 16384 = OPMM_MAX_STEPS
def test_edge_trace_lengths(opmm, h, n_steps):
    ctl = W.Control(n_steps=n_steps, dt_ms=1.0 if n_steps < 1000 else 0.05)
    rec = oracle.positions(W.truth_opc(), ctl) + W.noise(n_steps + 1)
    sp = W.paper_space(n_steps=n_steps, dt_ms=ctl.dt_ms)
    n = 300
    r, E = _fit(opmm, h, rec, ctl, sp, n)
    o = oracle.fit(rec, ctl, sp, 0, n, want_err=True)
    O = o["err"]
    rel, _, _ = oracle.relativize(rec, ctl.amplitude_deg)
    assert_fp64_errors(E, O, lambda i: oracle.generate(sp, i), rec, ctl, max(np.abs(rel).sum(), 1e-300))
    assert r["best_index"] == o["best_index"]


def test_edge_amplitude_from_trace_and_negative(opmm, h):
    sp = W.paper_space()
    for amp, th0, given in ((-12.0, 4.0, True), (10.0, 0.0, False)):
        ctl = W.Control(amplitude_deg=amp, theta0_deg=th0)
        rec = trace(ctl)
        use = ctl if given else W.Control(amplitude_deg=math.nan)
        r, E = _fit(opmm, h, rec, use, sp, 2000)
        o = oracle.fit(rec, use, sp, 0, 2000, want_err=True)
        assert r["best_index"] == o["best_index"]
        assert_fp64_errors(E, o["err"], lambda i: oracle.generate(sp, i), rec, use, 100.0)


# --------------------------------------------------------------------------- population
def test_fit_batch_population(opmm, h):
    S = 48
    amp, pw, truths = W.population(S)
    n_steps = 150
    ctls, recs = [], []
    for s in range(S):
        c = W.Control(n_steps=n_steps, amplitude_deg=amp[s], pw_default_ms=pw[s])
        ctls.append(c)
        recs.append(oracle.positions(truths[s], c) + W.noise(n_steps + 1, seed=1000 + s))
    recs = np.array(recs)
    sp = W.paper_space(n_steps=n_steps)
    n_per = 3000
    err = torch.full((S, n_per), -1.0, dtype=torch.float64, device="cuda")
    res = opmm.opmm_fit_batch(h, recs, ctls, sp, n_per, opmm.fit_options(err_out=err))
    E = err.cpu().numpy()
    for s in (0, 1, 17, 47):
        o = oracle.fit(recs[s], ctls[s], sp, 0, n_per, saccade=s, want_err=True)
        rel, _, _ = oracle.relativize(recs[s], ctls[s].amplitude_deg)
        assert_fp64_errors(E[s], o["err"], lambda i, s=s: oracle.generate(sp, i, saccade=s), recs[s], ctls[s],
                           np.abs(rel).sum())
        assert res[s]["best_index"] == o["best_index"], s
        assert abs(res[s]["opt_err"] - o["best_err"]) <= 1e-9 * max(o["best_err"], 1.0)
        assert abs(res[s]["cpu_check"] - res[s]["opt_err"]) <= 1e-9 * res[s]["opt_err"]


def test_nccl_single_rank_merge_path(opmm, h):
    """The multi-GPU path on one GPU: a 1-rank NCCL communicator (libnccl.so.2
    loaded at run time), the per-rank 32-byte partial, ncclAllGather on the
    handle's stream and the merge kernel -- same result as the plain fit."""
    import os
    import subprocess
    import sys
    code = r'''
import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import torch, oracle, workloads as W
from paper_2007_09884_b200 import opmm
ctl = W.Control(); sp = W.paper_space()
rec = oracle.positions(W.truth_opc(), ctl) + W.noise(101)
uid = opmm.opmm_nccl_unique_id()
with opmm.opmm_create_nccl(0, uid, 0, 1) as hn, opmm.opmm_create(0) as hp:
    for n in (1, 777, 100000):
        a = opmm.opmm_fit(hn, rec, ctl, sp, n)
        b = opmm.opmm_fit(hp, rec, ctl, sp, n)
        assert (a["best_index"], a["opt_err"], a["n_finite"], a["n_evaluated"]) == \
               (b["best_index"], b["opt_err"], b["n_finite"], b["n_evaluated"]), (n, a, b)
        assert a["opc"].tolist() == b["opc"].tolist()
    # the 544-byte rank results: exact top-K lists, and fp32 certification
    # re-scored by the merge kernel -- identical to the single-GPU handle
    for o in (opmm.fit_options(top_k=9), opmm.fit_options(precision=opmm.FP32, certify=1),
              opmm.fit_options(precision=opmm.FP32, certify=1, top_k=5, metric=1)):
        a = opmm.opmm_fit(hn, rec, ctl, sp, 100000, o)
        b = opmm.opmm_fit(hp, rec, ctl, sp, 100000, o)
        for k in ("best_index", "opt_err", "n_finite", "top_k", "certified", "topk_index", "topk_err"):
            assert a[k] == b[k], (k, a[k], b[k])
        assert a["top_k"] > 0 and (o.certify == 0 or a["certified"] == 1)
print("nccl-single-rank ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                       timeout=300)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "nccl-single-rank ok" in p.stdout



def test_nine_param_model_fit_and_generator(opmm, h):
    """9-parameter OPMM (Table 2 + D7): generated candidates and every error of
    a fit match the oracle; TRUTH-like data is fitted near the default."""
    sp = W.paper_space_9()
    n = 4096
    out = torch.zeros((18, n), dtype=torch.float64, device="cuda")
    opmm.opmm_generate(h, sp, 0, n, out, stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    g = out.cpu().numpy().T
    o = oracle.generate_batch(sp, 0, n)
    assert np.array_equal(np.isnan(g), np.isnan(o))
    f = ~np.isnan(o)
    assert np.max(np.abs(g[f] - o[f]) / np.abs(o[f])) <= 2 * ULP
    ctl = W.Control()
    rec = trace(ctl)
    r, E = _fit(opmm, h, rec, ctl, sp, 20000)
    orc = oracle.fit(rec, ctl, sp, 0, 20000, want_err=True)
    rel, _, _ = oracle.relativize(rec, ctl.amplitude_deg)
    assert_fp64_errors(E, orc["err"], lambda i: oracle.generate(sp, i), rec, ctl, np.abs(rel).sum())
    assert r["best_index"] == orc["best_index"]
    assert np.isnan(r["opc"][I["PW"]]) and r["opc"][I["K_SE_ANT"]] == r["opc"][I["K_SE_AG"]]


def test_fp32_certified_fit(opmm, h):
    """FP32 fit with certification: the exact top-K by
    (fp32 E, index) re-scored in fp64 (K = 8 by default, top_k when given); the returned winner and opt_err equal
    the fp64 fit's, the run reports itself certified, and the certificate is
    sound: the list is the host's exact top-K of all fp32 errors, every
    candidate within T* = E32[0] + 2 delta is in it, and every listed
    candidate's fp32 and fp64 errors agree within delta."""
    ctl = W.Control()
    rec = trace(ctl)
    sp = W.paper_space()
    n = 200000
    r64, E64 = _fit(opmm, h, rec, ctl, sp, n, precision=opmm.FP64)
    r32, E32 = _fit(opmm, h, rec, ctl, sp, n, precision=opmm.FP32)
    rc = opmm.opmm_fit(h, rec, ctl, sp, n, opmm.fit_options(precision=opmm.FP32, certify=1))
    order = np.lexsort((np.arange(n), E32))
    kept = np.array(rc["topk_index"])
    assert rc["top_k"] == 8 and kept.tolist() == order[:8].tolist()
    assert rc["topk_err"] == E64[kept].tolist()
    srel = np.abs(rec - rec[0]).sum()
    delta = 1e-4 * max(E32[order[0]], srel)
    tstar = E32[order[0]] + 2.0 * delta
    assert set(np.nonzero(E32 <= tstar)[0].tolist()) <= set(kept.tolist())
    assert np.all(np.abs(E64[kept] - E32[kept]) <= delta)
    assert rc["best_index"] == r64["best_index"] and rc["opt_err"] == r64["opt_err"]
    assert rc["certified"] == 1
    assert abs(rc["cpu_check"] - rc["opt_err"]) <= 1e-9 * rc["opt_err"]
    # K = top_k when given
    r32 = opmm.opmm_fit(h, rec, ctl, sp, n, opmm.fit_options(precision=opmm.FP32, certify=1, top_k=32))
    assert r32["top_k"] == 32 and r32["topk_index"] == order[:32].tolist() and r32["certified"] == 1
    assert r32["topk_err"] == E64[order[:32]].tolist()
    # RMS metric: the budget's floor is the RMS of the trace; still certified
    # and still the fp64 fit's winner
    r64r, E64r = _fit(opmm, h, rec, ctl, sp, n, precision=opmm.FP64, metric=1)
    rr = opmm.opmm_fit(h, rec, ctl, sp, n, opmm.fit_options(precision=opmm.FP32, certify=1, metric=1))
    assert rr["certified"] == 1 and rr["best_index"] == r64r["best_index"]
    assert rr["opt_err"] == r64r["opt_err"]
    # several super-tile passes per block (3e6 > 148 blocks x 8192): same winner
    big = 3 * 10**6
    b64 = opmm.opmm_fit(h, rec, ctl, sp, big, opmm.fit_options(precision=opmm.FP64))
    b32 = opmm.opmm_fit(h, rec, ctl, sp, big, opmm.fit_options(precision=opmm.FP32, certify=1))
    assert b32["certified"] == 1 and (b32["best_index"], b32["opt_err"]) == (b64["best_index"], b64["opt_err"])
    assert b32["n_finite"] == b64["n_finite"]
    # fewer finite candidates than K: certified; unused slots -1 / +inf
    small = opmm.opmm_fit(h, rec, ctl, sp, 3, opmm.fit_options(precision=opmm.FP32, certify=1))
    assert small["certified"] == 1 and small["topk_index"][3:] == [-1] * 5
    assert all(math.isinf(x) for x in small["topk_err"][3:])
    # fp64 ignores certify; fit3 refuses it
    assert opmm.opmm_fit(h, rec, ctl, sp, 1000, opmm.fit_options(certify=1))["top_k"] == 0
    with pytest.raises(opmm.OpmmError) as ei:
        opmm.opmm_fit(h, rec, ctl, sp, 1000, opmm.fit_options(precision=opmm.FP32, certify=1,
                                                              kernel_variant=3))
    assert ei.value.status == opmm.ERR_UNSUPPORTED


def test_fp32_certified_population(opmm, h):
    """FP32 certification per saccade of opmm_fit_batch: each saccade keeps
    its own exact fp32 top-8 and re-scores it in fp64; every saccade is
    certified and returns the fp64 batch's winner and error."""
    S = 24
    amp, pw, truths = W.population(S)
    ctls = [W.Control(n_steps=150, amplitude_deg=float(amp[k]), pw_default_ms=float(pw[k])) for k in range(S)]
    recs = np.array([oracle.positions(truths[k], ctls[k]) + W.noise(151, seed=300 + k) for k in range(S)])
    sp = W.paper_space(n_steps=150)
    n_per = 20000
    b64 = opmm.opmm_fit_batch(h, recs, ctls, sp, n_per, opmm.fit_options(precision=opmm.FP64))
    b32 = opmm.opmm_fit_batch(h, recs, ctls, sp, n_per, opmm.fit_options(precision=opmm.FP32, certify=1))
    for k in range(S):
        assert b32[k]["certified"] == 1 and b32[k]["top_k"] == 8, k
        assert (b32[k]["best_index"], b32[k]["opt_err"]) == (b64[k]["best_index"], b64[k]["opt_err"]), k
        assert b32[k]["n_finite"] == b64[k]["n_finite"], k


def test_fp32_certificate_refused_on_near_ties(opmm, h):
    """The certificate is not a formality: 64 candidates whose errors agree to
    ~1e-9 relative (K_LT_ANT varied by 1e-9) all lie within T*, so no list of
    K < 64 can hold every candidate within T*: certified = 0, and the fit
    still returns the fp64-best of its list."""
    ctl = W.Control()
    rec = trace(ctl)
    d = W.truth_opc()
    v = d[I["K_LT_ANT"]]
    sp = W.grid_space({"K_LT_ANT": (v, v * (1 + 1e-9), 64, False)})
    r64, E64 = _fit(opmm, h, rec, ctl, sp, 64, precision=opmm.FP64)
    rc = opmm.opmm_fit(h, rec, ctl, sp, 64, opmm.fit_options(precision=opmm.FP32, certify=1, top_k=4))
    assert rc["certified"] == 0 and rc["top_k"] == 4
    kept = rc["topk_index"]
    assert rc["opt_err"] == min(E64[kept])
    assert rc["best_index"] == kept[int(np.argmin(E64[kept]))]


@pytest.mark.parametrize("precision", [0, 1])
def test_topk_exact_against_all_errors(opmm, h, precision):
    """top_k = K returns exactly the K smallest (E, index) pairs over all
    candidates, in lexicographic order, for any K <= 32 and launch
    configuration (ragged N, several super-tile passes, small blocks)."""
    ctl = W.Control()
    rec = trace(ctl)
    sp = W.paper_space()
    n = 300001
    r0, E = _fit(opmm, h, rec, ctl, sp, n, precision=precision)
    order = np.lexsort((np.arange(n), E))
    for K, bs, gb in ((1, 0, 0), (7, 0, 0), (32, 0, 0), (32, 64, 3), (13, 128, 0), (32, 0, 1)):
        r, E2 = _fit(opmm, h, rec, ctl, sp, n, precision=precision, top_k=K, block_size=bs,
                     grid_blocks=gb)
        assert np.array_equal(E, E2)
        assert r["top_k"] == K
        assert r["topk_index"] == order[:K].tolist(), (K, bs, gb)
        assert r["topk_err"] == E[order[:K]].tolist()
        assert (r["best_index"], r["opt_err"]) == (r0["best_index"], r0["opt_err"])
    with pytest.raises(opmm.OpmmError) as ei:
        _fit(opmm, h, rec, ctl, sp, 100, top_k=33)
    assert ei.value.status == opmm.ERR_INVALID_ARG


def test_topk_exact_ties_and_population(opmm, h):
    """Exact ties keep the lowest indices first; opmm_fit_batch returns every
    saccade's own exact top-K (against the oracle's errors)."""
    ctl = W.Control()
    rec = trace(ctl)
    d = W.truth_opc()
    sp = W.grid_space({"N_SAC_AG": (d[15] * 0.99, d[15] * 1.01, 3, False),
                       "PW": (39.21, 40.0, 3, False)})
    r, E = _fit(opmm, h, rec, ctl, sp, 9, top_k=9)
    assert r["topk_index"][:9] == np.lexsort((np.arange(9), E)).tolist()
    S = 6
    amp, pw, truths = W.population(S)
    ctls = [W.Control(n_steps=150, amplitude_deg=amp[s], pw_default_ms=pw[s]) for s in range(S)]
    recs = np.array([oracle.positions(truths[s], ctls[s]) + W.noise(151, seed=1000 + s) for s in range(S)])
    spp = W.paper_space(n_steps=150)
    n_per = 4000
    res = opmm.opmm_fit_batch(h, recs, ctls, spp, n_per, opmm.fit_options(top_k=10))
    for s in (0, 3, 5):
        o = oracle.fit(recs[s], ctls[s], spp, 0, n_per, saccade=s, want_err=True)
        order = np.lexsort((np.arange(n_per), o["err"]))[:10]
        assert res[s]["topk_index"] == order.tolist(), s
        assert np.allclose(res[s]["topk_err"], o["err"][order], rtol=1e-9, atol=0)


# --------------------------------------------------------------------------- streams
def test_torch_default_stream_ordering(opmm, h):
    """Work passed torch's default stream is ordered with torch's own kernels
    (the binding maps the legacy NULL stream to cudaStreamLegacy): simulating
    one candidate at a time into a reused buffer and copying it out with torch,
    with no synchronisation in between, equals one batched simulate."""
    ctl = W.Control()
    cands = np.asarray(oracle.generate_batch(W.paper_space(), 0, 64))
    cands = cands[[i for i in range(64) if oracle.physical_penalty(cands[i]) == 0.0][:48]]
    n = len(cands)
    opc = soa(cands)
    ref = torch.zeros((ctl.n_steps + 1, n), dtype=torch.float64, device="cuda")
    opmm.opmm_simulate(h, opc, n, ctl, ref, stream=torch.cuda.current_stream())
    col = torch.zeros(ctl.n_steps + 1, dtype=torch.float64, device="cuda")
    out = torch.zeros_like(ref)
    for s in range(n):
        opmm.opmm_simulate(h, opc[:, s].contiguous(), 1, ctl, col, stream=torch.cuda.current_stream())
        out[:, s] = col
    torch.cuda.synchronize()
    assert torch.equal(out.isnan(), ref.isnan())
    assert torch.equal(torch.nan_to_num(out), torch.nan_to_num(ref))


def test_simulate_batch_equals_single_calls(opmm, h):
    """opmm_simulate_batch (one control per candidate) is bit-identical to
    single-candidate opmm_simulate calls; mixed-step batches are rejected."""
    amp, pw, truths = W.population(40)
    ctls = [W.Control(n_steps=150, amplitude_deg=float(a) * (-1) ** k, theta0_deg=0.5 * k,
                      pw_default_ms=float(p)) for k, (a, p) in enumerate(zip(amp, pw))]
    n = len(ctls)
    opc = soa(truths)
    got = torch.zeros((151, n), dtype=torch.float64, device="cuda")
    st = torch.zeros(n, dtype=torch.uint8, device="cuda")
    opmm.opmm_simulate_batch(h, opc, n, ctls, got, status=st, stream=torch.cuda.current_stream())
    ref = torch.zeros_like(got)
    for s in range(n):
        col = torch.zeros(151, dtype=torch.float64, device="cuda")
        opmm.opmm_simulate(h, opc[:, s].contiguous(), 1, ctls[s], col, stream=torch.cuda.current_stream())
        ref[:, s] = col
    torch.cuda.synchronize()
    assert torch.equal(got, ref)
    assert int(st.sum()) == 0
    bad = list(ctls)
    bad[3] = W.Control(n_steps=100)
    with pytest.raises(opmm.OpmmError):
        opmm.opmm_simulate_batch(h, opc, n, bad, got)


# --------------------------------------------------------------------------- substeps (Q25)
@pytest.mark.parametrize("integrator", [0, 1])
@pytest.mark.parametrize("substeps", [2, 3, 8])
def test_simulate_substeps_fp64(opmm, h, integrator, substeps):
    """s RK4 substeps per sample: the propagator composes the substep map s
    times (binary powering) into one sample map; the four-stage integrator
    runs the s substeps literally.  Both against the oracle's literal
    substeps, fp64 1e-9 on every finite trajectory."""
    ctl = W.Control(substeps=substeps)
    cands = candidate_set()
    n = len(cands)
    traj = torch.full((ctl.n_steps + 1, n), -1.0, dtype=torch.float64, device="cuda")
    status = torch.zeros(n, dtype=torch.uint8, device="cuda")
    opmm.opmm_simulate(h, soa(cands), n, ctl, traj, integrator=integrator, status=status,
                       stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    T, S = traj.cpu().numpy(), status.cpu().numpy()
    refs = oracle_dtheta(cands, ctl)
    checked = 0
    for i, ref in enumerate(refs):
        if ref is None:
            assert S[i] == 1
            continue
        if not (np.all(np.isfinite(ref)) and np.abs(ref).sum() < 1e20):
            assert S[i] == 2, i
            continue
        assert S[i] == 0, i
        err = np.max(np.abs(T[:, i] - ref)) / max(np.max(np.abs(ref)), 1.0)
        assert err <= 1e-9, (i, err)
        checked += 1
    assert checked > n // 3


@pytest.mark.parametrize("precision", [0, 1])
def test_fit_substeps_matches_oracle(opmm, h, precision):
    """Fit with 4 substeps per sample: every candidate's E against the oracle
    (fp64: Q22 rule with the substep-aware referee; fp32: finite/+inf
    classification and the winner), and substeps stabilise candidates that
    diverge at h = dt."""
    ctl = W.Control(substeps=4)
    rec = trace(W.Control())
    sp = W.paper_space()
    n = 2000
    r, E = _fit(opmm, h, rec, ctl, sp, n, precision=precision)
    o = oracle.fit(rec, ctl, sp, 0, n, want_err=True, nthreads=oracle.max_threads())
    O = o["err"]
    if precision == 0:
        assert_fp64_errors(E, O, lambda i: oracle.generate(sp, i), rec, ctl, np.abs(rec - rec[0]).sum())
        assert r["best_index"] == o["best_index"]
    else:
        assert np.array_equal(np.isinf(E), np.isinf(O))
    plain = oracle.fit(rec, W.Control(), sp, 0, n)
    assert o["n_finite"] > plain["n_finite"]
    assert r["n_finite"] == o["n_finite"]
    assert abs(r["cpu_check"] - o["best_err"]) <= 1e-9 * o["best_err"] or precision == 1


@pytest.mark.parametrize("schedule", [1, 2, 3], ids=["lockstep", "lane", "group"])
def test_nm_substeps_reference_bit_identical(opmm, h, schedule):
    """The reference-order NM objective with substeps is bit-identical to the
    oracle's serial Nelder-Mead with substeps, in both NM schedules; the
    propagator objective with substeps gives the same run in both."""
    ctl = W.Control(substeps=3, amplitude_deg=10.0)
    rec = trace(W.Control())
    res = opmm.opmm_estimate_batch(h, rec[None, :], [ctl],
                                   options=opmm.nm_options(objective=opmm.NM_OBJ_REFERENCE,
                                                           max_iter=60, cpu_check=0,
                                                           schedule=schedule))
    o = oracle.estimate_batch(rec[None, :], [ctl], max_iter=60)
    assert res[0]["iterations"] == int(o["iterations"][0])
    assert res[0]["f"] == float(o["f"][0])
    assert np.array_equal(np.array(res[0]["x"]), o["x"][0])
    fast = [opmm.opmm_estimate_batch(h, rec[None, :], [ctl],
                                     options=opmm.nm_options(max_iter=60, cpu_check=0, schedule=sc))[0]
            for sc in (1, 2, 3)]
    assert fast[0]["f"] == fast[1]["f"] == fast[2]["f"]
    assert fast[0]["x"].tolist() == fast[1]["x"].tolist() == fast[2]["x"].tolist()


def test_sync_fit_graph_replay_and_invalidation(opmm, h):
    """opmm_fit replays a captured graph (H2D + kernel + D2H) while the launch
    is unchanged and re-captures when it changes (trace length, N, precision,
    a host buffer grown by a batch call): every call equals the direct path."""
    ctl = W.Control()
    rec = trace(ctl)
    sp = W.paper_space()
    runs = [(rec, ctl, 3000, 0), (rec + 0.1, ctl, 3000, 0), (rec, ctl, 5000, 0), (rec, ctl, 3000, 1)]
    longc = W.Control(n_steps=150)
    runs.append((oracle.positions(W.truth_opc(), longc) + W.noise(151), longc, 3000, 0))
    got = [opmm.opmm_fit(h, r, c, sp, n, opmm.fit_options(precision=p)) for r, c, n, p in runs]
    # grow the pinned result buffer with a batch, then fit again
    amp, pw, _ = W.population(4)
    opmm.opmm_fit_batch(h, np.stack([rec] * 4), [W.Control(amplitude_deg=float(a)) for a in amp], sp, 500)
    got.append(opmm.opmm_fit(h, rec, ctl, sp, 3000))
    ng = opmm.FIT_FLAG_NO_GRAPH
    ref = [opmm.opmm_fit(h, r, c, sp, n, opmm.fit_options(precision=p, flags=ng)) for r, c, n, p in runs]
    ref.append(opmm.opmm_fit(h, rec, ctl, sp, 3000, opmm.fit_options(flags=ng)))
    for g, r in zip(got, ref):
        assert (g["best_index"], g["opt_err"], g["n_finite"], g["cpu_check"]) == \
               (r["best_index"], r["opt_err"], r["n_finite"], r["cpu_check"])
    assert got[1]["opt_err"] != got[0]["opt_err"]   # the new trace reached the replayed graph
