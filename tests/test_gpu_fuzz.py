"""Seeded random configurations against the oracle (-m gpu).

Each case draws a search space (random or grid; every dimension fixed,
linear or log with random bounds around Table 1, some crossing into the
non-physical region), a control (dt, n_steps, amplitude given or from the
trace, theta0, pw_default, substeps), a metric and the fit options
(precision, top_k, certify, kernel variant), then checks the fit against the
oracle's exhaustive evaluation of the same candidates: FP64 errors within the
parity rule, the argmin and n_finite identical, the
top-K list the exact lexicographic top-K of the errors; FP32 with the same
classification and, when certified, the FP64 winner.  Small sizes so the
oracle finishes in a second per case.
"""
import numpy as np
import pytest

import oracle
import workloads as W
from test_gpu_parity import assert_fp64_errors, rk4_stable

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

I = W.IDX


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


def draw_case(seed):
    rng = np.random.default_rng(seed)
    d = np.array(W.TABLE1_DEFAULTS, dtype=np.float64)
    d[I["PW"]] = 40.0
    dt = float(rng.choice([0.5, 1.0, 2.0]))
    n_steps = int(rng.choice([1, 2, 7, 50, 100, 151, 300]))
    ctl = W.Control(dt_ms=dt, n_steps=n_steps,
                    amplitude_deg=float(rng.choice([10.0, -7.5, 25.0, np.nan])),
                    theta0_deg=float(rng.uniform(-5, 5)), pw_default_ms=float(rng.uniform(5, 60)),
                    substeps=int(rng.choice([0, 0, 0, 2])))
    grid = rng.random() < 0.4
    lo, hi = d.copy(), d.copy()
    logs = np.zeros(18, dtype=np.uint8)
    levels = np.ones(18, dtype=np.int32)
    dims = rng.choice(18, size=int(rng.integers(1, 6 if grid else 18)), replace=False)
    for k in dims:
        kind = rng.choice(["log", "lin", "lin_cross"])
        if kind == "log":
            lo[k], hi[k], logs[k] = d[k] * rng.uniform(0.1, 0.9), d[k] * rng.uniform(1.1, 10), 1
        elif kind == "lin":
            lo[k], hi[k] = d[k] * rng.uniform(0.2, 0.9), d[k] * rng.uniform(1.1, 3)
        else:   # may cross zero: non-physical candidates
            lo[k], hi[k] = -0.3 * d[k], d[k] * rng.uniform(1.1, 3)
        if k == I["PW"]:
            lo[k] = dt * rng.uniform(0.5, 2)
            hi[k], logs[k] = max(dt * n_steps * rng.uniform(0.5, 1.5), 1.5 * lo[k]), 0
    if grid:
        for k in dims:
            levels[k] = int(rng.integers(2, 9))
        sp = W.SearchSpace(1, 0, lo, hi, logs, levels)
        n = int(np.prod(levels.astype(np.int64)))
    else:
        sp = W.SearchSpace(0, int(rng.integers(0, 2**40)), lo, hi, logs, levels)
        n = int(rng.choice([1, 33, 999, 4000]))
    metric = int(rng.integers(0, 2))
    precision = int(rng.integers(0, 2))
    top_k = int(rng.choice([0, 0, 1, 5, 32]))
    certify = int(precision == 1 and rng.random() < 0.5)
    kv = int(rng.choice([0, 0, 1, 5] + ([4, 4] if grid else [])))
    if grid and kv == 4 and rng.random() < 0.7:   # make superposition eligible most of the time
        k = I["N_SAC_AG"] if rng.random() < 0.5 else I["N_SAC_ANT"]
        lo[k], hi[k], logs[k] = d[k] * 0.5, d[k] * 2.0, 1
        levels[k] = int(rng.integers(8, 40))
        for j in range(18):
            if lo[j] < 0:
                lo[j] = 0.1 * max(hi[j], 1e-9)
        if I["PW"] in dims:
            lo[I["PW"]] = max(lo[I["PW"]], 1e-3)
        sp = W.SearchSpace(1, 0, lo, hi, logs, levels)
        n = int(np.prod(levels.astype(np.int64)))
        top_k, certify = 0, 0
    return ctl, sp, n, metric, precision, top_k, certify, kv


@pytest.mark.parametrize("seed", range(80))
def test_random_configuration(opmm, h, seed):
    ctl, sp, n, metric, precision, top_k, certify, kv = draw_case(seed)
    rng = np.random.default_rng(1000 + seed)
    truth = np.array(W.TABLE1_DEFAULTS, dtype=np.float64)
    truth[I["PW"]] = 0.4 * ctl.n_steps * ctl.dt_ms + ctl.dt_ms
    c0 = W.Control(dt_ms=ctl.dt_ms, n_steps=ctl.n_steps,
                   amplitude_deg=10.0 if np.isnan(ctl.amplitude_deg) else ctl.amplitude_deg,
                   theta0_deg=ctl.theta0_deg, pw_default_ms=ctl.pw_default_ms, substeps=ctl.substeps)
    rec = oracle.positions(truth, c0) + rng.normal(0.0, 0.02, ctl.n_steps + 1)
    err = torch.full((n,), -1.0, dtype=torch.float64, device="cuda")
    o = opmm.fit_options(precision=precision, metric=metric, top_k=top_k, certify=certify, kernel_variant=kv,
                         err_out=err)
    try:
        r = opmm.opmm_fit(h, rec, ctl, sp, n, o)
    except opmm.OpmmError as e:
        # the only refusals: variants that need a physical space / the propagator /
        # no top-K (5), or a grid with a superposable pulse height (4)
        assert e.status == opmm.ERR_UNSUPPORTED and kv in (4, 5), (seed, e)
        return
    E = err.cpu().numpy()
    orc = oracle.fit(rec, ctl, sp, 0, n, metric=metric, want_err=True)
    O = orc["err"]
    assert r["n_evaluated"] == n
    assert np.array_equal(np.isinf(E), np.isinf(O)), seed
    assert r["n_finite"] == orc["n_finite"], seed
    rel, _, _ = oracle.relativize(rec, ctl.amplitude_deg)
    scale = np.abs(rel).sum() if metric == 0 else np.sqrt(np.mean(rel ** 2))
    if precision == 0:
        assert_fp64_errors(E, O, lambda i: oracle.generate(sp, i), rec, ctl, scale, metric)
        assert r["best_index"] == orc["best_index"], seed
    else:
        # FP32 scope: RK4-stable candidates
        f = np.flatnonzero(np.isfinite(O))
        st = np.array([rk4_stable(oracle.generate(sp, int(i)), ctl) for i in f], dtype=bool)
        g = f[st] if f.size else f
        assert np.all(np.abs(E[g] - O[g]) <= 1e-4 * np.maximum(O[g], scale)), seed
        if certify and r["certified"] == 1:
            assert r["best_index"] == orc["best_index"], seed
    K = top_k if top_k else (8 if certify else 0)
    if K:
        m = min(K, n)
        order = np.lexsort((np.arange(n), E))[:m].tolist()
        assert r["top_k"] == K and r["topk_index"][:m] == order, seed


@pytest.mark.parametrize("seed", range(20))
def test_random_population_batch(opmm, h, seed):
    """opmm_fit_batch on random configurations: S saccades with their own
    amplitude / pw_default (Philox counter word 2 = saccade), every
    saccade's errors, argmin and n_finite against the oracle's fit of that
    saccade."""
    ctl, sp, n, metric, precision, top_k, certify, kv = draw_case(500 + seed)
    rng = np.random.default_rng(2000 + seed)
    S = int(rng.integers(1, 5))
    ctls, recs = [], []
    for s in range(S):
        c = W.Control(dt_ms=ctl.dt_ms, n_steps=ctl.n_steps, amplitude_deg=float(rng.uniform(5, 30)),
                      theta0_deg=ctl.theta0_deg, pw_default_ms=float(rng.uniform(5, 60)), substeps=ctl.substeps)
        truth = np.array(W.TABLE1_DEFAULTS, dtype=np.float64)
        truth[I["PW"]] = rng.uniform(0.2, 0.6) * ctl.n_steps * ctl.dt_ms + ctl.dt_ms
        ctls.append(c)
        recs.append(oracle.positions(truth, c) + rng.normal(0.0, 0.02, ctl.n_steps + 1))
    recs = np.array(recs)
    err = torch.full((S, n), -1.0, dtype=torch.float64, device="cuda")
    o = opmm.fit_options(precision=0, metric=metric, top_k=top_k, err_out=err,
                         kernel_variant=kv if kv in (0, 1) else 0)
    res = opmm.opmm_fit_batch(h, recs, ctls, sp, n, o)
    E = err.cpu().numpy()
    for s in range(S):
        orc = oracle.fit(recs[s], ctls[s], sp, 0, n, metric=metric, saccade=s, want_err=True)
        rel, _, _ = oracle.relativize(recs[s], ctls[s].amplitude_deg)
        scale = np.abs(rel).sum() if metric == 0 else np.sqrt(np.mean(rel ** 2))
        assert np.array_equal(np.isinf(E[s]), np.isinf(orc["err"])), (seed, s)
        assert_fp64_errors(E[s], orc["err"], lambda i, s=s: oracle.generate(sp, i, saccade=s), recs[s], ctls[s],
                           scale, metric)
        assert (res[s]["best_index"], res[s]["n_finite"]) == (orc["best_index"], orc["n_finite"]), (seed, s)
        if top_k:
            m = min(top_k, n)
            assert res[s]["topk_index"][:m] == np.lexsort((np.arange(n), E[s]))[:m].tolist(), (seed, s)


@pytest.mark.parametrize("seed", range(12))
def test_random_nelder_mead_reference_bit_exact(opmm, h, seed):
    """Batched Nelder-Mead with the reference-order objective on random
    controls, start vectors, metrics, tolerances and initial scales, in all
    three schedules: every run bit-identical to the oracle's serial
    Lagarias run (x, f, iterations, evaluations, exit reason)."""
    rng = np.random.default_rng(3000 + seed)
    n_steps = int(rng.choice([20, 60, 150]))
    dt = float(rng.choice([0.5, 1.0]))
    S = int(rng.integers(1, 6))
    ctls, recs = [], []
    for s in range(S):
        c = W.Control(dt_ms=dt, n_steps=n_steps, amplitude_deg=float(rng.uniform(5, 30)),
                      pw_default_ms=float(rng.uniform(0.2, 0.6) * n_steps * dt + dt))
        truth = np.array(W.TABLE1_DEFAULTS, dtype=np.float64)
        truth *= np.exp(rng.uniform(-0.2, 0.2, 18))
        truth[I["PW"]] = c.pw_default_ms
        ctls.append(c)
        recs.append(oracle.positions(truth, c) + rng.normal(0.0, 0.02, n_steps + 1))
    recs = np.array(recs)
    x0 = np.array(W.TABLE1_DEFAULTS, dtype=np.float64) * np.exp(rng.uniform(-0.3, 0.3, 18))
    x0[I["PW"]] = np.nan
    metric = int(rng.integers(0, 2))
    tol = float(rng.choice([1e-4, 1e-6]))
    scale = float(rng.choice([0.05, 0.1]))
    max_iter = int(rng.choice([30, 120]))
    o = oracle.estimate_batch(recs, ctls, x0=x0, metric=metric, init_scale=scale, tol_x=tol, tol_f=tol,
                              max_iter=max_iter)
    for schedule in (1, 2, 3):
        opts = opmm.nm_options(objective=opmm.NM_OBJ_REFERENCE, metric=metric, max_iter=max_iter, tol_x=tol,
                               tol_f=tol, init_scale=scale, schedule=schedule, cpu_check=0)
        res = opmm.opmm_estimate_batch(h, recs, ctls, x0=x0, options=opts)
        for s in range(S):
            r = res[s]
            assert r["x"].tolist() == o["x"][s].tolist(), (seed, schedule, s)
            assert r["f"] == o["f"][s] and (r["iterations"], r["func_evals"], r["exit_reason"]) == \
                   (o["iterations"][s], o["func_evals"][s], o["exit_reason"][s]), (seed, schedule, s)
