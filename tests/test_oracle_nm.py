"""Pins for the oracle's Nelder-Mead estimator (-m "not gpu").

PAPER.md:243-255 (3.3) and Alg. 1: Lagarias Nelder-Mead,
sorted every iteration, dual tolerance exit (tol_x on coordinates AND tol_f
on values) or max iterations.  Coefficients / initial simplex / defaults are
SPEC D9, D10, D13, D14.
"""
import numpy as np
import pytest

import oracle
import workloads as W
from conftest import read_golden_kv

I = W.IDX


def test_rosenbrock_matches_published_lagarias_fminsearch_run():
    g = read_golden_kv("nelder_mead_rosenbrock.txt")
    r = oracle.nm_test(oracle.NM_ROSENBROCK, [-1.2, 1.0])
    assert r["iterations"] == int(g["iterations"])
    assert r["func_evals"] == int(g["func_evals"])
    assert r["f"] == pytest.approx(g["f_best"], rel=1e-5)
    assert np.all(np.abs(r["x"] - [g["x1"], g["x2"]]) < 1e-4)
    assert r["exit_reason"] == 0 and r["iterations"] <= 400   # SPEC acceptance 3


def test_sphere_and_constant_spec_examples():
    r = oracle.nm_test(oracle.NM_SPHERE, [1.0, 1.0], tol_x=1e-6, tol_f=1e-6)
    assert np.all(np.abs(r["x"]) < 1e-3)
    assert r["exit_reason"] == 0


@pytest.mark.parametrize("fn,x0", [(oracle.NM_SPHERE, [0.7, -0.3, 1.1]),
                                   (oracle.NM_ROSENBROCK, [-1.2, 1.0, 0.5]),
                                   (oracle.NM_POWELL, [3.0, -1.0, 0.0, 1.0])])
def test_converges_on_spec_test_functions(fn, x0):
    """SPEC acceptance 3: dims 2-4 reach the minimum (0 for all three)."""
    r = oracle.nm_test(fn, x0, tol_x=1e-8, tol_f=1e-10, max_iter=20000)
    assert r["f"] < 1e-6
    assert r["exit_reason"] == 0
    # the returned point is the best vertex: f(x_best) == f_best
    assert oracle.test_fn(fn, r["x"]) == r["f"]


def test_zero_coordinate_initial_step_and_max_iter():
    """D9: a zero coordinate gets the absolute step scale * 0.00025; with
    max_iter = 1 the result is the best vertex of the initial simplex."""
    r = oracle.nm_test(oracle.NM_SPHERE, [0.0, 2.0], max_iter=1)
    assert r["iterations"] == 1 and r["func_evals"] == 3 and r["exit_reason"] == 1
    # vertices: (0, 2) f=4, (1.25e-5, 2) f=4+1.5625e-10, (0, 2.1) f=4.41 -> best (0, 2)
    assert r["x"].tolist() == [0.0, 2.0] and r["f"] == 4.0


def test_estimate_roundtrip_and_batch_equals_serial():
    """SPEC acceptance 4 (scaled): saccades generated from the defaults with
    +-20% perturbations on {K_SE_AG, B_AG, N_SAC_AG, PW}, estimated from the
    defaults: per-sample mean residual <= 0.5 deg on >= 90%.  D12: the batch
    result is identical for any thread count."""
    rng = np.random.default_rng(7)
    S = 10
    ctls, recs = [], []
    for s in range(S):
        t = W.truth_opc()
        for name in ("K_SE_AG", "B_AG", "N_SAC_AG", "PW"):
            t[I[name]] *= 1.0 + 0.2 * rng.choice([-1.0, 1.0])
        c = W.Control(pw_default_ms=40.0)
        ctls.append(c)
        recs.append(oracle.positions(t, c))
    recs = np.array(recs)
    r1 = oracle.estimate_batch(recs, ctls, nthreads=1, max_iter=600)
    r4 = oracle.estimate_batch(recs, ctls, nthreads=4, max_iter=600)
    assert np.array_equal(r1["x"], r4["x"]) and np.array_equal(r1["f"], r4["f"])
    per_sample = r1["f"] / 101.0
    assert np.mean(per_sample <= 0.5) >= 0.9
    # objective at the start (defaults) is never beaten by the result's f
    for s in range(S):
        x0 = W.truth_opc()
        e0 = oracle.objective(x0, recs[s], ctls[s])
        assert r1["f"][s] <= e0
        assert oracle.objective(r1["x"][s], recs[s], ctls[s]) == r1["f"][s]
