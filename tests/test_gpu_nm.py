"""GPU parity of the batched Nelder-Mead estimator (-m gpu).

Two schedules.  LOCKSTEP (the paper's) evaluates all n + 4
transformation points of an iteration at once, one warp per problem; LANE
runs one problem per lane and evaluates only the points the decision needs.
Both take the serial Lagarias decision, so with the same objective values
their iterates are the serial algorithm's.  With the
reference-order plant objective (explicitly rounded fp64, the RK4
definition's operation order) and on the SPEC test functions the GPU results
are bit-identical to the CPU oracle's serial Nelder-Mead: same best vertex,
same f, same iteration and evaluation counts.
"""
import numpy as np
import pytest

import oracle
import workloads as W

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


SCHEDULES = pytest.mark.parametrize("schedule", [1, 2, 3], ids=["lockstep", "lane", "group"])


@SCHEDULES
def test_rosenbrock_published_run_bit_exact(opmm, h, schedule):
    r = opmm.opmm_nm_minimize_test(h, opmm.NM_ROSENBROCK, [[-1.2, 1.0]],
                                   opmm.nm_options(schedule=schedule))[0]
    o = oracle.nm_test(oracle.NM_ROSENBROCK, [-1.2, 1.0])
    assert (r["iterations"], r["func_evals"]) == (85, 159) == (o["iterations"], o["func_evals"])
    assert r["x"].tolist() == o["x"].tolist() and r["f"] == o["f"]
    # lock-step: every iteration evaluates n + 4 points; lane: only the needed
    # ones; group: the four transformation points (and n per shrink)
    if schedule == 1:
        assert r["gpu_evals"] == 3 + 84 * 6
    elif schedule == 2:
        assert r["gpu_evals"] == 159
    else:
        assert r["gpu_evals"] >= 3 + 84 * 4 and (r["gpu_evals"] - 3 - 84 * 4) % 2 == 0


@SCHEDULES
@pytest.mark.parametrize("fn,dim", [(0, 1), (0, 3), (1, 2), (1, 4), (2, 4), (0, 18), (2, 16)])
def test_test_functions_many_starts_bit_exact(opmm, h, fn, dim, schedule):
    rng = np.random.default_rng(fn * 10 + dim)
    x0 = rng.uniform(-2, 2, size=(40, dim))        # lane: one full warp + a ragged one
    x0[0, 0] = 0.0                                  # zero-coordinate initial step (D9)
    res = opmm.opmm_nm_minimize_test(h, fn, x0, opmm.nm_options(tol_x=1e-7, tol_f=1e-9, max_iter=3000,
                                                                schedule=schedule))
    for s in range(len(x0)):
        o = oracle.nm_test(fn, x0[s], tol_x=1e-7, tol_f=1e-9, max_iter=3000)
        r = res[s]
        assert r["x"].tolist() == o["x"].tolist(), s
        assert (r["f"], r["iterations"], r["func_evals"], r["exit_reason"]) == \
               (o["f"], o["iterations"], o["func_evals"], o["exit_reason"]), s


def _roundtrip_set(S, seed=7, n_steps=100):
    rng = np.random.default_rng(seed)
    ctls, recs, truths = [], [], []
    for s in range(S):
        t = W.truth_opc()
        for name in ("K_SE_AG", "B_AG", "N_SAC_AG", "PW"):
            t[I[name]] *= 1.0 + 0.2 * rng.uniform(-1, 1)
        c = W.Control(n_steps=n_steps, amplitude_deg=float(rng.uniform(5, 15)), pw_default_ms=40.0)
        ctls.append(c)
        recs.append(oracle.positions(t, c) + W.noise(n_steps + 1, seed=100 + s))
        truths.append(t)
    return ctls, np.array(recs), truths


@SCHEDULES
def test_plant_reference_objective_bit_exact_vs_oracle(opmm, h, schedule):
    """Reference-order objective: every saccade's Nelder-Mead run identical to
    the oracle's serial run, bit for bit (x, f, iterations, evaluations)."""
    ctls, recs, _ = _roundtrip_set(6)
    opts = opmm.nm_options(objective=opmm.NM_OBJ_REFERENCE, max_iter=400, schedule=schedule)
    res = opmm.opmm_estimate_batch(h, recs, ctls, options=opts)
    o = oracle.estimate_batch(recs, ctls, max_iter=400)
    for s in range(len(ctls)):
        r = res[s]
        assert r["x"].tolist() == o["x"][s].tolist(), s
        assert r["f"] == o["f"][s]
        assert (r["iterations"], r["func_evals"], r["exit_reason"]) == \
               (o["iterations"][s], o["func_evals"][s], o["exit_reason"][s])
        assert abs(r["cpu_check"] - r["f"]) <= 1e-9 * r["f"]


@SCHEDULES
@pytest.mark.parametrize("precision", [0, 1])
def test_plant_fast_objective_roundtrip(opmm, h, precision, schedule):
    """Propagator objective (the fit path's evaluator): SPEC acceptance 4 --
    per-sample mean residual <= 0.5 deg on >= 90% of round-trip saccades;
    the result's objective agrees with the serial CPU_check re-score."""
    ctls, recs, _ = _roundtrip_set(40, seed=11)
    res = opmm.opmm_estimate_batch(h, recs, ctls,
                                   options=opmm.nm_options(precision=precision, schedule=schedule))
    f = np.array([r["f"] for r in res])
    assert np.mean(f / 101.0 <= 0.5) >= 0.9
    tol = 1e-9 if precision == 0 else 1e-4
    for r, rec, c in zip(res, recs, ctls):
        assert abs(r["cpu_check"] - r["f"]) <= tol * max(r["f"], 1.0)
        assert r["f"] <= oracle.objective(W.truth_opc(), rec, c)   # never worse than the start
        if schedule == 1:
            assert r["gpu_evals"] == 19 + (r["iterations"] - 1) * 22
        elif schedule == 2:
            assert r["gpu_evals"] == r["func_evals"]
        else:
            assert (r["gpu_evals"] - 19 - (r["iterations"] - 1) * 4) % 18 == 0


@pytest.mark.parametrize("precision", [0, 1])
def test_schedules_identical_with_fast_objective(opmm, h, precision):
    """Both schedules run the same evaluator arithmetic and the same serial
    decisions, so with the propagator objective their results are identical
    bit for bit (70 problems: two full warps of the lane schedule and a
    ragged third; 8 full groups-of-8 blocks and a ragged one)."""
    ctls, recs, _ = _roundtrip_set(70, seed=13)   # 70 = 2*32 + 6 = 8*8 + 6
    runs = [opmm.opmm_estimate_batch(h, recs, ctls,
                                     options=opmm.nm_options(precision=precision, schedule=sc,
                                                             cpu_check=0))
            for sc in (1, 2, 3)]
    for s in range(len(ctls)):
        a, b, c = runs[0][s], runs[1][s], runs[2][s]
        for key in ("f", "iterations", "func_evals", "exit_reason"):
            assert a[key] == b[key] == c[key], (s, key)
        assert a["x"].tolist() == b["x"].tolist() == c["x"].tolist(), s
        assert b["gpu_evals"] == b["func_evals"]


def test_auto_schedule_switches_at_1024_problems(opmm, h):
    """AUTO: lock-step below 1024 problems, group from 1024 on (the measured
    crossover); both equal the oracle's serial runs."""
    rng = np.random.default_rng(5)
    x0 = rng.uniform(-2, 2, size=(1024, 3))
    opts = opmm.nm_options(tol_x=1e-7, tol_f=1e-9, max_iter=600)
    small = opmm.opmm_nm_minimize_test(h, opmm.NM_SPHERE, x0[:1023], opts)
    big = opmm.opmm_nm_minimize_test(h, opmm.NM_SPHERE, x0, opts)
    # lock-step: n + 4 points per iteration; group: 4 per iteration + n per shrink
    assert all(r["gpu_evals"] == 4 + (r["iterations"] - 1) * 7 for r in small)
    assert all((r["gpu_evals"] - 4 - (r["iterations"] - 1) * 4) % 3 == 0 for r in big)
    assert any(r["gpu_evals"] != 4 + (r["iterations"] - 1) * 7 for r in big)
    for s in range(0, 1024, 41):
        o = oracle.nm_test(opmm.NM_SPHERE, x0[s], tol_x=1e-7, tol_f=1e-9, max_iter=600)
        assert big[s]["x"].tolist() == o["x"].tolist() and big[s]["f"] == o["f"], s
        assert small[s]["x"].tolist() == o["x"].tolist(), s



def test_schedule_option_validated(opmm, h):
    ctls, recs, _ = _roundtrip_set(1)
    with pytest.raises(opmm.OpmmError):
        opmm.opmm_estimate_batch(h, recs, ctls, options=opmm.nm_options(schedule=4))


@SCHEDULES
def test_long_trace_uses_global_trace_workspace(opmm, h, schedule):
    """Traces too long for the shared-memory copy (here 6000 samples) are
    relativized into a global workspace; the reference-order objective stays
    bit-identical to the oracle's serial Nelder-Mead."""
    ctl = W.Control(n_steps=6000, dt_ms=0.02, amplitude_deg=10.0)
    rec = oracle.positions(W.truth_opc(), ctl) + W.noise(6001)
    opts = opmm.nm_options(objective=opmm.NM_OBJ_REFERENCE, max_iter=15, cpu_check=0, schedule=schedule)
    res = opmm.opmm_estimate_batch(h, rec[None, :], [ctl], options=opts)
    o = oracle.estimate_batch(rec[None, :], [ctl], max_iter=15)
    assert res[0]["x"].tolist() == o["x"][0].tolist() and res[0]["f"] == o["f"][0]
    fast = opmm.opmm_estimate_batch(h, rec[None, :], [ctl],
                                    options=opmm.nm_options(max_iter=15, cpu_check=1, schedule=schedule))
    assert abs(fast[0]["cpu_check"] - fast[0]["f"]) <= 1e-9 * fast[0]["f"]


@SCHEDULES
def test_time_budget_exit(opmm, h, schedule):
    """The paper's time boundary (SPEC D13 time_budget): a
    budget shorter than any iteration stops every problem at its first check
    (iteration 1, after the initial simplex) with exit_reason 2 -- bit-equal
    to the oracle's run cut off by max_iter = 1 -- and a budget no run reaches
    changes nothing."""
    S = 12
    amp, pw, truths = W.population(S)
    ctls = [W.Control(n_steps=150, amplitude_deg=float(amp[s]), pw_default_ms=float(pw[s]))
            for s in range(S)]
    recs = np.array([oracle.positions(truths[s], ctls[s]) + W.noise(151, seed=1000 + s)
                     for s in range(S)])
    base = dict(objective=opmm.NM_OBJ_REFERENCE, max_iter=40, cpu_check=0, schedule=schedule)
    tiny = opmm.opmm_estimate_batch(h, recs, ctls, options=opmm.nm_options(time_budget_ms=1e-9, **base))
    o1 = oracle.estimate_batch(recs, ctls, max_iter=1)
    for s in range(S):
        assert (tiny[s]["iterations"], tiny[s]["exit_reason"]) == (1, 2), s
        assert tiny[s]["x"].tolist() == o1["x"][s].tolist() and tiny[s]["f"] == float(o1["f"][s])
    ref = opmm.opmm_estimate_batch(h, recs, ctls, options=opmm.nm_options(**base))
    big = opmm.opmm_estimate_batch(h, recs, ctls, options=opmm.nm_options(time_budget_ms=1e5, **base))
    for a, b in zip(ref, big):
        assert (a["iterations"], a["exit_reason"], a["f"]) == (b["iterations"], b["exit_reason"], b["f"])
        assert a["x"].tolist() == b["x"].tolist()
    with pytest.raises(opmm.OpmmError):
        opmm.opmm_estimate_batch(h, recs, ctls, options=opmm.nm_options(time_budget_ms=-1.0))


def test_group_schedule_refill_bit_identical(opmm, h):
    """More problems than one wave of group-schedule blocks: the grid is one
    wave and finished groups take the next problem.  Every run must still be
    the oracle's serial run, bit for bit (Rosenbrock, dim 4, seeded starts)."""
    S = 24000
    rng = np.random.default_rng(17)
    x0 = rng.uniform(-2.0, 2.0, size=(S, 4))
    res = opmm.opmm_nm_minimize_test(h, opmm.NM_ROSENBROCK, x0,
                                     opmm.nm_options(schedule=3, max_iter=300))
    for s in range(S):
        o = oracle.nm_test(oracle.NM_ROSENBROCK, x0[s], max_iter=300)
        r = res[s]
        assert (r["iterations"], r["func_evals"], r["exit_reason"]) == \
               (o["iterations"], o["func_evals"], o["exit_reason"]), s
        assert r["x"].tolist() == o["x"].tolist() and r["f"] == o["f"], s
