"""GPU parity at configs[3] scale (-m gpu): random S_paper fits of 10^8 (every
error against a full oracle sweep), 10^9 and 5 * 10^9 (sampled), and the
device generator at candidate indices >= 2^32 (Philox counter word 1 != 0).

configs[3] of BASELINE.json: "large-scale fit: single saccade, 10^8-10^9
candidates"; the exhaustive search is PAPER.md:202 (section 3), the argmin
"sorted for accuracy" PAPER.md:251.  Tolerances as tests/test_gpu_parity.py
(reading Q22 for RK4-unstable candidates).

The 10^8 sweep runs the oracle twice on all host cores:
  regen: the oracle regenerates every candidate itself (glibc exp; log
         dimensions may differ from the device's table exp by <= 2 ulp);
  dump:  the oracle scores the device generator's own values
         (opmm_generate, chunked), so both sides see bit-identical inputs
         and only the arithmetic differs (SURVEY.md:310).
"""
import numpy as np
import pytest

import oracle
import workloads as W
from test_gpu_parity import ULP, assert_fp64_errors, trace

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


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


def dump(opmm, h, sp, begin, count):
    """Device generator values of candidates [begin, begin + count), [18, count]."""
    buf = torch.empty((18, count), dtype=torch.float64, device="cuda")
    opmm.opmm_generate(h, sp, begin, count, buf, stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    return buf.cpu().numpy()


def rel_diff(E, O, scale):
    f = np.isfinite(O)
    d = np.zeros_like(O)
    d[f] = np.abs(E[f] - O[f]) / np.maximum(O[f], scale)
    return d


@pytest.mark.parametrize("begin", [2**32 - 4096, 2**33 + 5, 10**11 + 3])
def test_generate_beyond_2_32(opmm, h, begin):
    """Candidate indices whose Philox counter word 1 (i_hi) is non-zero, and a
    range straddling 2^32: device words equal the oracle's."""
    sp = W.paper_space()
    n = 8192
    g = dump(opmm, h, sp, begin, n).T
    o = np.array([oracle.generate(sp, begin + i) for i in range(n)])
    lin = sp.log_scale == 0
    assert np.array_equal(g[:, lin], o[:, lin])
    assert (np.abs(g[:, ~lin] - o[:, ~lin]) / np.abs(o[:, ~lin])).max() <= 2 * ULP


def test_fit_random_1e8_full_oracle_sweep(opmm, h):
    """configs[3] at 10^8: one random S_paper fit on one GPU (the launch bench
    times), every one of the 10^8 errors against the oracle -- regenerated
    and dump-fed -- with the argmin and n_finite identical."""
    ctl = W.Control()
    rec = trace(ctl)
    sp = W.paper_space()
    n = 10**8
    err = torch.empty(n, dtype=torch.float64, device="cuda")
    r = opmm.opmm_fit(h, rec, ctl, sp, n, opmm.fit_options(err_out=err))
    torch.cuda.synchronize()
    E = err.cpu().numpy()
    del err
    rel, _, _ = oracle.relativize(rec, ctl.amplitude_deg)
    scale = np.abs(rel).sum()
    nt = oracle.max_threads()

    # regen: the oracle's own generator
    o = oracle.fit(rec, ctl, sp, 0, n, nthreads=nt, want_err=True)
    O = o["err"]
    d = rel_diff(E, O, scale)
    st1, st2 = {}, {}
    assert_fp64_errors(E, O, lambda i: oracle.generate(sp, i), rec, ctl, scale, stats=st1)
    assert r["best_index"] == o["best_index"] and r["n_finite"] == o["n_finite"] == int(np.isfinite(E).sum())
    assert abs(r["opt_err"] - o["best_err"]) <= 1e-9 * max(o["best_err"], scale)

    # dump: the oracle scores the device generator's values
    O2 = np.empty(n)
    chunk = 10**7
    for b in range(0, n, chunk):
        c = min(chunk, n - b)
        O2[b:b + c] = oracle.objective_batch(dump(opmm, h, sp, b, c), rec, ctl, nthreads=nt)
    d2 = rel_diff(E, O2, scale)
    assert_fp64_errors(E, O2, lambda i: dump(opmm, h, sp, i, 1)[:, 0], rec, ctl, scale, stats=st2)
    fin = np.isfinite(O2)
    best2 = int(np.flatnonzero(O2 == O2[fin].min())[0])
    assert best2 == r["best_index"] and int(fin.sum()) == r["n_finite"]
    gen_diff = int(np.sum(O != O2))
    print(f"\n1e8 random S_paper: n_finite {o['n_finite']}, best {r['best_index']} E {r['opt_err']:.9f}\n"
          f"  regen: max rel diff {d.max():.3e}, {st1}\n"
          f"  dump:  max rel diff {d2.max():.3e}, {st2}\n"
          f"  oracle regen vs dump: {gen_diff} errors differ (generator ulps), "
          f"max rel {rel_diff(O2, O, scale).max():.3e}")


def _sampled_check(opmm, h, rec, ctl, sp, E_of, idx, scale):
    """Oracle errors of the candidates idx (dump-fed, bit-identical inputs)
    against the GPU's E_of(idx); returns the oracle errors."""
    P = np.stack([dump(opmm, h, sp, int(i), 1)[:, 0] for i in idx], 1)
    O = oracle.objective_batch(P, rec, ctl, nthreads=oracle.max_threads())
    E = E_of(idx)
    assert_fp64_errors(E, O, lambda j: P[:, j], rec, ctl, scale)
    return O


def test_fit_random_1e9_sampled(opmm, h):
    """configs[3] at 10^9: the reduction is checked on the device against the
    full error vector (min, lowest index of the min, n_finite), the winner and
    10^4 random candidates against the oracle, and no sampled candidate beats
    the winner."""
    ctl = W.Control()
    rec = trace(ctl)
    sp = W.paper_space()
    n = 10**9
    err = torch.empty(n, dtype=torch.float64, device="cuda")
    r = opmm.opmm_fit(h, rec, ctl, sp, n, opmm.fit_options(err_out=err))
    torch.cuda.synchronize()
    fin = torch.isfinite(err)
    assert int(fin.sum()) == r["n_finite"]
    emin = float(err[fin].min())
    assert emin == r["opt_err"]
    assert int(torch.nonzero(err == emin)[0, 0]) == r["best_index"]
    rel, _, _ = oracle.relativize(rec, ctl.amplitude_deg)
    scale = np.abs(rel).sum()
    rng = np.random.default_rng(9)
    idx = np.unique(np.concatenate([rng.integers(0, n, 10**4), [r["best_index"]]]))
    O = _sampled_check(opmm, h, rec, ctl, sp,
                       lambda ii: err[torch.as_tensor(ii, device="cuda")].cpu().numpy(), idx, scale)
    f = np.isfinite(O)
    assert np.all(O[f] >= O[idx == r["best_index"]][0])
    w = oracle.objective(oracle.generate(sp, r["best_index"]), rec, ctl)
    assert abs(w - r["opt_err"]) <= 1e-9 * max(w, scale)
    assert abs(r["cpu_check"] - r["opt_err"]) <= 1e-9 * r["opt_err"]
    print(f"\n1e9: best {r['best_index']} E {r['opt_err']:.9f}, n_finite {r['n_finite']}")


def test_fit_random_5e9_indices_beyond_2_32(opmm, h):
    """5 * 10^9 candidates: indices past 2^32 take Philox counter word 1 in the
    fit kernel itself.  The winner (regenerated on the device, and by the
    oracle from its index) and 2000 sampled candidates above 2^32 are checked
    against the oracle; none of them beats the winner."""
    ctl = W.Control()
    rec = trace(ctl)
    sp = W.paper_space()
    n = 5 * 10**9
    r = opmm.opmm_fit(h, rec, ctl, sp, n)
    assert r["n_evaluated"] == n
    o = oracle.generate(sp, r["best_index"])
    assert np.max(np.abs(r["opc"] - o) / np.abs(o)) <= 2 * ULP
    w = oracle.objective(o, rec, ctl)
    rel, _, _ = oracle.relativize(rec, ctl.amplitude_deg)
    scale = np.abs(rel).sum()
    assert abs(w - r["opt_err"]) <= 1e-9 * max(w, scale)
    rng = np.random.default_rng(11)
    idx = rng.integers(2**32, n, 2000)
    O = np.array([oracle.objective(oracle.generate(sp, int(i)), rec, ctl) for i in idx])
    assert np.all(O[np.isfinite(O)] > r["opt_err"] * (1 - 1e-9))
    print(f"\n5e9: best {r['best_index']} E {r['opt_err']:.9f}, n_finite {r['n_finite']}")


def test_population_bench_scale(opmm, h):
    """configs[4] at the bench's population size: 10^4 saccades x 10^5 S_paper
    candidates, n = 150, through opmm_fit_batch (Philox counter word 2 =
    saccade).  Traces are the bench recipe (workloads.population, simulated
    here by the oracle, + N(0, 0.02 deg)).  Every saccade's reduction is
    checked on the device against its full error row (min, lowest index of
    the min, n_finite); every winner is re-scored by the oracle; 8 sampled
    saccades get a full oracle sweep (all 10^5 errors, argmin, n_finite)."""
    S, n_per, n_steps = 10**4, 10**5, 150
    amp, pw, truths = W.population(S)
    ctls = [W.Control(n_steps=n_steps, amplitude_deg=float(a), pw_default_ms=float(p))
            for a, p in zip(amp, pw)]
    recs = np.stack([oracle.positions(truths[k], ctls[k]) for k in range(S)])
    recs += np.random.default_rng(W.SEED_NOISE).normal(0.0, 0.02, size=recs.shape)
    sp = W.paper_space(n_steps=n_steps)
    err = torch.empty((S, n_per), dtype=torch.float64, device="cuda")
    res = opmm.opmm_fit_batch(h, recs, ctls, sp, n_per, opmm.fit_options(err_out=err, cpu_check=0))
    torch.cuda.synchronize()
    fin = torch.isfinite(err)
    nf = fin.sum(1).cpu().numpy()
    emin = torch.where(fin, err, torch.full_like(err, float("inf"))).min(1).values
    first = (err == emin[:, None]).to(torch.int8).argmax(1).cpu().numpy()
    emin = emin.cpu().numpy()
    for k in range(S):
        r = res[k]
        assert r["n_finite"] == nf[k], k
        assert r["opt_err"] == emin[k] and r["best_index"] == first[k], k
        w = oracle.objective(oracle.generate(sp, r["best_index"], saccade=k), recs[k], ctls[k])
        assert abs(w - r["opt_err"]) <= 1e-9 * max(w, 1.0), k
    rng = np.random.default_rng(4)
    stats_all = {}
    for k in sorted(rng.choice(S, 8, replace=False)):
        o = oracle.fit(recs[k], ctls[k], sp, 0, n_per, saccade=int(k), nthreads=oracle.max_threads(),
                       want_err=True)
        assert (res[k]["best_index"], res[k]["n_finite"]) == (o["best_index"], o["n_finite"]), k
        rel, _, _ = oracle.relativize(recs[k], ctls[k].amplitude_deg)
        st = {}
        assert_fp64_errors(err[k].cpu().numpy(), o["err"], lambda i, k=k: oracle.generate(sp, i, saccade=int(k)),
                           recs[k], ctls[k], np.abs(rel).sum(), 0, stats=st)
        for key, v in st.items():
            if isinstance(v, (int, np.integer)):
                stats_all[key] = stats_all.get(key, 0) + int(v)
    print(f"\npopulation 1e4 x 1e5: all winners re-scored, 8 full sweeps, {stats_all}")
