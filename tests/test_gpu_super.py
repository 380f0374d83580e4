"""GPU parity of the superposition fit kernel (kernel_variant 4; SURVEY 8(f)
f3(ii)) against the CPU oracle (-m gpu).

The kernel scores every level a of one pulse height (N_SAC_AG or N_SAC_ANT)
of a grid node from two integrations, b (height 0) and u (unit pulse):
Delta-theta_k(a) = b_k + a u_k.  The oracle integrates every candidate
directly (PAPER.md:202 exhaustive search), so these tests check the identity
end to end: per-candidate errors within the FP64 budget of the oracle's, the
argmin identical, n_finite / n_evaluated exact, and nodes whose trajectories
blow up handled by the direct evaluator (bit-identical to variant 1).
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


def trace(ctl, noisy=True):
    rec = oracle.positions(W.truth_opc(), ctl)
    return rec + W.noise(ctl.n_steps + 1) if noisy else rec


def fit_with_err(opmm, h, rec, ctl, sp, variant, metric=0):
    n = sp.n_grid()
    err = torch.full((n,), -1.0, dtype=torch.float64, device="cuda")
    r = opmm.opmm_fit(h, rec, ctl, sp, n,
                      opmm.fit_options(metric=metric, err_out=err, kernel_variant=variant))
    return r, err.cpu().numpy()


def check_against_oracle(opmm, h, rec, ctl, sp, metric=0):
    n = sp.n_grid()
    r4, E4 = fit_with_err(opmm, h, rec, ctl, sp, 4, metric)
    r1, E1 = fit_with_err(opmm, h, rec, ctl, sp, 1, metric)
    o = oracle.fit(rec, ctl, sp, 0, n, metric=metric, want_err=True)
    O = o["err"]
    rel, _, _ = oracle.relativize(rec, ctl.amplitude_deg)
    scale = np.abs(rel).sum() if metric == 0 else np.sqrt(np.mean(rel ** 2))
    assert not np.any(E4 == -1.0), "a candidate was not scored"
    assert np.array_equal(np.isinf(E4), np.isinf(O))
    f = np.isfinite(O)
    d = np.abs(E4[f] - O[f]) / np.maximum(O[f], scale)
    assert d.max() <= 1e-9, d.max()
    # against the direct kernel (same propagator, different association)
    d1 = np.abs(E4[f] - E1[f]) / np.maximum(E1[f], scale)
    assert d1.max() <= 1e-11, d1.max()
    assert r4["best_index"] == o["best_index"] == r1["best_index"]
    assert r4["n_finite"] == o["n_finite"] == r1["n_finite"]
    assert r4["n_evaluated"] == n
    assert r4["opc"].tolist() == r1["opc"].tolist()
    assert abs(r4["opt_err"] - o["best_err"]) <= 1e-9 * max(o["best_err"], scale)
    assert abs(r4["cpu_check"] - r4["opt_err"]) <= 1e-9 * max(r4["opt_err"], scale)
    return r4, E4, E1


@pytest.mark.parametrize("metric", [0, 1])
@pytest.mark.parametrize("noisy", [False, True])
def test_super_nsac_ag_grid(opmm, h, metric, noisy):
    """37 N_SAC_AG levels (two ragged register chunks of 19 + 18) x K_SE_AG x
    B_AG x PW; TRUTH is a node (N_SAC_AG level 18, PW 40 ms)."""
    ctl = W.Control()
    rec = trace(ctl, noisy)
    d = W.truth_opc()
    sp = W.grid_space({
        "K_SE_AG": (d[I["K_SE_AG"]] / 1.02 ** 2, d[I["K_SE_AG"]] * 1.02 ** 2, 5, True),
        "B_AG": (d[I["B_AG"]] / 1.05, d[I["B_AG"]] * 1.05 ** 2, 4, True),
        "N_SAC_AG": (d[I["N_SAC_AG"]] / 1.01 ** 18, d[I["N_SAC_AG"]] * 1.01 ** 18, 37, True),
        "PW": (30.0, 55.0, 6, False),
    })
    r4, _, _ = check_against_oracle(opmm, h, rec, ctl, sp, metric)
    if not noisy:
        planted = 2 + 5 * (1 + 4 * (18 + 37 * 2))
        assert r4["best_index"] == planted


def test_super_nsac_ant_linear_levels(opmm, h):
    """Superposition over N_SAC_ANT (linear levels from 0, more than one chunk:
    70 levels -> 3 chunks), negative amplitude, odd and even pulse ends."""
    ctl = W.Control(amplitude_deg=-12.0)
    rec = oracle.positions(W.truth_opc(), ctl) + W.noise(ctl.n_steps + 1)
    sp = W.grid_space({
        "N_SAC_ANT": (0.0, 3.45, 70, False),
        "PW": (33.0, 47.0, 15, False),
        "J": (W.truth_opc()[I["J"]] * 0.8, W.truth_opc()[I["J"]] * 1.25, 3, True),
    })
    check_against_oracle(opmm, h, rec, ctl, sp)


def test_super_unstable_nodes_take_the_direct_path(opmm, h):
    """Nodes whose RK4 recurrence blows up (tiny B_AG: stiff, |rho| > 1) are
    scored by the direct evaluator: +inf exactly where the oracle says so and
    the finite ones bit-identical to variant 1."""
    ctl = W.Control()
    rec = trace(ctl)
    d = W.truth_opc()
    sp = W.grid_space({
        "B_AG": (d[I["B_AG"]] * 1e-3, d[I["B_AG"]], 6, True),
        "N_SAC_AG": (20.0, 90.0, 11, False),
        "PW": (35.0, 45.0, 3, False),
    })
    r4, E4, E1 = check_against_oracle(opmm, h, rec, ctl, sp)
    assert np.isinf(E4).any() and np.isfinite(E4).any()
    # the blown-up nodes are evaluated by the same evaluator as variant 1
    n_nodes = sp.n_grid() // 11
    E4n = E4.reshape(3, 11, 6)
    E1n = E1.reshape(3, 11, 6)
    for pw in range(3):
        for b in range(6):
            if np.isinf(E1n[pw, :, b]).any():
                assert np.array_equal(E4n[pw, :, b], E1n[pw, :, b])
    assert n_nodes == 18


def test_super_population_batch(opmm, h):
    """opmm_fit_batch with variant 4: every saccade's winner equals the oracle's."""
    sp = W.g4_space(per_dim=10)
    S = 3
    ctls, recs = [], []
    for s in range(S):
        c = W.Control(amplitude_deg=6.0 + 4.0 * s)
        ctls.append(c)
        recs.append(oracle.positions(W.truth_opc(), c) + W.noise(c.n_steps + 1, seed=100 + s))
    n = sp.n_grid()
    res = opmm.opmm_fit_batch(h, np.array(recs), ctls, sp, n,
                              opmm.fit_options(kernel_variant=4))
    for s in range(S):
        o = oracle.fit(recs[s], ctls[s], sp, 0, n, saccade=s)
        assert res[s]["best_index"] == o["best_index"]
        assert abs(res[s]["opt_err"] - o["best_err"]) <= 1e-9 * max(o["best_err"], 1.0)


def test_super_g4_planted_1e8(opmm, h):
    """G4 (10^8 grid) through the superposition kernel: the
    planted node wins and sampled errors match the oracle."""
    ctl = W.Control()
    rec = trace(ctl, noisy=False)
    sp = W.g4_space(100)
    n = sp.n_grid()
    err = torch.empty(n, dtype=torch.float64, device="cuda")
    r = opmm.opmm_fit(h, rec, ctl, sp, n, opmm.fit_options(err_out=err, kernel_variant=4))
    planted = W.g4_planted_index()
    assert r["best_index"] == planted
    assert r["n_evaluated"] == n
    rel, _, _ = oracle.relativize(rec, ctl.amplitude_deg)
    scale = np.abs(rel).sum()
    assert r["opt_err"] <= 1e-9 * scale
    rng = np.random.default_rng(7)
    idx = np.sort(rng.choice(n, 3000, replace=False))
    E = err[torch.as_tensor(idx, device="cuda")].cpu().numpy()
    O = np.array([oracle.objective(oracle.generate(sp, int(i)), rec, ctl) for i in idx])
    assert np.array_equal(np.isinf(E), np.isinf(O))
    f = np.isfinite(O)
    assert (np.abs(E[f] - O[f]) / np.maximum(O[f], scale)).max() <= 1e-9
    r1 = opmm.opmm_fit(h, rec, ctl, sp, n, opmm.fit_options(kernel_variant=1))
    assert r1["best_index"] == planted and r1["n_finite"] == r["n_finite"]


def test_super_rejects_ineligible(opmm, h):
    ctl = W.Control()
    rec = trace(ctl)
    sp = W.paper_space()          # random mode: no grid levels to superpose
    with pytest.raises(opmm.OpmmError):
        opmm.opmm_fit(h, rec, ctl, sp, 1000, opmm.fit_options(kernel_variant=4))
    g = W.g4_space(per_dim=6)
    with pytest.raises(opmm.OpmmError):   # the literal four-stage integrator is not superposed
        opmm.opmm_fit(h, rec, ctl, g, g.n_grid(),
                      opmm.fit_options(integrator=opmm.INTEG_RK4_STAGES, kernel_variant=4))
    with pytest.raises(opmm.OpmmError):   # nor the certified fp32 fit (fit_kernel's top-8)
        opmm.opmm_fit(h, rec, ctl, g, g.n_grid(),
                      opmm.fit_options(precision=opmm.FP32, certify=1, kernel_variant=4))


def test_super_generic_generator_path(opmm, h):
    """More grid levels than the kernel's shared level tables hold (sum of
    levels > 2048): nodes come from the generic grid generator instead."""
    ctl = W.Control()
    rec = trace(ctl)
    sp = W.grid_space({
        "N_SAC_AG": (40.0, 70.0, 8, False),
        "PW": (20.0, 60.0, 2100, False),
    })
    check_against_oracle(opmm, h, rec, ctl, sp)


def test_super_exact_ties_lowest_index(opmm, h):
    """PW 39.21 / 39.6 / 40 ms share n_pulse = 40: their nodes are computed
    identically, so the errors tie exactly and the lowest index wins (Q12)."""
    ctl = W.Control()
    rec = trace(ctl)
    d = W.truth_opc()
    sp = W.grid_space({"N_SAC_AG": (d[15] * 0.99, d[15] * 1.01, 3, False),
                       "PW": (39.21, 40.0, 3, False)})
    o = oracle.fit(rec, ctl, sp, 0, 9)
    r, E = fit_with_err(opmm, h, rec, ctl, sp, 4)
    assert r["best_index"] == o["best_index"]
    e = E.reshape(3, 3)
    assert np.all(e[0] == e[1]) and np.all(e[1] == e[2])


def test_super_is_the_auto_choice_for_pulse_height_grids(opmm, h):
    """kernel_variant 0 picks the superposition kernel for an eligible grid
    with >= 8 pulse-height levels: identical result to an explicit 4."""
    ctl = W.Control()
    rec = trace(ctl)
    sp = W.g4_space(per_dim=10)
    r0, E0 = fit_with_err(opmm, h, rec, ctl, sp, 0)
    r4, E4 = fit_with_err(opmm, h, rec, ctl, sp, 4)
    assert np.array_equal(E0, E4)
    assert r0["best_index"] == r4["best_index"] and r0["opt_err"] == r4["opt_err"]


def test_super_nccl_single_rank_node_sharding(opmm, h):
    """Variant 4 on an NCCL handle (1-rank communicator): the rank's share is a
    node range, its 32-byte partial goes through ncclAllGather and the merge
    kernel -- same result as the single-GPU handle."""
    import os
    import subprocess
    import sys
    code = r'''
import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import torch, oracle, workloads as W
from paper_2007_09884_b200 import opmm
ctl = W.Control()
rec = oracle.positions(W.truth_opc(), ctl) + W.noise(101)
uid = opmm.opmm_nccl_unique_id()
with opmm.opmm_create_nccl(0, uid, 0, 1) as hn, opmm.opmm_create(0) as hp:
    for per in (6, 20):
        sp = W.g4_space(per)
        n = sp.n_grid()
        o = opmm.fit_options(kernel_variant=4)
        a = opmm.opmm_fit(hn, rec, ctl, sp, n, o)
        b = opmm.opmm_fit(hp, rec, ctl, sp, n, o)
        assert (a["best_index"], a["opt_err"], a["n_finite"], a["n_evaluated"]) == \
               (b["best_index"], b["opt_err"], b["n_finite"], b["n_evaluated"]), (per, a, b)
        assert a["n_evaluated"] == n
        assert a["opc"].tolist() == b["opc"].tolist()
print("nccl-super ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                       timeout=300)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "nccl-super ok" in p.stdout


def test_super_tmem_and_smem_layouts_agree_bitwise(opmm, h):
    """The tensor-memory column layout (TMEM warps + shared-memory warps, one
    block per SM) and the shared-memory-only layout compute every error with
    the same operations in the same order: bit-identical err_out and result.
    The shared-memory layout is forced with OPMM_FIT_FLAG_SUPER_SMEM."""
    ctl = W.Control()
    rec = oracle.positions(W.truth_opc(), ctl) + W.noise(101)
    for sp in (W.g4_space(12), W.g4_space(40)):
        n = sp.n_grid()
        out = []
        for flags in (opmm.FIT_FLAG_SUPER_SMEM, 0):
            err = torch.empty(n, dtype=torch.float64, device="cuda")
            r = opmm.opmm_fit(h, rec, ctl, sp, n, opmm.fit_options(kernel_variant=4, err_out=err,
                                                                   flags=flags))
            out.append((r["best_index"], r["opt_err"], r["n_finite"], err.cpu().numpy()))
        assert out[0][:3] == out[1][:3]
        assert np.array_equal(out[0][3], out[1][3])


@pytest.mark.parametrize("metric", [0, 1])
def test_super_fp32_columns_within_fp32_budget(opmm, h, metric):
    """precision = FP32: b and u are integrated in fp64, stored as fp32
    columns and scored in fp32.  North-star FP32 bar: errors
    within 1e-4 relative of the fp64 oracle's, finite/+inf classification
    identical, and the fp32 winner's fp64 error within 1e-4 of the best."""
    ctl = W.Control()
    rec = trace(ctl)
    d = W.truth_opc()
    sp = W.grid_space({
        "K_SE_AG": (d[I["K_SE_AG"]] / 1.02 ** 2, d[I["K_SE_AG"]] * 1.02 ** 2, 5, True),
        "B_AG": (d[I["B_AG"]] * 1e-3, d[I["B_AG"]] * 1.05 ** 2, 6, True),
        "N_SAC_AG": (d[I["N_SAC_AG"]] / 1.01 ** 18, d[I["N_SAC_AG"]] * 1.01 ** 18, 37, True),
        "PW": (30.0, 55.0, 6, False),
    })
    n = sp.n_grid()
    err = torch.full((n,), -1.0, dtype=torch.float64, device="cuda")
    r = opmm.opmm_fit(h, rec, ctl, sp, n, opmm.fit_options(precision=opmm.FP32, metric=metric,
                                                           err_out=err, kernel_variant=4))
    E = err.cpu().numpy()
    o = oracle.fit(rec, ctl, sp, 0, n, metric=metric, want_err=True)
    O = o["err"]
    rel, _, _ = oracle.relativize(rec, ctl.amplitude_deg)
    scale = np.abs(rel).sum() if metric == 0 else np.sqrt(np.mean(rel ** 2))
    assert np.array_equal(np.isinf(E), np.isinf(O))
    assert np.isinf(E).any()   # the stiff B_AG levels blow up (direct path)
    f = np.isfinite(O)
    assert (np.abs(E[f] - O[f]) / np.maximum(O[f], scale)).max() <= 1e-4
    e64 = O[r["best_index"]]
    assert e64 <= (1 + 1e-4) * o["best_err"] + 1e-4 * scale
    assert r["n_finite"] == o["n_finite"]
