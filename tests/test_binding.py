"""The ctypes binding's batch conversions (CPU): the column-wise paths of
opmm_fit_batch / opmm_estimate_batch give exactly the per-struct dicts."""
import math

import numpy as np
import pytest

import workloads as W


@pytest.fixture(scope="module")
def opmm():
    from paper_2007_09884_b200 import build
    build.build()   # the binding loads libopmm.so at import
    from paper_2007_09884_b200 import opmm as m
    return m


def _same(d1, d2):
    assert d1.keys() == d2.keys()
    for k in d1:
        a, b = d1[k], d2[k]
        if isinstance(a, np.ndarray):
            assert np.array_equal(a, b, equal_nan=True), k
        elif isinstance(a, float) and math.isnan(a):
            assert math.isnan(b), k
        else:
            assert a == b and type(a) is type(b), (k, a, b)


def test_fit_results_match_as_dict(opmm):
    rng = np.random.default_rng(3)
    S = 7
    out = (opmm.FitResult * S)()
    for k in range(S):
        r = out[k]
        r.best_index, r.opt_err, r.cpu_check = int(rng.integers(-1, 10**12)), float(rng.random()), math.nan
        for j in range(18):
            r.opc[j] = float(rng.normal())
        r.n_finite, r.n_evaluated, r.top_k, r.certified = 5 * k, 9 * k, k % 4 * 9 % 33, k % 2
        for j in range(opmm.MAX_TOPK):
            r.topk_index[j], r.topk_err[j] = int(rng.integers(0, 10**9)), float(rng.random())
    for lo, hi in ((0, S), (2, 5), (3, 3)):
        res = opmm._fit_results(out, lo, hi)
        assert len(res) == S
        for k in range(S):
            if lo <= k < hi:
                _same(res[k], out[k].as_dict())
            else:
                assert res[k] is None


def test_nm_results_match_as_dict(opmm):
    rng = np.random.default_rng(4)
    S = 5
    out = (opmm.NmResult * S)()
    for k in range(S):
        r = out[k]
        for j in range(18):
            r.x[j] = float(rng.normal())
        r.f_best, r.cpu_check = float(rng.random()), float(rng.random())
        r.iterations, r.func_evals, r.gpu_evals, r.exit_reason = k, 2 * k, 3 * k, k % 3
    res = opmm._nm_results(out, 1, 4)
    for k in range(S):
        if 1 <= k < 4:
            _same(res[k], out[k].as_dict())
        else:
            assert res[k] is None


def test_control_array_matches_per_struct(opmm):
    ctls = [W.Control(n_steps=150, amplitude_deg=5.0 + k, pw_default_ms=30.0 + k, substeps=k % 3)
            for k in range(9)]
    ref = (opmm.Control * 9)(*[opmm.control(c) for c in ctls])
    assert bytes(opmm._ctl_array(ctls)) == bytes(ref)
    assert bytes(opmm._ctl_array([opmm.control(c) for c in ctls])) == bytes(ref)
    nanc = [W.Control(amplitude_deg=math.nan)]
    assert bytes(opmm._ctl_array(nanc)) == bytes((opmm.Control * 1)(opmm.control(nanc[0])))
