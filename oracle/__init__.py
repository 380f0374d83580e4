"""CPU oracle for the OPMM candidate-sweep hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product (paper_2007_09884_b200)
never imports it, and it imports nothing from the product: the two share no
code.  Shared inputs come from the arithmetic-free `workloads` module.

The arithmetic lives in opmm_oracle.c (plain C99, fp64, -ffp-contract=off),
one function per step of the method, each citing PAPER.md / SPEC.md; this file
is ctypes marshalling only.  See that file's header for citations.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "opmm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
NPARAM = 18
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c99", "-fopenmp", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (building the checker is not using it)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        dp = C.POINTER(C.c_double)
        u8p = C.POINTER(C.c_uint8)
        i32p = C.POINTER(C.c_int32)
        i64p = C.POINTER(C.c_int64)
        u32p = C.POINTER(C.c_uint32)
        L.orc_philox4x32_10.argtypes = [u32p, u32p, u32p]
        L.orc_philox4x32_10.restype = None
        L.orc_generate.argtypes = [C.c_int, C.c_int, C.c_uint64, dp, dp, u8p, i32p, C.c_uint32,
                                   C.c_int64, dp]
        L.orc_generate.restype = C.c_int
        L.orc_physical_penalty.argtypes = [dp]
        L.orc_physical_penalty.restype = C.c_double
        L.orc_rhs.argtypes = [dp, dp, C.c_double, C.c_double, C.c_double, C.c_double, dp]
        L.orc_rhs.restype = None
        L.orc_equilibrium.argtypes = [dp, C.c_double, C.c_double, dp]
        L.orc_equilibrium.restype = None
        L.orc_step_levels.argtypes = [dp, C.c_double, dp]
        L.orc_step_levels.restype = None
        L.orc_n_pulse.argtypes = [C.c_double, C.c_double]
        L.orc_n_pulse.restype = C.c_int64
        L.orc_simulate.argtypes = [dp, C.c_double, C.c_int32, C.c_double, C.c_double, dp, dp]
        L.orc_simulate.restype = C.c_int
        L.orc_simulate_sub.argtypes = [dp, C.c_double, C.c_int32, C.c_int32, C.c_double, C.c_double,
                                       dp, dp]
        L.orc_simulate_sub.restype = C.c_int
        L.orc_relativize.argtypes = [dp, C.c_int32, C.c_double, dp, dp, dp]
        L.orc_relativize.restype = None
        L.orc_score.argtypes = [dp, dp, C.c_int32, C.c_int]
        L.orc_score.restype = C.c_double
        L.orc_objective.argtypes = [dp, dp, C.c_int32, C.c_double, C.c_double, C.c_double, C.c_int, dp]
        L.orc_objective.restype = C.c_double
        L.orc_objective_sub.argtypes = [dp, dp, C.c_int32, C.c_double, C.c_int32, C.c_double,
                                        C.c_double, C.c_int, dp]
        L.orc_objective_sub.restype = C.c_double
        L.orc_fit.argtypes = [dp, C.c_int32, C.c_double, C.c_int32, C.c_double, C.c_double, C.c_int, C.c_int,
                              C.c_int, C.c_uint64, dp, dp, u8p, i32p, C.c_uint32, C.c_int64,
                              C.c_int64, C.c_int, dp, i64p, dp, dp]
        L.orc_expand_9param.argtypes = [dp]
        L.orc_expand_9param.restype = None
        L.orc_fit.restype = C.c_int64
        L.orc_objective_batch.argtypes = [dp, C.c_int64, C.c_int64, dp, C.c_int32, C.c_double, C.c_int32,
                                          C.c_double, C.c_double, C.c_int, C.c_int, dp]
        L.orc_objective_batch.restype = None
        L.orc_max_threads.argtypes = []
        L.orc_max_threads.restype = C.c_int
        ip = C.POINTER(C.c_int)
        L.orc_nm_test.argtypes = [C.c_int, C.c_int, dp, C.c_double, C.c_double, C.c_double, C.c_int,
                                  dp, dp, ip, ip, ip]
        L.orc_nm_test.restype = C.c_int
        L.orc_test_fn.argtypes = [C.c_int, C.c_int, dp]
        L.orc_test_fn.restype = C.c_double
        L.orc_estimate_batch.argtypes = [dp, C.c_int64, C.c_int32, C.c_double, C.c_int32, dp, dp, dp, C.c_int,
                                         C.c_double, C.c_double, C.c_double, C.c_int, C.c_int,
                                         dp, dp, i32p, i32p, i32p]
        L.orc_estimate_batch.restype = C.c_int
        _lib = L
    return _lib


def _d(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(C.POINTER(C.c_double))


def _space_args(space):
    lo, plo = _d(space.lo)
    hi, phi = _d(space.hi)
    ls = np.ascontiguousarray(space.log_scale, dtype=np.uint8)
    lv = np.ascontiguousarray(space.levels, dtype=np.int32)
    keep = (lo, hi, ls, lv)
    return keep, (int(space.mode), int(getattr(space, "model", 0)), C.c_uint64(int(space.seed)), plo, phi,
                  ls.ctypes.data_as(C.POINTER(C.c_uint8)), lv.ctypes.data_as(C.POINTER(C.c_int32)))


def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    p = C.POINTER(C.c_uint32)
    lib().orc_philox4x32_10(c.ctypes.data_as(p), k.ctypes.data_as(p), out.ctypes.data_as(p))
    return out


def generate(space, index: int, saccade: int = 0) -> np.ndarray:
    keep, sa = _space_args(space)
    out = np.zeros(NPARAM)
    rc = lib().orc_generate(*sa, C.c_uint32(saccade), C.c_int64(index),
                            out.ctypes.data_as(C.POINTER(C.c_double)))
    if rc != 0:
        raise ValueError("orc_generate failed")
    return out


def generate_batch(space, begin: int, count: int, saccade: int = 0) -> np.ndarray:
    """[count, 18] candidates, row i = gen(begin + i)."""
    return np.stack([generate(space, begin + i, saccade) for i in range(count)]) if count else np.zeros((0, NPARAM))


def expand_9param(p9_in_18) -> np.ndarray:
    """SPEC D7 expansion of a 9-parameter OPC held in the 18-vector slots."""
    a = np.array(p9_in_18, dtype=np.float64)
    lib().orc_expand_9param(a.ctypes.data_as(C.POINTER(C.c_double)))
    return a


def physical_penalty(opc) -> float:
    return lib().orc_physical_penalty(_d(opc)[1])


def rhs(opc, y, n_ag, n_ant, tau_ag_ms, tau_ant_ms) -> np.ndarray:
    o, po = _d(opc)
    yy, py = _d(y)
    dy = np.zeros(6)
    lib().orc_rhs(po, py, n_ag, n_ant, tau_ag_ms, tau_ant_ms, dy.ctypes.data_as(C.POINTER(C.c_double)))
    return dy


def equilibrium(opc, n_ag, n_ant) -> np.ndarray:
    o, po = _d(opc)
    y = np.zeros(6)
    lib().orc_equilibrium(po, n_ag, n_ant, y.ctypes.data_as(C.POINTER(C.c_double)))
    return y


def step_levels(opc, Aprime) -> np.ndarray:
    o, po = _d(opc)
    out = np.zeros(2)
    lib().orc_step_levels(po, Aprime, out.ctypes.data_as(C.POINTER(C.c_double)))
    return out


def n_pulse(pw_ms, dt_ms) -> int:
    return int(lib().orc_n_pulse(pw_ms, dt_ms))


def _sub(ctl) -> int:
    """RK4 substeps per sample interval of a Control (0 or 1: none)."""
    return int(getattr(ctl, "substeps", 0) or 0)


def simulate(opc, dt_ms: float, n_steps: int, Aprime: float, pw_default_ms: float = 40.0,
             states: bool = False, substeps: int = 1):
    """Delta-theta trajectory [n_steps+1] (and states [n_steps+1, 6] if asked);
    substeps > 1 integrates each sample interval with that many RK4 steps."""
    o, po = _d(opc)
    dth = np.zeros(n_steps + 1)
    st = np.zeros((n_steps + 1, 6)) if states else None
    rc = lib().orc_simulate_sub(po, dt_ms, n_steps, substeps, Aprime, pw_default_ms,
                                dth.ctypes.data_as(C.POINTER(C.c_double)),
                                st.ctypes.data_as(C.POINTER(C.c_double)) if states else None)
    if rc != 0:
        raise ValueError("non-physical OPC")
    return (dth, st) if states else dth


def positions(opc, ctl) -> np.ndarray:
    """Absolute positions theta0 + s * Delta-theta (D6 mirroring, Q7)."""
    A = ctl.amplitude_deg
    s = -1.0 if A < 0 else 1.0
    dth = simulate(opc, ctl.dt_ms, ctl.n_steps, abs(A), ctl.pw_default_ms, substeps=max(_sub(ctl), 1))
    return ctl.theta0_deg + s * dth


def relativize(rec, amplitude: float):
    r, pr = _d(rec)
    rel = np.zeros(len(r))
    s = C.c_double()
    Ap = C.c_double()
    lib().orc_relativize(pr, len(r), amplitude, rel.ctypes.data_as(C.POINTER(C.c_double)),
                         C.byref(s), C.byref(Ap))
    return rel, s.value, Ap.value


def score(dtheta, rel, metric: int = 0) -> float:
    a, pa = _d(dtheta)
    b, pb = _d(rel)
    return lib().orc_score(pa, pb, len(a), metric)


def objective(opc, rec, ctl, metric: int = 0) -> float:
    rel, s, Ap = relativize(rec, ctl.amplitude_deg)
    o, po = _d(opc)
    rr, prr = _d(rel)
    buf = np.zeros(ctl.n_steps + 1)
    return lib().orc_objective_sub(po, prr, ctl.n_steps, ctl.dt_ms, _sub(ctl), Ap, ctl.pw_default_ms,
                                   metric, buf.ctypes.data_as(C.POINTER(C.c_double)))


def fit(rec, ctl, space, begin: int, end: int, metric: int = 0, saccade: int = 0,
        nthreads: int = 1, want_err: bool = False):
    """Exhaustive argmin over candidate indices [begin, end).  Returns dict with
    best_index (-1 if no finite), best_err, opc, n_finite, err (optional)."""
    r, pr = _d(rec)
    assert len(r) == ctl.n_steps + 1
    keep, sa = _space_args(space)
    err = np.zeros(max(end - begin, 0)) if want_err else None
    bi = C.c_int64()
    be = C.c_double()
    opc = np.zeros(NPARAM)
    nf = lib().orc_fit(pr, ctl.n_steps, ctl.dt_ms, _sub(ctl), ctl.amplitude_deg, ctl.pw_default_ms, metric,
                       *sa, C.c_uint32(saccade), begin, end, nthreads,
                       err.ctypes.data_as(C.POINTER(C.c_double)) if want_err else None,
                       C.byref(bi), C.byref(be), opc.ctypes.data_as(C.POINTER(C.c_double)))
    out = {"best_index": bi.value, "best_err": be.value, "opc": opc, "n_finite": nf}
    if want_err:
        out["err"] = err
    return out


def objective_batch(opc_soa, rec, ctl, metric: int = 0, nthreads: int = 1) -> np.ndarray:
    """E of every column of an explicit SoA batch opc_soa [18, n] (e.g. a
    generator dump): the per-candidate step of fit() on supplied inputs."""
    o = np.ascontiguousarray(opc_soa, dtype=np.float64)
    assert o.shape[0] == NPARAM
    n = o.shape[1]
    r, pr = _d(rec)
    assert len(r) == ctl.n_steps + 1
    err = np.zeros(n)
    lib().orc_objective_batch(o.ctypes.data_as(C.POINTER(C.c_double)), n, n, pr, ctl.n_steps, ctl.dt_ms,
                              _sub(ctl), ctl.amplitude_deg, ctl.pw_default_ms, metric, nthreads,
                              err.ctypes.data_as(C.POINTER(C.c_double)))
    return err


def max_threads() -> int:
    return lib().orc_max_threads()


# ---------------------------------------------------------------- Nelder-Mead
NM_SPHERE, NM_ROSENBROCK, NM_POWELL = 0, 1, 2


def nm_test(fn_id: int, x0, init_scale=0.05, tol_x=1e-4, tol_f=1e-4, max_iter=None) -> dict:
    """Serial Lagarias Nelder-Mead on a test function (SPEC acceptance 3)."""
    x, px = _d(x0)
    n = len(x)
    xb = np.zeros(n)
    fb, it, ev, why = C.c_double(), C.c_int(), C.c_int(), C.c_int()
    lib().orc_nm_test(fn_id, n, px, init_scale, tol_x, tol_f, 200 * n if max_iter is None else max_iter,
                      xb.ctypes.data_as(C.POINTER(C.c_double)), C.byref(fb), C.byref(it), C.byref(ev),
                      C.byref(why))
    return {"x": xb, "f": fb.value, "iterations": it.value, "func_evals": ev.value, "exit_reason": why.value}


def test_fn(fn_id: int, x) -> float:
    xx, px = _d(x)
    return lib().orc_test_fn(fn_id, len(xx), px)


def estimate_batch(recs, ctls, x0=None, metric=0, init_scale=0.05, tol_x=1e-4, tol_f=1e-4,
                   max_iter=None, nthreads=1) -> dict:
    """Nelder-Mead OPC estimation of S saccades (SPEC estimate_batch), each
    from x0 (default Table 1 with PW NaN -> the saccade's pw_default)."""
    recs = np.ascontiguousarray(recs, dtype=np.float64)
    S, ns = recs.shape
    c0 = ctls[0]
    assert ns == c0.n_steps + 1
    amp = np.array([c.amplitude_deg for c in ctls], dtype=np.float64)
    pwd = np.array([c.pw_default_ms for c in ctls], dtype=np.float64)
    if x0 is None:
        from workloads import TABLE1_DEFAULTS
        x0 = np.array(TABLE1_DEFAULTS, dtype=np.float64)
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    xb = np.zeros((S, NPARAM))
    fb = np.zeros(S)
    it = np.zeros(S, dtype=np.int32)
    ev = np.zeros(S, dtype=np.int32)
    why = np.zeros(S, dtype=np.int32)
    P = C.POINTER(C.c_double)
    I32 = C.POINTER(C.c_int32)
    assert all(_sub(c) == _sub(c0) for c in ctls)
    lib().orc_estimate_batch(recs.ctypes.data_as(P), S, c0.n_steps, c0.dt_ms, _sub(c0), amp.ctypes.data_as(P),
                             pwd.ctypes.data_as(P), x0.ctypes.data_as(P), metric, init_scale, tol_x,
                             tol_f, 200 * NPARAM if max_iter is None else max_iter, nthreads,
                             xb.ctypes.data_as(P), fb.ctypes.data_as(P), it.ctypes.data_as(I32),
                             ev.ctypes.data_as(I32), why.ctypes.data_as(I32))
    return {"x": xb, "f": fb, "iterations": it, "func_evals": ev, "exit_reason": why}
