"""Equivalence of the library's call paths (-m gpu).

One fit can reach the kernels through several host paths: the synchronous
opmm_fit (CUDA-graph replay for plain fits, plain launches for top-K /
certified fits), opmm_fit_async on device buffers, opmm_fit_batch
(gridDim.y = saccades), and opmm_fit_shard (one rank's share).  The kernels
are the same, so every path must give the same result for the same inputs,
whatever the handle did before.  These tests sweep the option combinations
(precision, metric, top_k, certify, kernel variant, grid tables) over fresh
handles and over handles that just fitted a different trace -- the kind of
cross-call state that hid a stale-trace bug in the plain-launch path of
opmm_fit until round 2.
"""
import ctypes

import numpy as np
import pytest

import oracle
import workloads as W

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


def traces(ctl):
    a = oracle.positions(W.truth_opc(), ctl) + W.noise(ctl.n_steps + 1)
    b = oracle.positions(W.truth_opc(pw_ms=31.0), ctl) + W.noise(ctl.n_steps + 1, seed=99)
    return a, b


def key(r):
    return (r["best_index"], r["opt_err"], r["n_finite"], r["n_evaluated"], r["top_k"], r["certified"],
            tuple(r["topk_index"]), tuple(r["topk_err"]))


def via_async(opmm, h, rec, ctl, sp, n, o):
    out = torch.zeros(ctypes.sizeof(opmm.FitResult), dtype=torch.uint8, device="cuda")
    opmm.opmm_fit_async(h, torch.as_tensor(rec, device="cuda"), ctl, sp, n, out, o)
    torch.cuda.synchronize()
    return opmm.decode_result(bytes(out.cpu().numpy()))


CASES = [
    ("fp64", "paper", dict()),
    ("fp64 rms", "paper", dict(metric=1)),
    ("fp64 top7", "paper", dict(top_k=7)),
    ("fp32", "paper", dict(precision=1)),
    ("fp32 certify", "paper", dict(precision=1, certify=1)),
    ("fp32 certify rms top12", "paper", dict(precision=1, certify=1, metric=1, top_k=12)),
    ("refill", "paper", dict(kernel_variant=5)),
    ("grid tables", "grid", dict(kernel_variant=1)),
    ("grid tables top3", "grid", dict(kernel_variant=1, top_k=3)),
    ("superposition", "grid", dict()),
    ("superposition fp32", "grid", dict(precision=1)),
]


@pytest.mark.parametrize("name,space,kw", CASES, ids=[c[0] for c in CASES])
def test_sync_async_and_history_agree(opmm, name, space, kw):
    """opmm_fit on a fresh handle, opmm_fit right after a fit of another
    trace, opmm_fit_async on device buffers, and opmm_fit without the CUDA
    graph: identical results (winner, counts, top-K list, certificate)."""
    ctl = W.Control()
    a, b = traces(ctl)
    sp = W.paper_space() if space == "paper" else W.g4_space(16)
    n = 60001 if space == "paper" else sp.n_grid()
    o = opmm.fit_options(cpu_check=0, **kw)
    with opmm.opmm_create(0) as h:
        ref = via_async(opmm, h, b, ctl, sp, n, o)
    with opmm.opmm_create(0) as h:
        fresh = opmm.opmm_fit(h, b, ctl, sp, n, o)
    with opmm.opmm_create(0) as h:
        opmm.opmm_fit(h, a, ctl, sp, n, opmm.fit_options(cpu_check=0))              # graph path, trace a
        opmm.opmm_fit(h, a, ctl, sp, n, opmm.fit_options(cpu_check=0, top_k=4))     # plain path, trace a
        after = opmm.opmm_fit(h, b, ctl, sp, n, o)
        nograph = opmm.opmm_fit(h, b, ctl, sp, n, opmm.fit_options(cpu_check=0, flags=opmm.FIT_FLAG_NO_GRAPH,
                                                                    **kw))
        again = via_async(opmm, h, b, ctl, sp, n, o)
    for r in (fresh, after, nograph, again):
        assert key(r) == key(ref), name


@pytest.mark.parametrize("kw", [dict(), dict(top_k=6), dict(precision=1, certify=1)],
                         ids=["plain", "top6", "fp32-certify"])
def test_batch_saccade0_equals_single_fit(opmm, kw):
    """Saccade 0 of opmm_fit_batch (Philox counter word 2 = 0, per-saccade
    amplitude and pw_default from the batch's control table, one slice per
    block) equals opmm_fit of the same trace and control."""
    ctl0 = W.Control(amplitude_deg=12.0, pw_default_ms=35.0)
    a, b = traces(ctl0)
    sp = W.paper_space()
    n = 40000
    ctls = [ctl0, W.Control(amplitude_deg=7.0, pw_default_ms=25.0), W.Control(amplitude_deg=20.0)]
    recs = np.stack([a, b, a])
    o = opmm.fit_options(cpu_check=0, **kw)
    with opmm.opmm_create(0) as h:
        res = opmm.opmm_fit_batch(h, recs, ctls, sp, n, o)
        single = opmm.opmm_fit(h, a, ctl0, sp, n, o)
    assert key(res[0]) == key(single)


def test_workspace_growth_and_reuse(opmm):
    """One handle through fits of growing and shrinking size and changing
    options (its workspaces -- partials, counters, top-K buffers, error
    workspace, staging -- grow and are reused) gives each fit the result a
    fresh handle gives."""
    ctl = W.Control()
    a, b = traces(ctl)
    sp = W.paper_space()
    seq = [(a, 1000, dict()), (b, 200001, dict(top_k=32)), (a, 37, dict(top_k=5)),
           (b, 1000003, dict(precision=1, certify=1)), (a, 1000, dict(top_k=9, metric=1)),
           (b, 5, dict(precision=1, certify=1, top_k=3)), (a, 300000, dict(kernel_variant=5)),
           (b, 1000, dict())]
    with opmm.opmm_create(0) as h:
        got = [opmm.opmm_fit(h, r, ctl, sp, n, opmm.fit_options(cpu_check=0, **kw)) for r, n, kw in seq]
    for (r, n, kw), g in zip(seq, got):
        with opmm.opmm_create(0) as hf:
            ref = opmm.opmm_fit(hf, r, ctl, sp, n, opmm.fit_options(cpu_check=0, **kw))
        assert key(g) == key(ref), (n, kw)


def test_explicit_entry_points_host_equals_device(opmm):
    """opmm_generate / opmm_simulate / opmm_score / opmm_simulate_score with
    host (numpy) buffers give exactly the device-buffer results; a host
    output with a leading dimension larger than n keeps the entries the call
    does not write; opmm_fit_batch and opmm_estimate_batch take device traces
    with the same results as host ones."""
    ctl = W.Control()
    a, b = traces(ctl)
    sp = W.paper_space()
    n, ld = 300, 311
    with opmm.opmm_create(0) as h:
        s = torch.cuda.current_stream()
        opc_d = torch.zeros((18, ld), dtype=torch.float64, device="cuda")
        opmm.opmm_generate(h, sp, 1000, n, opc_d, ld=ld, stream=s)
        opc_h = np.full((18, ld), 7.0)
        opmm.opmm_generate(h, sp, 1000, n, opc_h, ld=ld)
        torch.cuda.synchronize()
        assert np.array_equal(opc_h[:, :n], opc_d.cpu().numpy()[:, :n]) and np.all(opc_h[:, n:] == 7.0)
        tr_d = torch.zeros((101, n), dtype=torch.float64, device="cuda")
        st_d = torch.zeros(n, dtype=torch.uint8, device="cuda")
        opmm.opmm_simulate(h, opc_d, n, ctl, tr_d, ld=ld, status=st_d, stream=s)
        tr_h, st_h = np.zeros((101, n)), np.zeros(n, dtype=np.uint8)
        opmm.opmm_simulate(h, opc_h, n, ctl, tr_h, ld=ld, status=st_h)
        torch.cuda.synchronize()
        assert np.array_equal(tr_h, tr_d.cpu().numpy(), equal_nan=True)
        assert np.array_equal(st_h, st_d.cpu().numpy())
        for metric in (0, 1):
            e_d = torch.zeros(n, dtype=torch.float64, device="cuda")
            opmm.opmm_score(h, tr_d, n, 101, torch.as_tensor(b, device="cuda"), e_d, metric=metric, stream=s)
            e_h = np.zeros(n)
            opmm.opmm_score(h, tr_h, n, 101, b, e_h, metric=metric)
            f_d = torch.zeros(n, dtype=torch.float64, device="cuda")
            opmm.opmm_simulate_score(h, opc_d, n, ctl, torch.as_tensor(b, device="cuda"), f_d, metric=metric,
                                     ld=ld, stream=s)
            f_h = np.zeros(n)
            opmm.opmm_simulate_score(h, opc_h, n, ctl, b, f_h, metric=metric, ld=ld)
            torch.cuda.synchronize()
            assert np.array_equal(e_h, e_d.cpu().numpy(), equal_nan=True)
            assert np.array_equal(f_h, f_d.cpu().numpy(), equal_nan=True)
        recs = np.stack([a, b, b, a])
        ctls = [W.Control(amplitude_deg=10.0 + k) for k in range(4)]
        fh = opmm.opmm_fit_batch(h, recs, ctls, sp, 3000, opmm.fit_options(cpu_check=1))
        fd = opmm.opmm_fit_batch(h, torch.as_tensor(recs, device="cuda"), ctls, sp, 3000,
                                 opmm.fit_options(cpu_check=1))
        assert [key(x) + (x["cpu_check"],) for x in fh] == [key(x) + (x["cpu_check"],) for x in fd]
        o = opmm.nm_options(max_iter=300)
        nh = opmm.opmm_estimate_batch(h, recs, ctls, options=o)
        nd = opmm.opmm_estimate_batch(h, torch.as_tensor(recs, device="cuda"), ctls, options=o)
        for x, y in zip(nh, nd):
            assert np.array_equal(x["x"], y["x"]) and (x["f"], x["iterations"], x["cpu_check"]) == \
                   (y["f"], y["iterations"], y["cpu_check"])


def test_kernel_timing_is_opt_in(opmm):
    """opmm_last_kernel_ms needs opmm_set_kernel_timing: off by default (no
    timing events on the stream), then every entry point's launch is timed,
    the synchronous graph path included; turning it off again drops it."""
    ctl = W.Control()
    a, _ = traces(ctl)
    sp = W.paper_space()
    with opmm.opmm_create(0) as h:
        opmm.opmm_fit(h, a, ctl, sp, 20000)
        with pytest.raises(opmm.OpmmError) as ei:
            opmm.opmm_last_kernel_ms(h)
        assert ei.value.status == opmm.ERR_INVALID_ARG
        opmm.opmm_set_kernel_timing(h, True)
        for o in (opmm.fit_options(), opmm.fit_options(top_k=4), opmm.fit_options(precision=1, certify=1)):
            r = opmm.opmm_fit(h, a, ctl, sp, 20000, o)
            assert opmm.opmm_last_kernel_ms(h) > 0.0 and r["best_index"] >= 0
        via_async(opmm, h, a, ctl, sp, 20000, opmm.fit_options())
        assert opmm.opmm_last_kernel_ms(h) > 0.0
        opmm.opmm_set_kernel_timing(h, False)
        with pytest.raises(opmm.OpmmError):
            opmm.opmm_last_kernel_ms(h)
    with opmm.opmm_create(0, kernel_timing=True) as h:
        opmm.opmm_fit(h, a, ctl, sp, 20000)
        assert opmm.opmm_last_kernel_ms(h) > 0.0
