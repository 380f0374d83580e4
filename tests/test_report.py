"""Front end + Fig. 4 report (paper_2007_09884_b200/report.py):
host-side plumbing, tested on CPU against the paper's printed table and
synthetic recordings built from the oracle."""
import os

import numpy as np
import pytest

import oracle
import workloads as W
from paper_2007_09884_b200 import report

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "fig4_example.txt")
I = W.IDX


def _golden_lines():
    return [ln.rstrip("\n") for ln in open(GOLDEN) if not ln.startswith("#")]


def test_fig4_header_byte_exact():
    assert report.FIG4_HEADER == _golden_lines()[0]
    assert report.FIG4_HEADER == W.FIG4_HEADER


def test_fig4_column_mapping_follows_the_paper_descriptions():
    """PAPER.md:352 names each column; the Fig. 4 order differs from Table 1's.
    Rebuilding the paper's two rows from Table-1-ordered OPCs reproduces them
    (to the printed digits; row 1's W is truncated in the source)."""
    names = report.FIG4_HEADER.split(",")[3:]
    want = {"SE_ag": "K_SE_AG", "SE_ant": "K_SE_ANT", "LT_ag": "K_LT_AG", "LT_ant": "K_LT_ANT",
            "PE_ag": "N_C_AG", "PE_ant": "N_C_ANT", "Vis": "B_P", "FV_ag": "B_AG",
            "FV_ant": "B_ANT", "Inert": "J", "Act_ag": "TAU_AC_AG", "Act_ant": "TAU_AC_ANT",
            "Deact_ag": "TAU_DE_AG", "Deact_ant": "TAU_DE_ANT", "Step": "N_C_FIX",
            "H_ag": "N_SAC_AG", "H_ant": "N_SAC_ANT", "W": "PW"}
    assert [W.PARAM_NAMES[j] for j in report.FIG4_FROM_TABLE1] == [want[n] for n in names]
    rows = [ln.split(",") for ln in _golden_lines()[1:]]
    results = []
    for r in rows:
        opc = np.zeros(18)
        for col, j in enumerate(report.FIG4_FROM_TABLE1):
            opc[j] = float(r[3 + col])
        results.append({"opc": opc, "opt_err": float(r[1]), "cpu_check": float(r[2])})
    out = report.fig4_rows(results).splitlines()
    assert out[0] == report.FIG4_HEADER
    for got, ref in zip(out[1:], rows):
        g = got.split(",")
        assert g[0] == ref[0]
        assert np.allclose([float(v) for v in g[1:]], [float(v) for v in ref[1:]], rtol=0, atol=5e-7)
    # Table 1 defaults land in their documented columns
    d = W.truth_opc()
    row = report.fig4_rows([{"opc": d, "opt_err": 0.0, "cpu_check": 0.0}]).splitlines()[1].split(",")
    assert row[3 + names.index("Inert")] == "0.000043" and row[3 + names.index("Step")] == "14.000000"


def _recording(events, fix_ms=150, noise=0.02, seed=3):
    """Fixation / saccade sequence.  A float event is the oracle's TRUTH
    response (100 ms window) of that amplitude from the current position; a
    ("ramp", a) event is a 15 ms raised-cosine jump of a degrees (a small
    saccade the model's fixed 55 g / 40 ms pulse cannot produce)."""
    x = [np.zeros(fix_ms)]
    pos = 0.0
    truth = []
    for ev in events:
        onset = sum(len(a) for a in x) - 1
        if isinstance(ev, tuple):
            amp = ev[1]
            seg = pos + amp * 0.5 * (1 - np.cos(np.linspace(0, np.pi, 16)))
        else:
            amp = ev
            seg = oracle.positions(W.truth_opc(), W.Control(amplitude_deg=amp, theta0_deg=pos))
        x.append(seg[1:])
        pos = seg[-1]
        truth.append((onset, amp))
        x.append(np.full(fix_ms, pos))
    rec = np.concatenate(x)
    return rec + np.random.default_rng(seed).normal(0.0, noise, rec.size), truth


def test_ivt_detects_synthetic_saccades_and_applies_the_filters():
    rec, truth = _recording([10.0, -8.0, ("ramp", 2.0), 12.0, ("ramp", 6.0)])
    sacs = report.ivt_saccades(rec, 1.0)
    # the 2 deg saccade is below the 4 deg amplitude filter
    assert len(report.ivt_saccades(rec, 1.0, min_amplitude=0.0)) == 5
    assert len(sacs) == 4
    for s, (onset, amp) in zip(sacs, [t for t in truth if abs(t[1]) >= 4]):
        assert 0 <= s.onset - onset <= 6   # a velocity threshold fires after the true onset
        assert np.sign(s.amplitude) == np.sign(amp) and abs(s.amplitude - amp) < 0.25 * abs(amp)
        assert s.duration_ms >= 6
    # the duration filter: a 3-sample jump is not a saccade
    step = np.concatenate([np.zeros(50), np.linspace(0, 10, 3), np.full(50, 10.0)])
    assert report.ivt_saccades(step, 1.0) == []
    assert len(report.ivt_saccades(step, 1.0, min_duration_ms=2)) == 1


def test_fit_inputs_windows_and_controls():
    rec, truth = _recording([10.0, -8.0])
    sacs = report.ivt_saccades(rec, 1.0)
    recs, ctls, kept = report.fit_inputs(rec, sacs, n_steps=80)
    assert recs.shape == (2, 81) and len(ctls) == 2
    for r, c, s in zip(recs, ctls, kept):
        assert r[0] == rec[s.onset] and c.n_steps == 80
        assert c.amplitude_deg == s.amplitude and c.pw_default_ms == max(s.duration_ms - 6, 1.0)
    # a saccade too close to the end of the recording is dropped
    assert len(report.fit_inputs(rec[: kept[1].onset + 40], sacs, n_steps=80)[2]) == 1


@pytest.mark.gpu
def test_recording_to_fig4_end_to_end():
    """Recording -> I-VT -> per-saccade windows -> opmm_fit_batch on the GPU ->
    Fig. 4 CSV; every row's OptErr agrees with its CPU_check column."""
    import torch  # noqa: F401
    from paper_2007_09884_b200 import opmm
    rec, _ = _recording([10.0, -8.0, 12.0])
    sacs = report.ivt_saccades(rec, 1.0)
    recs, ctls, kept = report.fit_inputs(rec, sacs, n_steps=90)
    with opmm.opmm_create(0) as h:
        res = opmm.opmm_fit_batch(h, recs, ctls, W.paper_space(n_steps=90), 20000)
    csv = report.fig4_rows(res).splitlines()
    assert csv[0] == report.FIG4_HEADER and len(csv) == 1 + len(kept) == 4
    for line, r in zip(csv[1:], res):
        v = line.split(",")
        assert np.isfinite(float(v[1])) and abs(float(v[1]) - float(v[2])) <= 1e-6 * float(v[1]) + 1e-6
