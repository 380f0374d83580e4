"""Front end and reporting around the fit: saccade detection
in a recorded eye-position trace (I-VT), the per-saccade fit inputs, and the
paper's result table (Fig. 4).  Host-side plumbing in numpy -- no method
arithmetic: every candidate evaluation runs in libopmm's kernels.

* I-VT: a sample belongs to a saccade when its angular
  velocity exceeds a threshold; runs of such samples are saccades.  The paper
  gives no threshold or velocity filter: 30 deg/s on a 5-point central
  difference by default (reading Q26).  Saccades with amplitude < 4 deg or duration < 6 ms are
  discarded (whose "4 deg/s amplitude" is read as 4 deg, Q17).
* Fit inputs: each saccade's trace starts at its onset sample and spans a
  fixed window of n_steps + 1 samples (so a population shares n_steps, as
  opmm_fit_batch requires); amplitude = the detected end-point displacement;
  the default pulse width is "saccade duration - 6 ms".
* Fig. 4: one CSV row per saccade, columns SacNo, OptErr
  (the fit's error), CPU_check (its serial re-score), then the OPC in the
  figure's order, which differs from Table 1's (mapping below, from the
  column descriptions at PAPER.md:352 and the Table 1 names).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

#: Fig. 4 header, byte for byte.
FIG4_HEADER = ("SacNo,OptErr,CPU_check,SE_ag,SE_ant,LT_ag,LT_ant,PE_ag,PE_ant,Vis,FV_ag,FV_ant,"
               "Inert,Act_ag,Act_ant,Deact_ag,Deact_ant,Step,H_ag,H_ant,W")

#: Fig. 4 OPC column -> Table 1 slot (series elasticity K_SE,
#: length-tension K_LT, tension slope N_C, passive viscosity B_P,
#: force-velocity B, inertial mass J, activation / deactivation tau_AC /
#: tau_DE, tension intercept N_C_FIX, pulse height N_SAC, pulse width PW).
FIG4_FROM_TABLE1 = (0, 1, 2, 3, 7, 8, 6, 4, 5, 9, 10, 11, 12, 13, 14, 15, 16, 17)


def fig4_rows(results, first_sacno: int = 1) -> str:
    """Fig. 4 CSV text (header + one row per result).  `results`: dicts with
    opc[18] (Table 1 order), opt_err and cpu_check -- opmm_fit /
    opmm_fit_batch results, or Nelder-Mead results (x, f, cpu_check)."""
    lines = [FIG4_HEADER]
    for k, r in enumerate(results):
        opc = np.asarray(r["opc"] if "opc" in r else r["x"], dtype=np.float64)
        err = r["opt_err"] if "opt_err" in r else r["f"]
        vals = [err, r.get("cpu_check", math.nan)] + [opc[j] for j in FIG4_FROM_TABLE1]
        lines.append(",".join([str(first_sacno + k)] + [f"{v:.6f}" for v in vals]))
    return "\n".join(lines) + "\n"


@dataclasses.dataclass
class Saccade:
    onset: int          # first sample of the saccade
    offset: int         # last sample of the saccade
    amplitude: float    # position[offset] - position[onset], deg
    duration_ms: float  # (offset - onset) * dt


def ivt_saccades(position_deg, dt_ms: float = 1.0, velocity_threshold: float = 30.0,
                 min_amplitude: float = 4.0, min_duration_ms: float = 6.0,
                 velocity_halfwidth: int = 2) -> list[Saccade]:
    """I-VT saccade detection.  The angular velocity of
    sample k is the central difference (x_{k+w} - x_{k-w}) / (2 w dt), w =
    velocity_halfwidth (w = 2 keeps 1 kHz tracker noise of ~0.02 deg well
    below 30 deg/s); a maximal run of samples with |v| > velocity_threshold
    (deg/s) is one saccade, onset = its first sample, offset = its last.
    Returns saccades with |amplitude| >= min_amplitude and duration >=
    min_duration_ms, in time order.  Thresholds: reading Q26."""
    x = np.asarray(position_deg, dtype=np.float64)
    w = max(int(velocity_halfwidth), 1)
    if x.size < 2 * w + 1:
        return []
    v = np.zeros(x.size)
    v[w:-w] = np.abs(x[2 * w:] - x[:-2 * w]) / (2 * w * dt_ms * 1e-3)
    fast = np.concatenate([[False], v > velocity_threshold, [False]])
    edges = np.flatnonzero(fast[1:] != fast[:-1])
    out = []
    for k0, k1 in zip(edges[0::2], edges[1::2]):   # samples k0 .. k1-1 are fast
        onset, offset = int(k0), int(k1) - 1
        amp = float(x[offset] - x[onset])
        dur = (offset - onset) * dt_ms
        if abs(amp) >= min_amplitude and dur >= min_duration_ms:
            out.append(Saccade(onset, offset, amp, dur))
    return out


def fit_inputs(position_deg, saccades, n_steps: int, dt_ms: float = 1.0, control_cls=None):
    """Per-saccade fit inputs: traces [S, n_steps+1] (from each onset) and
    controls (amplitude = detected displacement, pw_default = duration - 6 ms,
    at least dt).  Saccades whose window runs past the recording are dropped;
    returns (traces, controls, kept saccades)."""
    if control_cls is None:
        from .opmm import control as control_cls
    x = np.asarray(position_deg, dtype=np.float64)
    recs, ctls, kept = [], [], []
    for s in saccades:
        if s.onset + n_steps >= x.size:
            continue
        recs.append(x[s.onset:s.onset + n_steps + 1])
        ctls.append(control_cls(dt_ms=dt_ms, n_steps=n_steps, amplitude_deg=s.amplitude,
                                theta0_deg=float(x[s.onset]),
                                pw_default_ms=max(s.duration_ms - 6.0, dt_ms)))
        kept.append(s)
    return (np.array(recs) if recs else np.zeros((0, n_steps + 1))), ctls, kept
