"""Seeded synthetic workloads shared by tests/, bench.py and smoke().

This module holds NO arithmetic of the method (no plant, integrator, score or
reduction).  It only states data the paper prints (Table 1 / Table 2 defaults),
the search-space bounds read from it, seeds, and numpy random
draws used as inputs (measurement noise, population amplitudes).  Both the CPU
oracle (oracle/) and the CUDA product (paper_2007_09884_b200/) consume these
plain arrays; neither imports the other.

The input recipe is restated in DESIGN.md "Input recipe".
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

NPARAM = 18

#: Table-1 order and shorthand (Table 1).
PARAM_NAMES = (
    "K_SE_AG", "K_SE_ANT", "K_LT_AG", "K_LT_ANT", "B_AG", "B_ANT", "B_P",
    "N_C_AG", "N_C_ANT", "J", "TAU_AC_AG", "TAU_AC_ANT", "TAU_DE_AG",
    "TAU_DE_ANT", "N_C_FIX", "N_SAC_AG", "N_SAC_ANT", "PW",
)
IDX = {n: i for i, n in enumerate(PARAM_NAMES)}

#: Table 1 default values.  PW's default is "saccade
#: duration - 6 ms", i.e. a per-saccade placeholder: NaN here.
TABLE1_DEFAULTS = (
    2.5, 2.5, 1.2, 1.2, 0.046, 0.022, 0.06, 0.8, 0.5, 0.000043,
    11.7, 2.4, 2.0, 1.9, 14.0, 55.0, 0.5, float("nan"),
)

#: Table 2 (9-parameter OPMM) names and defaults.
TABLE2_NAMES = ("K_SE", "K_LT", "B_AG", "B_ANT", "B_P", "N_C_AG", "N_C_ANT", "J", "N_C_FIX")
TABLE2_DEFAULTS = (2.5, 1.2, 0.046, 0.022, 0.06, 0.8, 0.5, 0.000043, 14.0)

#: Fig. 4 result-row column order; differs from Table 1 order.
FIG4_HEADER = ("SacNo,OptErr,CPU_check,SE_ag,SE_ant,LT_ag,LT_ant,PE_ag,PE_ant,Vis,"
               "FV_ag,FV_ant,Inert,Act_ag,Act_ant,Deact_ag,Deact_ant,Step,H_ag,H_ant,W")

SEED_PAPER_SPACE = 9884   # Philox key for S_paper
SEED_NOISE = 2007         # measurement-noise seed
SEED_POPULATION = 5       # population amplitudes / truths


@dataclasses.dataclass
class Control:
    """Pulse-step control + integration grid for one saccade."""
    dt_ms: float = 1.0
    n_steps: int = 100
    amplitude_deg: float = 10.0      # NaN -> rec[n] - rec[0] (D5, Q8)
    theta0_deg: float = 0.0
    pw_default_ms: float = 40.0      # used when a candidate's PW is NaN
    substeps: int = 0                # RK4 steps per sample interval (0 or 1: h = dt), Q25


@dataclasses.dataclass
class SearchSpace:
    """Candidate generator description (SURVEY 8(b) opmm_search_space)."""
    mode: int                      # 0 = Philox random, 1 = grid
    seed: int
    lo: np.ndarray                 # [18] float64
    hi: np.ndarray                 # [18] float64
    log_scale: np.ndarray          # [18] uint8
    levels: np.ndarray             # [18] int32 (grid mode; product = N)
    model: int = 0                 # 0 = 18-parameter (Table 1), 1 = 9-parameter (Table 2, D7)

    def n_grid(self) -> int:
        return int(np.prod(self.levels.astype(np.int64)))


def truth_opc(pw_ms: float = 40.0) -> np.ndarray:
    """TRUTH = Table 1 defaults with PW = 40 ms (46 ms saccade - 6 ms)."""
    v = np.array(TABLE1_DEFAULTS, dtype=np.float64)
    v[IDX["PW"]] = pw_ms
    return v


def paper_space(n_steps: int = 100, dt_ms: float = 1.0, seed: int = SEED_PAPER_SPACE) -> SearchSpace:
    """S_paper (Q14): log-uniform [0.1x, 10x] of Table 1 for the 17 non-PW
    parameters; PW linear-uniform [dt, n_steps*dt]."""
    d = np.array(TABLE1_DEFAULTS, dtype=np.float64)
    lo = d * 0.1
    hi = d * 10.0
    log_scale = np.ones(NPARAM, dtype=np.uint8)
    lo[IDX["PW"]] = dt_ms
    hi[IDX["PW"]] = n_steps * dt_ms
    log_scale[IDX["PW"]] = 0
    return SearchSpace(0, seed, lo, hi, log_scale, np.ones(NPARAM, dtype=np.int32))


def grid_space(dims: dict, base: np.ndarray | None = None) -> SearchSpace:
    """Grid search space.  dims maps parameter name -> (lo, hi, levels, log).
    All other dimensions are fixed at `base` (default TRUTH)."""
    b = truth_opc() if base is None else np.asarray(base, dtype=np.float64)
    lo = b.copy()
    hi = b.copy()
    log_scale = np.zeros(NPARAM, dtype=np.uint8)
    levels = np.ones(NPARAM, dtype=np.int32)
    for name, (l, h, n, lg) in dims.items():
        i = IDX[name]
        lo[i], hi[i], levels[i], log_scale[i] = l, h, n, 1 if lg else 0
    return SearchSpace(1, 0, lo, hi, log_scale, levels)


def g4_space(per_dim: int = 100) -> SearchSpace:
    """G4 planted grid: K_SE_AG, B_AG, N_SAC_AG at
    default*1.01^(j-c), j = 0..per_dim-1, c = per_dim//2; PW integer ms j+1."""
    d = truth_opc()
    c = per_dim // 2
    dims = {}
    for name in ("K_SE_AG", "B_AG", "N_SAC_AG"):
        v = d[IDX[name]]
        dims[name] = (v * 1.01 ** (-c), v * 1.01 ** (per_dim - 1 - c), per_dim, True)
    dims["PW"] = (1.0, float(per_dim), per_dim, False)
    return grid_space(dims)


def g4_planted_index(per_dim: int = 100, pw_ms: int = 40) -> int:
    """Mixed-radix index (dimension 0 fastest) of the TRUTH node of g4_space."""
    c = per_dim // 2
    return c + per_dim * c + per_dim ** 2 * c + per_dim ** 3 * (pw_ms - 1)


def noise(n: int, sigma: float = 0.02, seed: int = SEED_NOISE) -> np.ndarray:
    """i.i.d. N(0, sigma^2) measurement noise in degrees (EyeLink-class; invented)."""
    return np.random.default_rng(seed).normal(0.0, sigma, size=n)


def population(S: int, seed: int = SEED_POPULATION):
    """Population batch recipe: amplitudes U[5, 30] deg,
    duration D = 2.2 A + 21 ms (main-sequence rule, invented), PW = D - 6 ms,
    truths = Table 1 defaults with log-uniform +-20% on K_SE_AG, B_AG, N_SAC_AG
    (SPEC.md:553 set).  Returns (amplitudes[S], pw[S], truths[S, 18])."""
    rng = np.random.default_rng(seed)
    amp = rng.uniform(5.0, 30.0, size=S)
    dur = 2.2 * amp + 21.0
    pw = dur - 6.0
    truths = np.tile(np.array(TABLE1_DEFAULTS, dtype=np.float64), (S, 1))
    truths[:, IDX["PW"]] = pw
    for name in ("K_SE_AG", "B_AG", "N_SAC_AG"):
        f = np.exp(rng.uniform(math.log(0.8), math.log(1.2), size=S))
        truths[:, IDX[name]] *= f
    return amp, pw, truths


# 9-parameter OPMM (Table 2) in the 18-vector slots: the free
# parameters K_SE (slot K_SE_AG), K_LT (slot K_LT_AG), B_AG, B_ANT, B_P,
# N_C_AG, N_C_ANT, J, N_C_FIX; the others are set by the D7 expansion.
NINE_SLOTS = ("K_SE_AG", "K_LT_AG", "B_AG", "B_ANT", "B_P", "N_C_AG", "N_C_ANT", "J", "N_C_FIX")


def paper_space_9(seed: int = SEED_PAPER_SPACE) -> SearchSpace:
    """S_paper for the 9-parameter model: log-uniform [0.1x, 10x] of Table 2
    over the 9 free parameters; all other slots fixed (the generator's D7
    expansion overwrites them)."""
    lo = np.ones(NPARAM)
    hi = np.ones(NPARAM)
    log_scale = np.zeros(NPARAM, dtype=np.uint8)
    for name, d in zip(NINE_SLOTS, TABLE2_DEFAULTS):
        i = IDX[name]
        lo[i], hi[i], log_scale[i] = 0.1 * d, 10.0 * d, 1
    return SearchSpace(0, seed, lo, hi, log_scale, np.ones(NPARAM, dtype=np.int32), model=1)
