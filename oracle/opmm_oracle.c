/*
 * opmm_oracle.c -- CPU ORACLE for the OPMM candidate-sweep hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product library (libopmm, paper_2007_09884_b200/) never links, calls
 * or includes anything from here, and nothing here comes from the product:
 * no shared headers, tables, constants or helpers.
 *
 * Plain, slow, obviously-correct scalar C99 in IEEE double, compiled with
 * -O2 -ffp-contract=off (no FMA contraction, no fast-math).  Every function
 * follows the paper (PAPER.md = arXiv 2007.09884 LaTeX source) and, where the
 * paper is silent, the readings Q1..Q20 of SURVEY.md 8(c), restated in
 * DESIGN.md "Readings".  Notation follows the paper's Table 1.
 *
 *   PAPER.md:150-167 (Table 1)  the 18 OPC parameters, Table-1 order.
 *   PAPER.md:106-117 (2.1)      pulse-step neuronal control signal.
 *   PAPER.md:134-139 (Fig. 1)   plant topology; equations = SPEC.md:126 (D1).
 *   PAPER.md:201-204 (3)        exhaustive search over OPC values.
 *   PAPER.md:366     (3.4)      error = absolute difference recorded vs simulated.
 *   PAPER.md:251     (3.3)      solutions sorted for accuracy -> argmin.
 *
 * Parity-pinned by tests/test_oracle_pins.py (P1..P12b of SURVEY 8(c)); the
 * RMS metric option is pinned only by its closed-form special cases.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Table 1 order. */
enum {
  P_KSE_AG = 0, P_KSE_ANT, P_KLT_AG, P_KLT_ANT, P_B_AG, P_B_ANT, P_B_P,
  P_NC_AG, P_NC_ANT, P_J, P_TAU_AC_AG, P_TAU_AC_ANT, P_TAU_DE_AG, P_TAU_DE_ANT,
  P_NC_FIX, P_NSAC_AG, P_NSAC_ANT, P_PW, ORC_NP
};

#define ORC_CAP 1e20         /* Q10: E >= CAP or non-finite  ->  +inf          */
#define ORC_PENALTY 1e10     /* D8: non-physical penalty base    */
#define ORC_NANT_FLOOR 0.01  /* D4: antagonist step floor, g     */

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon et al., SC'11), counter-based generator (Q15).      */
/* ------------------------------------------------------------------------ */
void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2],
                       uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  int r;
  for (r = 0; r < 10; ++r) {
    uint64_t prod0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t prod1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(prod0 >> 32), lo0 = (uint32_t)prod0;
    uint32_t hi1 = (uint32_t)(prod1 >> 32), lo1 = (uint32_t)prod1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* ------------------------------------------------------------------------ */
/* Candidate generator: index i -> OPC vector (Q14/Q15).       */
/*   mode 0 (random): words 4j..4j+3 = Philox(ctr=(i_lo,i_hi,saccade,j),      */
/*     key=(seed_lo,seed_hi)), j = 0..4; u = (w + 0.5) * 2^-32;              */
/*     log dim: lo * exp(u * log(hi/lo)); linear dim: lo + u * (hi - lo);    */
/*     lo == hi: lo.                                                         */
/*   mode 1 (grid): mixed-radix digits of i, dimension 0 fastest;            */
/*     log dim: lo * exp(d * (log(hi/lo) / (L-1)));                           */
/*     linear dim: lo + d * ((hi - lo) / (L-1)); L == 1: lo.                  */
/* ------------------------------------------------------------------------ */
/* 9-parameter OPMM (Table 2) inside the 18-vector, SPEC D7
   (SPEC.md:132): shared K_SE and K_LT (the AG entries), the canonical pulse
   55 / 0.5 g of width "saccade duration - 6 ms" (PW NaN -> pw_default), and
   -- reading Q23 -- the Table 1 activation/deactivation times. */
void orc_expand_9param(double p[ORC_NP]) {
  p[P_KSE_ANT] = p[P_KSE_AG];
  p[P_KLT_ANT] = p[P_KLT_AG];
  p[P_TAU_AC_AG] = 11.7;
  p[P_TAU_AC_ANT] = 2.4;
  p[P_TAU_DE_AG] = 2.0;
  p[P_TAU_DE_ANT] = 1.9;
  p[P_NSAC_AG] = 55.0;
  p[P_NSAC_ANT] = 0.5;
  p[P_PW] = NAN;
}

static int orc_generate18(int mode, uint64_t seed, const double* lo, const double* hi,
                          const uint8_t* log_scale, const int32_t* levels,
                          uint32_t saccade, int64_t index, double out[ORC_NP]);

/* model 0 = 18-parameter OPC (Table 1); model 1 = 9-parameter (Table 2, D7) */
int orc_generate(int mode, int model, uint64_t seed, const double* lo, const double* hi,
                 const uint8_t* log_scale, const int32_t* levels,
                 uint32_t saccade, int64_t index, double out[ORC_NP]) {
  int rc = orc_generate18(mode, seed, lo, hi, log_scale, levels, saccade, index, out);
  if (rc == 0 && model == 1) orc_expand_9param(out);
  return rc;
}

static int orc_generate18(int mode, uint64_t seed, const double* lo, const double* hi,
                          const uint8_t* log_scale, const int32_t* levels,
                          uint32_t saccade, int64_t index, double out[ORC_NP]) {
  int d;
  if (mode == 0) {
    uint32_t words[20];
    uint32_t key[2];
    int j;
    key[0] = (uint32_t)(seed & 0xffffffffu);
    key[1] = (uint32_t)(seed >> 32);
    for (j = 0; j < 5; ++j) {
      uint32_t ctr[4];
      ctr[0] = (uint32_t)((uint64_t)index & 0xffffffffu);
      ctr[1] = (uint32_t)((uint64_t)index >> 32);
      ctr[2] = saccade;
      ctr[3] = (uint32_t)j;
      orc_philox4x32_10(ctr, key, &words[4 * j]);
    }
    for (d = 0; d < ORC_NP; ++d) {
      double u = ((double)words[d] + 0.5) * (1.0 / 4294967296.0);
      if (lo[d] == hi[d]) {
        out[d] = lo[d];
      } else if (log_scale[d]) {
        double L = log(hi[d] / lo[d]);
        out[d] = lo[d] * exp(u * L);
      } else {
        out[d] = lo[d] + u * (hi[d] - lo[d]);
      }
    }
    return 0;
  } else if (mode == 1) {
    int64_t rem = index;
    for (d = 0; d < ORC_NP; ++d) {
      int64_t L = levels[d];
      int64_t digit;
      if (L < 1) return 1;
      digit = rem % L;
      rem = rem / L;
      if (L == 1 || lo[d] == hi[d]) {
        out[d] = lo[d];
      } else if (log_scale[d]) {
        double step = log(hi[d] / lo[d]) / (double)(L - 1);
        out[d] = lo[d] * exp((double)digit * step);
      } else {
        double step = (hi[d] - lo[d]) / (double)(L - 1);
        out[d] = lo[d] + (double)digit * step;
      }
    }
    return 0;
  }
  return 1;
}

/* ------------------------------------------------------------------------ */
/* Physical check (D8 SPEC.md:248, Q13).  Returns 0 if physical, else the    */
/* penalty 1e10 * (1 + sum of violation amounts).                            */
/* ------------------------------------------------------------------------ */
double orc_physical_penalty(const double p[ORC_NP]) {
  /* strictly positive: divisors, series elasticities, PW (NaN PW = default) */
  static const int strict[] = {P_KSE_AG, P_KSE_ANT, P_B_AG, P_B_ANT, P_J,
                               P_TAU_AC_AG, P_TAU_AC_ANT, P_TAU_DE_AG,
                               P_TAU_DE_ANT, P_PW};
  int bad = 0, i;
  double amount = 0.0;
  for (i = 0; i < ORC_NP; ++i) {
    double v = p[i];
    int is_strict = 0, s;
    if (i == P_PW && isnan(v)) continue;
    for (s = 0; s < (int)(sizeof(strict) / sizeof(strict[0])); ++s)
      if (strict[s] == i) is_strict = 1;
    if (!isfinite(v)) { bad = 1; amount += 1.0; continue; }
    if (is_strict ? !(v > 0.0) : !(v >= 0.0)) {
      bad = 1;
      if (v < 0.0) amount += -v;
    }
  }
  if (!bad) {
    /* the static balance needs G > 0 (Statics) */
    double g_ag = p[P_KSE_AG] / (p[P_KLT_AG] + p[P_KSE_AG]);
    double g_ant = p[P_KSE_ANT] / (p[P_KLT_ANT] + p[P_KSE_ANT]);
    double G = g_ag * (p[P_NC_AG] + p[P_KLT_AG]) + g_ant * (p[P_NC_ANT] + p[P_KLT_ANT]);
    if (!(G > 0.0)) bad = 1;
  }
  return bad ? ORC_PENALTY * (1.0 + amount) : 0.0;
}

/* ------------------------------------------------------------------------ */
/* Plant right-hand side, SPEC D1, Fig. 1.  */
/* State y = (theta, omega, x_AG, x_ANT, f_AG, f_ANT); mechanics in seconds  */
/* (theta deg, omega deg/s, forces g, K g/deg, B g.s/deg, J g.s^2/deg);      */
/* tau given in ms and converted (Q2).                                       */
/*   T_m      = K_SE_m (x_m - theta_m),   theta_AG = +theta, theta_ANT = -theta */
/*   B_m x_m' = f_m - N_C_m theta_m - K_LT_m x_m - T_m                        */
/*   f_m'     = (n_m - f_m) / tau_m                                           */
/*   J omega' = T_AG - T_ANT - B_P omega,   theta' = omega                    */
/* ------------------------------------------------------------------------ */
void orc_rhs(const double p[ORC_NP], const double y[6], double n_ag, double n_ant,
             double tau_ag_ms, double tau_ant_ms, double dy[6]) {
  double theta = y[0], omega = y[1], x_ag = y[2], x_ant = y[3], f_ag = y[4], f_ant = y[5];
  double theta_ag = theta, theta_ant = -theta;
  double T_ag = p[P_KSE_AG] * (x_ag - theta_ag);
  double T_ant = p[P_KSE_ANT] * (x_ant - theta_ant);
  double tau_ag = 1e-3 * tau_ag_ms, tau_ant = 1e-3 * tau_ant_ms;
  dy[0] = omega;
  dy[1] = (T_ag - T_ant - p[P_B_P] * omega) / p[P_J];
  dy[2] = (f_ag - p[P_NC_AG] * theta_ag - p[P_KLT_AG] * x_ag - T_ag) / p[P_B_AG];
  dy[3] = (f_ant - p[P_NC_ANT] * theta_ant - p[P_KLT_ANT] * x_ant - T_ant) / p[P_B_ANT];
  dy[4] = (n_ag - f_ag) / tau_ag;
  dy[5] = (n_ant - f_ant) / tau_ant;
}

/* ------------------------------------------------------------------------ */
/* Statics (SURVEY 8(c) "Statics", derived from D1 with all derivatives 0). */
/*   g_m = K_SE_m/(K_LT_m+K_SE_m), Lambda_m = N_C_m + K_LT_m,                 */
/*   G = g_AG Lambda_AG + g_ANT Lambda_ANT,                                   */
/*   theta_ss = (g_AG n_AG - g_ANT n_ANT) / G.                                */
/* Fixation equilibrium (step 4, Q5): n = f = N_C_FIX.                       */
/* ------------------------------------------------------------------------ */
void orc_equilibrium(const double p[ORC_NP], double n_ag, double n_ant, double y[6]) {
  double g_ag = p[P_KSE_AG] / (p[P_KLT_AG] + p[P_KSE_AG]);
  double g_ant = p[P_KSE_ANT] / (p[P_KLT_ANT] + p[P_KSE_ANT]);
  double G = g_ag * (p[P_NC_AG] + p[P_KLT_AG]) + g_ant * (p[P_NC_ANT] + p[P_KLT_ANT]);
  double theta = (g_ag * n_ag - g_ant * n_ant) / G;
  y[0] = theta;
  y[1] = 0.0;
  y[2] = (n_ag - (p[P_NC_AG] - p[P_KSE_AG]) * theta) / (p[P_KLT_AG] + p[P_KSE_AG]);
  y[3] = (n_ant + (p[P_NC_ANT] - p[P_KSE_ANT]) * theta) / (p[P_KLT_ANT] + p[P_KSE_ANT]);
  y[4] = n_ag;
  y[5] = n_ant;
}

/* Post-pulse step levels (D4 generalised, Q4): settle at theta* + A'. */
void orc_step_levels(const double p[ORC_NP], double Aprime, double out[2]) {
  double F = p[P_NC_FIX];
  double g_ag = p[P_KSE_AG] / (p[P_KLT_AG] + p[P_KSE_AG]);
  double g_ant = p[P_KSE_ANT] / (p[P_KLT_ANT] + p[P_KSE_ANT]);
  double G = g_ag * (p[P_NC_AG] + p[P_KLT_AG]) + g_ant * (p[P_NC_ANT] + p[P_KLT_ANT]);
  double delta = G * Aprime / (g_ag + g_ant);
  double n_ag = F + delta, n_ant = F - delta;
  if (n_ant < ORC_NANT_FLOOR) {
    double theta_star = (g_ag * F - g_ant * F) / G;
    n_ant = ORC_NANT_FLOOR;
    n_ag = (G * (theta_star + Aprime) + ORC_NANT_FLOOR * g_ant) / g_ag;
  }
  out[0] = n_ag;
  out[1] = n_ant;
}

/* Pulse window in steps (Q6): onset at step 0, n_pulse = ceil(PW/dt). */
int64_t orc_n_pulse(double pw_ms, double dt_ms) { return (int64_t)ceil(pw_ms / dt_ms); }

/* ------------------------------------------------------------------------ */
/* Simulation (D2 SPEC.md:127): classical RK4, h = dt, control sampled       */
/* zero-order-hold at the start of each step.  Output dtheta[k] = theta_k -  */
/* theta* for k = 0..n_steps (Fig. 1 "Delta theta", Q5).  Optional states    */
/* [(n_steps+1) x 6].  Returns 0, or 1 if the OPC is non-physical.           */
/* ------------------------------------------------------------------------ */
/* Integer substeps (reading Q25): each sample interval */
/* of dt is integrated by `substeps` classical RK4 steps of h = dt/substeps, */
/* the control held (ZOH) over the whole interval; substeps <= 1 is the     */
/* plain h = dt integration above.                                          */
int orc_simulate_sub(const double p_in[ORC_NP], double dt_ms, int32_t n_steps, int32_t substeps,
                     double Aprime, double pw_default_ms, double* dtheta, double* states) {
  double p[ORC_NP];
  double y[6], ystar[6], levels[2];
  int32_t nsub = substeps > 1 ? substeps : 1;
  double h = 1e-3 * dt_ms / (double)nsub;
  int32_t j;
  int64_t n_pulse;
  int32_t k;
  int i;
  memcpy(p, p_in, sizeof(p));
  if (isnan(p[P_PW])) p[P_PW] = pw_default_ms;
  if (orc_physical_penalty(p) != 0.0) return 1;
  orc_equilibrium(p, p[P_NC_FIX], p[P_NC_FIX], ystar);
  orc_step_levels(p, Aprime, levels);
  n_pulse = orc_n_pulse(p[P_PW], dt_ms);
  for (i = 0; i < 6; ++i) y[i] = ystar[i];
  dtheta[0] = y[0] - ystar[0];
  if (states) for (i = 0; i < 6; ++i) states[i] = y[i];
  for (k = 0; k < n_steps; ++k) {
    double n_ag, n_ant, tau_ag, tau_ant;
    double k1[6], k2[6], k3[6], k4[6], yt[6];
    if ((int64_t)k < n_pulse) {
      n_ag = p[P_NSAC_AG]; n_ant = p[P_NSAC_ANT];
      tau_ag = p[P_TAU_AC_AG]; tau_ant = p[P_TAU_AC_ANT];
    } else {
      n_ag = levels[0]; n_ant = levels[1];
      tau_ag = p[P_TAU_DE_AG]; tau_ant = p[P_TAU_DE_ANT];
    }
    for (j = 0; j < nsub; ++j) {
      orc_rhs(p, y, n_ag, n_ant, tau_ag, tau_ant, k1);
      for (i = 0; i < 6; ++i) yt[i] = y[i] + 0.5 * h * k1[i];
      orc_rhs(p, yt, n_ag, n_ant, tau_ag, tau_ant, k2);
      for (i = 0; i < 6; ++i) yt[i] = y[i] + 0.5 * h * k2[i];
      orc_rhs(p, yt, n_ag, n_ant, tau_ag, tau_ant, k3);
      for (i = 0; i < 6; ++i) yt[i] = y[i] + h * k3[i];
      orc_rhs(p, yt, n_ag, n_ant, tau_ag, tau_ant, k4);
      for (i = 0; i < 6; ++i) y[i] = y[i] + h / 6.0 * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);
    }
    dtheta[k + 1] = y[0] - ystar[0];
    if (states) for (i = 0; i < 6; ++i) states[(int64_t)(k + 1) * 6 + i] = y[i];
  }
  return 0;
}

int orc_simulate(const double p_in[ORC_NP], double dt_ms, int32_t n_steps, double Aprime,
                 double pw_default_ms, double* dtheta, double* states) {
  return orc_simulate_sub(p_in, dt_ms, n_steps, 1, Aprime, pw_default_ms, dtheta, states);
}

/* ------------------------------------------------------------------------ */
/* Trace staging (D5/D6 SPEC.md:130-131, Q7/Q8): s = sign(A) (+1 for A=0),   */
/* A' = |A|, rel_k = s (rec_k - rec_0).  A NaN -> A = rec[n] - rec[0].       */
/* ------------------------------------------------------------------------ */
void orc_relativize(const double* rec, int32_t n_samples, double amplitude,
                    double* rel, double* s_out, double* Aprime_out) {
  double A = isnan(amplitude) ? rec[n_samples - 1] - rec[0] : amplitude;
  double s = (A < 0.0) ? -1.0 : 1.0;
  int32_t k;
  for (k = 0; k < n_samples; ++k) rel[k] = s * (rec[k] - rec[0]);
  *s_out = s;
  *Aprime_out = fabs(A);
}

/* Score (Q9): metric 0 = sum_k |dtheta_k - rel_k| (L1, paper  */
/* default); metric 1 = sqrt(sum_k d_k^2 / n_samples) (RMS option).  Q10:    */
/* accumulated value >= 1e20 or non-finite -> +inf.                          */
double orc_score(const double* dtheta, const double* rel, int32_t n_samples, int metric) {
  double acc = 0.0;
  int32_t k;
  for (k = 0; k < n_samples; ++k) {
    double d = dtheta[k] - rel[k];
    if (metric == 0) acc += fabs(d);
    else acc += d * d;
  }
  if (!(acc < ORC_CAP)) return INFINITY;
  return metric == 0 ? acc : sqrt(acc / (double)n_samples);
}

/* Objective of one OPC against a relativized trace: penalty if non-physical, */
/* else simulate + score.  dtheta_buf must hold n_steps+1 doubles.           */
double orc_objective_sub(const double p[ORC_NP], const double* rel, int32_t n_steps,
                         double dt_ms, int32_t substeps, double Aprime, double pw_default_ms,
                         int metric, double* dtheta_buf) {
  double pen;
  double pp[ORC_NP];
  memcpy(pp, p, sizeof(pp));
  if (isnan(pp[P_PW])) pp[P_PW] = pw_default_ms;
  pen = orc_physical_penalty(pp);
  if (pen != 0.0) return pen;
  orc_simulate_sub(pp, dt_ms, n_steps, substeps, Aprime, pw_default_ms, dtheta_buf, NULL);
  return orc_score(dtheta_buf, rel, n_steps + 1, metric);
}

double orc_objective(const double p[ORC_NP], const double* rel, int32_t n_steps,
                     double dt_ms, double Aprime, double pw_default_ms, int metric,
                     double* dtheta_buf) {
  return orc_objective_sub(p, rel, n_steps, dt_ms, 1, Aprime, pw_default_ms, metric, dtheta_buf);
}

/* ------------------------------------------------------------------------ */
/* Fit = exhaustive search over candidate indices [begin,end): */
/* result = lexicographic min over (E_i, i) with +inf never winning (Q12).   */
/* err_out (optional) receives E_i at [i - begin].  nthreads > 1 uses OpenMP  */
/* with contiguous chunks merged lexicographically.  Returns the number of   */
/* finite E_i; *best_index = -1 if none.                                     */
/* ------------------------------------------------------------------------ */
int64_t orc_fit(const double* rec, int32_t n_steps, double dt_ms, int32_t substeps, double amplitude,
                double pw_default_ms, int metric, int mode, int model, uint64_t seed,
                const double* lo, const double* hi, const uint8_t* log_scale,
                const int32_t* levels, uint32_t saccade, int64_t begin, int64_t end,
                int nthreads, double* err_out, int64_t* best_index, double* best_err,
                double best_opc[ORC_NP]) {
  int32_t ns = n_steps + 1;
  double* rel = (double*)malloc(sizeof(double) * (size_t)ns);
  double s, Aprime;
  int64_t n_finite = 0, bi = -1;
  double be = INFINITY;
  orc_relativize(rec, ns, amplitude, rel, &s, &Aprime);
  if (nthreads < 1) nthreads = 1;
#ifdef _OPENMP
#pragma omp parallel num_threads(nthreads) reduction(+ : n_finite)
#endif
  {
    int tid = 0, nt = 1;
    int64_t cb, ce, i, lbi = -1;
    double lbe = INFINITY;
    double* buf = (double*)malloc(sizeof(double) * (size_t)ns);
    double opc[ORC_NP];
#ifdef _OPENMP
    tid = omp_get_thread_num();
    nt = omp_get_num_threads();
#endif
    cb = begin + (end - begin) * tid / nt;
    ce = begin + (end - begin) * (tid + 1) / nt;
    for (i = cb; i < ce; ++i) {
      double e;
      orc_generate(mode, model, seed, lo, hi, log_scale, levels, saccade, i, opc);
      e = orc_objective_sub(opc, rel, n_steps, dt_ms, substeps, Aprime, pw_default_ms, metric, buf);
      if (err_out) err_out[i - begin] = e;
      if (isfinite(e)) n_finite++;
      if (e < lbe) { lbe = e; lbi = i; }
    }
    free(buf);
#ifdef _OPENMP
#pragma omp critical
#endif
    {
      if (lbi >= 0 && (lbe < be || (lbe == be && lbi < bi))) { be = lbe; bi = lbi; }
    }
  }
  free(rel);
  *best_index = bi;
  *best_err = be;
  if (bi >= 0 && best_opc)
    orc_generate(mode, model, seed, lo, hi, log_scale, levels, saccade, bi, best_opc);
  return n_finite;
}

/* ------------------------------------------------------------------------ */
/* Objective of an explicit batch of OPC vectors (SoA opc[d * ld + i]) against */
/* one recorded trace: err_out[i] = orc_objective_sub(opc_i) -- the same      */
/* definition as orc_fit's per-candidate step, with the  */
/* candidates supplied instead of generated (e.g. a generator dump, so that   */
/* both sides score bit-identical inputs).  No reduction.                     */
/* ------------------------------------------------------------------------ */
void orc_objective_batch(const double* opc, int64_t n, int64_t ld, const double* rec,
                         int32_t n_steps, double dt_ms, int32_t substeps, double amplitude,
                         double pw_default_ms, int metric, int nthreads, double* err_out) {
  int32_t ns = n_steps + 1;
  double* rel = (double*)malloc(sizeof(double) * (size_t)ns);
  double s, Aprime;
  int64_t i;
  orc_relativize(rec, ns, amplitude, rel, &s, &Aprime);
  if (nthreads < 1) nthreads = 1;
#ifdef _OPENMP
#pragma omp parallel num_threads(nthreads)
#endif
  {
    double* buf = (double*)malloc(sizeof(double) * (size_t)ns);
    double p[ORC_NP];
    int d;
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
    for (i = 0; i < n; ++i) {
      for (d = 0; d < ORC_NP; ++d) p[d] = opc[(int64_t)d * ld + i];
      err_out[i] = orc_objective_sub(p, rel, n_steps, dt_ms, substeps, Aprime, pw_default_ms,
                                     metric, buf);
    }
    free(buf);
  }
  free(rel);
}

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ======================================================================== */
/* Nelder-Mead estimator: PAPER.md:243-255 (3.3), Alg. 1   */
/* PAPER.md:300-339, "based on a serial implementation by Lagarias"         */
/* (PAPER.md:248).  SPEC D9 (initial simplex), D10 (rho = 1,   */
/* chi = 2, gamma = 0.5, sigma = 0.5), D11 (NaN -> worst),     */
/* D13 (tol_x = tol_f = 1e-4, max_iterations = 200 n), D14     */
/* (stable sort).  Exit when BOTH the max coordinate distance  */
/* of the other vertices to the best <= tol_x AND the max |f_i - f_best| <= */
/* tol_f, or after max_iter iterations.  Plain serial    */
/* Lagarias steps: only the points the decision needs are evaluated.        */
/* ======================================================================== */
typedef double (*orc_objfn)(const double* x, void* ctx);

static void orc_sort_simplex(int n, double* v, double* fv, double* tmp) {
  /* stable insertion sort of n+1 vertices (rows of v, length n) by fv */
  int i, j, k;
  for (i = 1; i <= n; ++i) {
    double f = fv[i];
    for (k = 0; k < n; ++k) tmp[k] = v[i * n + k];
    j = i - 1;
    while (j >= 0 && fv[j] > f) {
      fv[j + 1] = fv[j];
      for (k = 0; k < n; ++k) v[(j + 1) * n + k] = v[j * n + k];
      --j;
    }
    fv[j + 1] = f;
    for (k = 0; k < n; ++k) v[(j + 1) * n + k] = tmp[k];
  }
}

static double orc_nm_eval(orc_objfn f, void* ctx, const double* x) {
  double y = f(x, ctx);
  return isnan(y) ? INFINITY : y; /* D11 */
}

int orc_nelder_mead(orc_objfn f, void* ctx, int n, const double* x0, double init_scale,
                    double tol_x, double tol_f, int max_iter, double* x_best, double* f_best,
                    int* iterations, int* func_evals, int* exit_reason) {
  const double rho = 1.0, chi = 2.0, psi = 0.5, sigma = 0.5;
  double* v = (double*)malloc(sizeof(double) * (size_t)(n + 1) * (size_t)n);
  double* fv = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  double* xbar = (double*)malloc(sizeof(double) * (size_t)n);
  double* xr = (double*)malloc(sizeof(double) * (size_t)n);
  double* xe = (double*)malloc(sizeof(double) * (size_t)n);
  double* tmp = (double*)malloc(sizeof(double) * (size_t)n);
  int i, j, itercount, evals, reason = 1;
  /* initial simplex (D9): vertex 0 = x0; vertex j+1 = x0 with coordinate j
     scaled by (1 + scale), or set to scale * 0.00025 when it is zero */
  for (j = 0; j < n; ++j) v[j] = x0[j];
  fv[0] = orc_nm_eval(f, ctx, v);
  for (i = 1; i <= n; ++i) {
    for (j = 0; j < n; ++j) v[i * n + j] = x0[j];
    if (x0[i - 1] != 0.0) v[i * n + i - 1] = (1.0 + init_scale) * x0[i - 1];
    else v[i * n + i - 1] = init_scale * 0.00025;
    fv[i] = orc_nm_eval(f, ctx, v + i * n);
  }
  orc_sort_simplex(n, v, fv, tmp);
  itercount = 1;
  evals = n + 1;
  while (itercount < max_iter) {
    double dfmax = 0.0, dxmax = 0.0;
    int shrink = 0;
    for (i = 1; i <= n; ++i) {
      double df = fabs(fv[i] - fv[0]);
      if (!(df <= dfmax)) dfmax = df; /* NaN/inf propagate as "not converged" */
      for (j = 0; j < n; ++j) {
        double dx = fabs(v[i * n + j] - v[j]);
        if (dx > dxmax) dxmax = dx;
      }
    }
    if (dfmax <= tol_f && dxmax <= tol_x) { reason = 0; break; }
    /* centroid of the n best vertices */
    for (j = 0; j < n; ++j) {
      double s = 0.0;
      for (i = 0; i < n; ++i) s += v[i * n + j];
      xbar[j] = s / (double)n;
    }
    for (j = 0; j < n; ++j) xr[j] = (1.0 + rho) * xbar[j] - rho * v[n * n + j];
    {
      double fxr = orc_nm_eval(f, ctx, xr);
      evals++;
      if (fxr < fv[0]) {
        double fxe;
        for (j = 0; j < n; ++j) xe[j] = (1.0 + rho * chi) * xbar[j] - rho * chi * v[n * n + j];
        fxe = orc_nm_eval(f, ctx, xe);
        evals++;
        if (fxe < fxr) { for (j = 0; j < n; ++j) v[n * n + j] = xe[j]; fv[n] = fxe; }
        else { for (j = 0; j < n; ++j) v[n * n + j] = xr[j]; fv[n] = fxr; }
      } else if (fxr < fv[n - 1]) {
        for (j = 0; j < n; ++j) v[n * n + j] = xr[j];
        fv[n] = fxr;
      } else if (fxr < fv[n]) { /* outside contraction */
        double fxc;
        for (j = 0; j < n; ++j) xe[j] = (1.0 + psi * rho) * xbar[j] - psi * rho * v[n * n + j];
        fxc = orc_nm_eval(f, ctx, xe);
        evals++;
        if (fxc <= fxr) { for (j = 0; j < n; ++j) v[n * n + j] = xe[j]; fv[n] = fxc; }
        else shrink = 1;
      } else { /* inside contraction */
        double fxcc;
        for (j = 0; j < n; ++j) xe[j] = (1.0 - psi) * xbar[j] + psi * v[n * n + j];
        fxcc = orc_nm_eval(f, ctx, xe);
        evals++;
        if (fxcc < fv[n]) { for (j = 0; j < n; ++j) v[n * n + j] = xe[j]; fv[n] = fxcc; }
        else shrink = 1;
      }
      if (shrink) {
        for (i = 1; i <= n; ++i) {
          for (j = 0; j < n; ++j) v[i * n + j] = v[j] + sigma * (v[i * n + j] - v[j]);
          fv[i] = orc_nm_eval(f, ctx, v + i * n);
        }
        evals += n;
      }
    }
    orc_sort_simplex(n, v, fv, tmp);
    itercount++;
  }
  for (j = 0; j < n; ++j) x_best[j] = v[j];
  *f_best = fv[0];
  *iterations = itercount;
  *func_evals = evals;
  *exit_reason = reason;
  free(v); free(fv); free(xbar); free(xr); free(xe); free(tmp);
  return 0;
}

/* Test objectives (SPEC acceptance 3). */
static double orc_fn_sphere(const double* x, void* ctx) {
  int n = *(const int*)ctx, i;
  double s = 0.0;
  for (i = 0; i < n; ++i) s += x[i] * x[i];
  return s;
}
static double orc_fn_rosenbrock(const double* x, void* ctx) {
  int n = *(const int*)ctx, i;
  double s = 0.0;
  for (i = 0; i + 1 < n; ++i) {
    double a = x[i + 1] - x[i] * x[i], b = 1.0 - x[i];
    s += 100.0 * (a * a) + b * b;
  }
  return s;
}
static double orc_fn_powell(const double* x, void* ctx) {
  int n = *(const int*)ctx, i;
  double s = 0.0;
  for (i = 0; i + 3 < n; i += 4) {
    double a = x[i] + 10.0 * x[i + 1], b = x[i + 2] - x[i + 3];
    double c = x[i + 1] - 2.0 * x[i + 2], d = x[i] - x[i + 3];
    s += a * a + 5.0 * (b * b) + (c * c) * (c * c) + 10.0 * ((d * d) * (d * d));
  }
  return s;
}

int orc_nm_test(int fn_id, int n, const double* x0, double init_scale, double tol_x, double tol_f,
                int max_iter, double* x_best, double* f_best, int* iterations, int* func_evals,
                int* exit_reason) {
  orc_objfn f = fn_id == 0 ? orc_fn_sphere : fn_id == 1 ? orc_fn_rosenbrock : orc_fn_powell;
  return orc_nelder_mead(f, &n, n, x0, init_scale, tol_x, tol_f, max_iter, x_best, f_best,
                         iterations, func_evals, exit_reason);
}

double orc_test_fn(int fn_id, int n, const double* x) {
  orc_objfn f = fn_id == 0 ? orc_fn_sphere : fn_id == 1 ? orc_fn_rosenbrock : orc_fn_powell;
  return f(x, &n);
}

/* Plant objective for the estimator: E(x) of the full 18-parameter OPC
   against one relativized trace (penalty / +inf rules as orc_objective). */
typedef struct {
  const double* rel;
  int32_t n_steps, substeps;
  double dt_ms, Aprime, pw_default_ms;
  int metric;
  double* buf;
} orc_plant_ctx;

static double orc_fn_plant(const double* x, void* ctx) {
  orc_plant_ctx* c = (orc_plant_ctx*)ctx;
  return orc_objective_sub(x, c->rel, c->n_steps, c->dt_ms, c->substeps, c->Aprime,
                           c->pw_default_ms, c->metric, c->buf);
}

/* estimate_batch (Alg. 1): saccade s is fitted from x0
   (Table 1 defaults; PW NaN -> the saccade's pw_default) independently of the
   others; results in input order, identical for any nthreads (D12). */
int orc_estimate_batch(const double* rec, int64_t S, int32_t n_steps, double dt_ms, int32_t substeps,
                       const double* amplitude, const double* pw_default, const double* x0,
                       int metric, double init_scale, double tol_x, double tol_f, int max_iter,
                       int nthreads, double* x_best, double* f_best, int32_t* iterations,
                       int32_t* func_evals, int32_t* exit_reason) {
  int64_t s;
  if (nthreads < 1) nthreads = 1;
#ifdef _OPENMP
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 1)
#endif
  for (s = 0; s < S; ++s) {
    double* rel = (double*)malloc(sizeof(double) * (size_t)(n_steps + 1));
    double* buf = (double*)malloc(sizeof(double) * (size_t)(n_steps + 1));
    double sgn, Ap, xs[ORC_NP];
    int it, ev, why, d;
    orc_plant_ctx ctx;
    orc_relativize(rec + s * (int64_t)(n_steps + 1), n_steps + 1, amplitude[s], rel, &sgn, &Ap);
    for (d = 0; d < ORC_NP; ++d) xs[d] = x0[d];
    if (isnan(xs[P_PW])) xs[P_PW] = pw_default[s];
    ctx.rel = rel; ctx.n_steps = n_steps; ctx.substeps = substeps; ctx.dt_ms = dt_ms; ctx.Aprime = Ap;
    ctx.pw_default_ms = pw_default[s]; ctx.metric = metric; ctx.buf = buf;
    orc_nelder_mead(orc_fn_plant, &ctx, ORC_NP, xs, init_scale, tol_x, tol_f, max_iter,
                    x_best + s * ORC_NP, f_best + s, &it, &ev, &why);
    iterations[s] = it; func_evals[s] = ev; exit_reason[s] = why;
    free(rel); free(buf);
  }
  return 0;
}
