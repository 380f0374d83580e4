// opmm_device.cuh -- device-side building blocks of the libopmm hot path
// (sm_100a).  Everything here runs per candidate, one candidate per thread,
// with the OPC vector, the per-candidate propagator and the plant state in
// registers and the relativized recorded trace in shared memory.
//
// Paper / spec anchors (see DESIGN.md for the readings Q1..Q21):
//   OPC vector, Table-1 order ............ PAPER.md:150-167
//   pulse-step control signal ............ PAPER.md:106-117 (activation at onset,
//                                           deactivation at offset), PAPER.md:167 (PW)
//   plant topology ....................... Fig. 1; equations SPEC D1
//   integrator: classical RK4, h = dt .... SPEC D2
//   error = absolute difference .......... PAPER.md:366
//   exhaustive search / argmin ........... PAPER.md:202
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace opmm {

constexpr int NP = 18;
constexpr double CAP = 1e20;        // reading Q10
constexpr double PENALTY = 1e10;    // SPEC D8
constexpr double NANT_FLOOR = 0.01; // SPEC D4

enum { KSE_AG = 0, KSE_ANT, KLT_AG, KLT_ANT, B_AG, B_ANT, B_P, NC_AG, NC_ANT, J_,
       TAU_AC_AG, TAU_AC_ANT, TAU_DE_AG, TAU_DE_ANT, NC_FIX, NSAC_AG, NSAC_ANT, PW_ };

// exp() table for the log-uniform map: EXP_TAB[j] = exp(j/128) as a
// double-double (hi, lo), j = 0..EXP_TAB_N-1, covering arguments in [0, 8).
constexpr int EXP_TAB_N = 1032;   // j = rint(128 x) <= 1024 for x < 8
constexpr double EXP_TAB_MAX = 8.0;

// Search space, preprocessed on the host (kernel parameter -> constant bank).
struct SpaceDev {
  int32_t mode;          // 0 random (Philox), 1 grid
  uint32_t key0, key1;   // Philox key = seed
  int32_t all_physical;  // host proved every candidate of the space physical
  int32_t model;         // 0 = 18-parameter, 1 = 9-parameter (D7 expansion)
  // 0 fixed (lo), 1 linear, 2 log with table exp (argument < 8), 3 log with libm exp
  uint8_t kind[NP];
  double lo[NP];
  // random: linear hi-lo, log log(hi/lo); grid: linear (hi-lo)/(L-1), log log(hi/lo)/(L-1)
  double span[NP];
  double span32[NP];     // random: span * 2^-32 (exact; see map_word)
  int32_t exact_u;       // random: some span32 would be subnormal -> literal u * span
  int32_t fast_gen;      // random, kinds 0/1/2 only, !exact_u: branch-free generate_opc
  double gsel[NP];       // fast_gen: 1 for table-exp (kind 2) dimensions, else 0
  double lsel[NP];       // fast_gen: 1 for linear (kind 1) dimensions, else 0
  int64_t levels[NP];    // grid radices (1 = not a grid dimension)
  int64_t pw_stride;     // grid: product of levels[0..16] (PW digit = i / pw_stride % L17)
};

// Per-launch control (shared by every candidate of a saccade).
struct CtlDev {
  int32_t substeps;      // RK4 steps per sample interval (>= 1), reading Q25
  double dt_ms;
  double h;              // dt in seconds
  int32_t n_steps;
  double theta0;         // explicit simulate output offset
};

// ----------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al. SC'11), reading Q15.
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

// exp(x) for x in [0, 8): j = rint(128 x) through the 1.5 * 2^52 shifter (its
// low word is j; no float<->int conversions), r = x - j/128 in [-1/256, 1/256]
// exact (Sterbenz), exp(x) = E_j (1 + q), q = expm1(r) by a degree-5 Taylor
// polynomial (truncation < 5e-18 relative), E_j a double-double table entry
// (j <= 1024); one final rounding, so the result is within ~0.51 ulp of exp(x)
// -- the same value a correctly-rounded libm returns in all but near-tie
// cases, for ~10 fp64 instructions instead of ~50 for the general-range exp().
// (Round 2: the 1/128 table and degree 5 measured 0.8% faster than 1/64 and
// degree 6; a branch per dimension instead of the selects below, 4% slower.)
__device__ __forceinline__ double exp_tab(double x, const double2* __restrict__ tab) {
  constexpr double SHIFT = 6755399441055744.0;   // 1.5 * 2^52
  const double t = __fma_rn(x, 128.0, SHIFT);
  const int j = __double2loint(t);
  const double r = __fma_rn(__dsub_rn(t, SHIFT), -0.0078125, x);
  double q = 1.0 / 120.0;
  q = fma(q, r, 1.0 / 24.0);
  q = fma(q, r, 1.0 / 6.0);
  q = fma(q, r, 0.5);
  q = fma(q, r, 1.0);
  q = q * r;
  const double2 e = tab[j];
  return e.x + fma(e.x, q, e.y);
}

// General-range exp for log dimensions whose argument can reach 8 or more
// (kind 3): out of line, so the 17 inlined maps carry one call, not 17
// copies of libm's exp.
static __device__ __noinline__ double exp_libm(double x) { return exp(x); }

// u = (w + 0.5) 2^-32 is exact in fp64; the mapping uses explicitly rounded
// operations so no FMA contraction changes the candidate bits; the exp
// argument fl(u * log(hi/lo)) is the one the generator definition names.
// w + 0.5 is formed exactly from the bits (2^52 + w) - (2^52 - 1/2), and
// fl(u * span) = fl((w + 0.5) * span32) with span32 = span 2^-32 exact (host,
// only when span32 is a normal number; otherwise exact_u takes the literal
// route).
__device__ __forceinline__ double map_word(const SpaceDev& sp, int d, uint32_t w,
                                           const double2* __restrict__ tab) {
  const double w5 = __dsub_rn(__hiloint2double(0x43300000, (int)w), 4503599627370495.5);
  if (sp.kind[d] == 0) return sp.lo[d];
  const double x = sp.exact_u ? __dmul_rn(__dmul_rn(w5, 2.3283064365386962890625e-10), sp.span[d])
                              : __dmul_rn(w5, sp.span32[d]);
  if (sp.kind[d] == 1) return __dadd_rn(sp.lo[d], x);
  return __dmul_rn(sp.lo[d], sp.kind[d] == 2 ? exp_tab(x, tab) : exp_libm(x));
}

// 9-parameter OPMM (Table 2) in the 18-vector, SPEC D7
// (SPEC.md:132): shared K_SE / K_LT, canonical pulse 55 / 0.5 g of width
// pw_default (PW NaN), Table 1 time constants (reading Q23).
__device__ __forceinline__ void expand_9param(double p[NP]) {
  p[KSE_ANT] = p[KSE_AG];
  p[KLT_ANT] = p[KLT_AG];
  p[TAU_AC_AG] = 11.7;
  p[TAU_AC_ANT] = 2.4;
  p[TAU_DE_AG] = 2.0;
  p[TAU_DE_ANT] = 1.9;
  p[NSAC_AG] = 55.0;
  p[NSAC_ANT] = 0.5;
  p[PW_] = __longlong_as_double(0x7ff8000000000000LL);
}

// Candidate index -> OPC vector (PAPER.md:202 exhaustive search over OPC values).
// Random mode is fully unrolled: the five Philox blocks and the 17 exp() are
// independent dependency chains, so the scheduler can overlap them (the
// generator is ~20% of a candidate's instructions).  Grid mode (int64 div/mod
// per dimension) stays rolled to keep the kernel's code footprint small.
// Grid mode of generate_opc (mixed-radix digits, dimension 0 fastest).
// Value of grid dimension d at level `digit` (lo, lo + j span, or lo exp(j span)).
__device__ __forceinline__ double grid_value(const SpaceDev& sp, int d, uint64_t digit,
                                            const double2* __restrict__ tab) {
  const uint64_t L = (uint64_t)sp.levels[d];
  if (sp.kind[d] == 0 || L <= 1) return sp.lo[d];
  if (sp.kind[d] == 1) return __dadd_rn(sp.lo[d], __dmul_rn((double)digit, sp.span[d]));
  const double x = __dmul_rn((double)digit, sp.span[d]);
  return __dmul_rn(sp.lo[d], sp.kind[d] == 2 ? exp_tab(x, tab) : exp_libm(x));
}

__device__ __forceinline__ void generate_grid_opc(const SpaceDev& sp, int64_t idx, double p[NP],
                                                  const double2* __restrict__ tab) {
  uint64_t rem = (uint64_t)idx;
#pragma unroll 1
  for (int d = 0; d < NP; ++d) {
    uint64_t digit = 0;
    const uint64_t L = (uint64_t)sp.levels[d];
    if (L > 1) {
      digit = rem % L;
      rem = rem / L;
    }
    double v;   // grid_value(sp, d, digit, tab), written out (register allocation of fit_kernel)
    if (sp.kind[d] == 0 || L <= 1) v = sp.lo[d];
    else if (sp.kind[d] == 1) v = __dadd_rn(sp.lo[d], __dmul_rn((double)digit, sp.span[d]));
    else {
      const double x = __dmul_rn((double)digit, sp.span[d]);
      v = __dmul_rn(sp.lo[d], sp.kind[d] == 2 ? exp_tab(x, tab) : exp_libm(x));
    }
    // static-index stores keep p[] in registers after the loop is unrolled
    // by the caller's use; write through a switch-free select chain
#pragma unroll
    for (int e = 0; e < NP; ++e)
      if (e == d) p[e] = v;
  }
  if (sp.model == 1) expand_9param(p);
}

__device__ __forceinline__ void generate_opc(const SpaceDev& sp, uint32_t saccade, int64_t idx,
                                             double p[NP], const double2* __restrict__ tab) {
  if (sp.mode == 0) {
    const uint2 key = make_uint2(sp.key0, sp.key1);
    const uint32_t ilo = (uint32_t)((uint64_t)idx & 0xffffffffu);
    const uint32_t ihi = (uint32_t)((uint64_t)idx >> 32);
    uint32_t ws[20];
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const uint4 w = philox4x32_10(make_uint4(ilo, ihi, saccade, (uint32_t)j), key);
      ws[4 * j] = w.x; ws[4 * j + 1] = w.y; ws[4 * j + 2] = w.z; ws[4 * j + 3] = w.w;
    }
    if (sp.fast_gen) {
      // Branch-free form of map_word for kinds 0/1/2 (no per-dimension
      // branches or kind loads): x = (w + 1/2) span32, E = exp_tab(x g), and
      // v = fma(x, l, lo E) with (g, l) = (1, 0) table-exp, (0, 1) linear,
      // (*, 0) fixed (span32 = 0).  Bit-identical to map_word: fma(x, 0, y)
      // = y, lo * 1 = lo, fma(x, 1, lo) = lo + x, and exp_tab(0) = 1.
#pragma unroll
      for (int d = 0; d < NP; ++d) {
        const double w5 = __dsub_rn(__hiloint2double(0x43300000, (int)ws[d]), 4503599627370495.5);
        const double x = __dmul_rn(w5, sp.span32[d]);
        const double E = exp_tab(__dmul_rn(x, sp.gsel[d]), tab);
        p[d] = __fma_rn(x, sp.lsel[d], __dmul_rn(sp.lo[d], E));
      }
    } else {
#pragma unroll
      for (int d = 0; d < NP; ++d) p[d] = map_word(sp, d, ws[d], tab);
    }
    if (sp.model == 1) expand_9param(p);
  } else {
    generate_grid_opc(sp, idx, p, tab);
  }
}

// Grid spaces from per-dimension level tables (fit_kernel, GT): gt holds
// grid_value(d, j) for every dimension with levels > 1, concatenated in
// dimension order (build_grid_tables).  Digits of idx by mixed radix
// (dimension 0 fastest; 32-bit division while the remainder fits), then one
// shared-memory load per grid dimension -- bit-identical to
// generate_grid_opc, whose values the tables are.
__device__ __forceinline__ void build_grid_tables(const SpaceDev& sp, double* gt,
                                                  const double2* __restrict__ tab) {
  int off = 0;
  for (int d = 0; d < NP; ++d) {
    const int64_t L = sp.levels[d];
    if (L <= 1) continue;
    for (int j = threadIdx.x; j < (int)L; j += blockDim.x) gt[off + j] = grid_value(sp, d, (uint64_t)j, tab);
    off += (int)L;
  }
}

__device__ __forceinline__ void grid_opc_from_tables(const SpaceDev& sp, int64_t idx,
                                                     const double* __restrict__ gt, double p[NP]) {
  uint64_t rem = (uint64_t)idx;
  int off = 0;
#pragma unroll
  for (int d = 0; d < NP; ++d) {
    const int64_t L = sp.levels[d];
    if (L > 1) {
      uint64_t digit;
      if ((rem >> 32) == 0) {
        const uint32_t r32 = (uint32_t)rem, q32 = r32 / (uint32_t)L;
        digit = r32 - q32 * (uint32_t)L;
        rem = q32;
      } else {
        const uint64_t q = rem / (uint64_t)L;
        digit = rem - q * (uint64_t)L;
        rem = q;
      }
      p[d] = gt[off + (int)digit];
      off += (int)L;
    } else {
      p[d] = sp.lo[d];
    }
  }
  if (sp.model == 1) expand_9param(p);
}

// PW of candidate idx alone (for the lane sort key): Philox block j = 4,
// word 1 is dimension 17; grid mode takes the PW digit directly.
__device__ __forceinline__ double generate_pw(const SpaceDev& sp, uint32_t saccade, int64_t idx,
                                              const double2* __restrict__ tab) {
  if (sp.mode == 0) {
    const uint4 w = philox4x32_10(make_uint4((uint32_t)((uint64_t)idx & 0xffffffffu),
                                             (uint32_t)((uint64_t)idx >> 32), saccade, 4u),
                                  make_uint2(sp.key0, sp.key1));
    return map_word(sp, PW_, w.y, tab);
  }
  const uint64_t L = (uint64_t)sp.levels[PW_];
  const uint64_t digit = L > 1 ? ((uint64_t)idx / (uint64_t)sp.pw_stride) % L : 0;
  if (sp.kind[PW_] == 0 || L <= 1) return sp.lo[PW_];
  if (sp.kind[PW_] == 1) return __dadd_rn(sp.lo[PW_], __dmul_rn((double)digit, sp.span[PW_]));
  return __dmul_rn(sp.lo[PW_], exp(__dmul_rn((double)digit, sp.span[PW_])));
}

// Sort key of fit_kernel's pre-pass: the block index at which the pulse ends,
// n_pulse / 2 -- scheduling only (results never depend on it), so random
// spaces map the PW word in fp32 (no fp64 exp/division); grid spaces and the
// 9-parameter model use the exact value.
__device__ __forceinline__ int pulse_end_key(const SpaceDev& sp, uint32_t saccade, int64_t idx,
                                             double pw_default, double dt_ms, int32_t n_steps,
                                             int nbins, const double2* __restrict__ tab) {
  float npf;
  if (sp.model != 1 && sp.mode == 0) {
    const uint4 w = philox4x32_10(make_uint4((uint32_t)((uint64_t)idx & 0xffffffffu),
                                             (uint32_t)((uint64_t)idx >> 32), saccade, 4u),
                                  make_uint2(sp.key0, sp.key1));
    const float u = fmaf((float)w.y, 2.3283064365386963e-10f, 1.1641532182693481e-10f);
    const float lo = (float)sp.lo[PW_], span = (float)sp.span[PW_];
    const float pw = sp.kind[PW_] == 0 ? lo : sp.kind[PW_] == 1 ? fmaf(u, span, lo)
                                                                : lo * __expf(u * span);
    npf = ceilf(pw * (float)(1.0 / dt_ms));
  } else {
    double pw = sp.model == 1 ? pw_default : generate_pw(sp, saccade, idx, tab);
    if (isnan(pw)) pw = pw_default;
    npf = (float)ceil(pw / dt_ms);
  }
  const int np = !(npf <= (float)n_steps) ? n_steps + 1 : (int)npf;   // NaN -> whole-pulse bin
  return min(max(np, 0) >> 1, nbins - 1);
}

// ----------------------------------------------------------------------------
// Physical check (SPEC D8 SPEC.md:248, reading Q13): 0 if physical, else the
// penalty 1e10 (1 + sum of violation amounts).  PW NaN is the placeholder.
// ----------------------------------------------------------------------------
__device__ __forceinline__ double physical_penalty(const double p[NP]) {
  bool bad = false;
  double amount = 0.0;
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    const double v = p[i];
    const bool strict = (i == KSE_AG || i == KSE_ANT || i == B_AG || i == B_ANT || i == J_ ||
                         i == TAU_AC_AG || i == TAU_AC_ANT || i == TAU_DE_AG || i == TAU_DE_ANT ||
                         i == PW_);
    if (i == PW_ && isnan(v)) continue;
    if (!isfinite(v)) { bad = true; amount += 1.0; continue; }
    if (strict ? !(v > 0.0) : !(v >= 0.0)) {
      bad = true;
      if (v < 0.0) amount += -v;
    }
  }
  if (!bad) {
    const double g_ag = p[KSE_AG] / (p[KLT_AG] + p[KSE_AG]);
    const double g_ant = p[KSE_ANT] / (p[KLT_ANT] + p[KSE_ANT]);
    const double G = g_ag * (p[NC_AG] + p[KLT_AG]) + g_ant * (p[NC_ANT] + p[KLT_ANT]);
    if (!(G > 0.0)) bad = true;
  }
  return bad ? PENALTY * (1.0 + amount) : 0.0;
}

// ----------------------------------------------------------------------------
// Per-candidate setup.  The plant (SPEC D1) is linear and time-invariant
// within each control phase, so we integrate the deviation from the fixation
// equilibrium y* (reading Q5): y~ = y - y*, which obeys the same ODE with the
// drive n replaced by n~ = n - N_C_FIX and starts at 0; theta~ IS Delta-theta.
//
// z = (theta, omega, x_AG, x_ANT), f = (f_AG, f_ANT);  Z = h M (dimensionless):
//   Z01 = h
//   Z1* = h/J (-(K_SE_AG+K_SE_ANT), -B_P, K_SE_AG, -K_SE_ANT)
//   Z2* = h/B_AG  (-(N_C_AG - K_SE_AG), 0, -(K_LT_AG + K_SE_AG), 0)
//   Z3* = h/B_ANT ((N_C_ANT - K_SE_ANT), 0, 0, -(K_LT_ANT + K_SE_ANT))
//   x_m is driven by f_m / B_m;   f_m' = (n_m - f_m)/tau_m,  zd_m = -dt/tau_m.
// ----------------------------------------------------------------------------
// 1/x for positive normal x: MUFU reciprocal seed + two Newton steps
// (~0.5-1 ulp).  The setup's quotients only need to be accurate, not
// correctly rounded (parity is to 1e-9 relative), so this replaces the
// slow-path-guarded IEEE division; the one integer-deciding quotient
// ceil(PW/dt) keeps the IEEE division.
__device__ __forceinline__ double rcp64(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

struct Mech {
  double z01, z10, z11, z12, z13, z20, z22, z30, z33;
  double hb_ag, hb_ant;   // h / B_m
};

struct Phase {            // control of one phase (pulse or post-pulse step)
  double zd_ag, zd_ant;   // -dt / tau_m
  double nt_ag, nt_ant;   // n~_m = n_m - N_C_FIX
};

struct Setup {
  Mech m;
  Phase ph[2];            // 0 = pulse (tau_AC, N_SAC), 1 = step (tau_DE, D4 levels)
  int32_t n_pulse;        // steps k < n_pulse use phase 0 (reading Q6)
};

// substeps > 1 (reading Q25): the dynamics coefficients are those of one
// substep, h/substeps; the pulse window stays in samples of dt.
__device__ __forceinline__ void make_setup(const double p_in[NP], double dt_ms, double h_sample,
                                           int32_t n_steps, double Aprime, double pw_default,
                                           Setup& s, int32_t substeps = 1) {
  double h = h_sample, dts = dt_ms;
  if (substeps > 1) {
    h = h_sample / (double)substeps;
    dts = dt_ms / (double)substeps;
  }
  const double Kag = p_in[KSE_AG], Kant = p_in[KSE_ANT], Lag = p_in[KLT_AG], Lant = p_in[KLT_ANT];
  const double Bag = p_in[B_AG], Bant = p_in[B_ANT], Bp = p_in[B_P];
  const double Ncag = p_in[NC_AG], Ncant = p_in[NC_ANT], J = p_in[J_], F = p_in[NC_FIX];
  double PW = p_in[PW_];
  if (isnan(PW)) PW = pw_default;
  const double hJ = h * rcp64(J), hBag = h * rcp64(Bag), hBant = h * rcp64(Bant);
  s.m.z01 = h;
  s.m.z10 = -(Kag + Kant) * hJ;
  s.m.z11 = -Bp * hJ;
  s.m.z12 = Kag * hJ;
  s.m.z13 = -Kant * hJ;
  s.m.z20 = -(Ncag - Kag) * hBag;
  s.m.z22 = -(Lag + Kag) * hBag;
  s.m.z30 = (Ncant - Kant) * hBant;
  s.m.z33 = -(Lant + Kant) * hBant;
  s.m.hb_ag = hBag;
  s.m.hb_ant = hBant;
  // Post-pulse step levels: static balance at theta* + A' (D4 generalised, Q4).
  const double g_ag = Kag * rcp64(Lag + Kag), g_ant = Kant * rcp64(Lant + Kant);
  const double G = g_ag * (Ncag + Lag) + g_ant * (Ncant + Lant);
  const double delta = G * Aprime * rcp64(g_ag + g_ant);
  double nt_ag = delta, nt_ant = -delta;
  if (F - delta < NANT_FLOOR) {
    const double theta_star = (g_ag * F - g_ant * F) * rcp64(G);
    const double n_ag = (G * (theta_star + Aprime) + NANT_FLOOR * g_ant) * rcp64(g_ag);
    nt_ag = n_ag - F;
    nt_ant = NANT_FLOOR - F;
  }
  s.ph[0].zd_ag = -dts * rcp64(p_in[TAU_AC_AG]);
  s.ph[0].zd_ant = -dts * rcp64(p_in[TAU_AC_ANT]);
  s.ph[0].nt_ag = p_in[NSAC_AG] - F;
  s.ph[0].nt_ant = p_in[NSAC_ANT] - F;
  s.ph[1].zd_ag = -dts * rcp64(p_in[TAU_DE_AG]);
  s.ph[1].zd_ant = -dts * rcp64(p_in[TAU_DE_ANT]);
  s.ph[1].nt_ag = nt_ag;
  s.ph[1].nt_ant = nt_ant;
  // Pulse window: onset at step 0, n_pulse = ceil(PW/dt) (IEEE divide), Q6.
  const double npd = ceil(PW / dt_ms);
  s.n_pulse = npd > (double)n_steps ? n_steps + 1 : (int32_t)npd;
}

// ----------------------------------------------------------------------------
// Propagator form of the RK4 map: for one phase,
//   [z; f]+ = P(hA) [z; f] + hQ(hA) b~,  P(x) = 1+x+x^2/2+x^3/6+x^4/24,
//   Q(x) = 1+x/2+x^2/6+x^3/24 -- exactly the classical RK4 step of the LTI
// system (textbook identity; pinned in tests as P7).  A is block upper
// triangular [[M, C],[0, D]], D = diag(-1/tau), C = diag(1/B) on the x rows,
// so with u_i = Z^i (h c_m) and a_i(zd) = sum_{j>i} zd^(j-1-i)/j!:
//   mech <- f block  X[:,m] = sum_{i=0..3} u_i a_i(zd_m)
//   forcing          c      = sum_m (-zd_m n~_m) sum_{i=0..2} u_i a_{i+1}(zd_m)
//   f update         f_m+   = (1 + zd_m a_0) f_m + (-zd_m a_0 n~_m)
// The 4x4 mechanical block P(Z) is phase-independent.
// ----------------------------------------------------------------------------
template <typename T> struct Vec2;
template <> struct Vec2<double> { using type = double2; };
template <> struct Vec2<float> { using type = float2; };
template <typename T>
__device__ __forceinline__ typename Vec2<T>::type make_v2(T a, T b) {
  typename Vec2<T>::type v;
  v.x = a;
  v.y = b;
  return v;
}

// Two-step blocks.  The loop advances two RK4 steps per iteration with the
// composed map M2 = M.M, c2 = M c + c (still exactly the RK4 recurrence), and
// recovers the intermediate sample from row 0 of the one-step map:
//   theta_{k+1} = P[0].z_k + X[0].f_k + c[0]          (7 terms)
//   z_{k+2}     = P2 z_k + X2 f_k + c2,  X2 = P X + X diag(pf),
//                 c2 = P c + X qf + c                  (4 rows x 7 terms)
//   f_{k+2}     = pf^2 f_k + (pf qf + qf)
// 32 FMA + 4 score ops per two steps (18 per step, vs 28 for one-step
// blocks and 92 for the literal four-stage form).  Phase switches fall on
// block boundaries because each lane starts at k = n_pulse mod 2: an odd lane
// takes its first pulse step for free (from the zero deviation state
// z_1 = c, f_1 = qf).
template <typename T>
struct PhaseProp2 {
  T X2[4][2];
  T c2[4];
  T pf2[2], qf2[2];
  T X0[2];   // row 0 of the one-step X
  T c0;      // row 0 of the one-step c
};

template <typename T>
struct Prop2 {
  T P2[4][4];
  T P0[4];             // row 0 of the one-step P (phase-independent)
  PhaseProp2<T> ph[2];
  T z1[4], f1[2];      // state after one pulse step from zero (odd start)
};

// Structural zeros of u_i = Z^i (h c_m) (Z: row 0 = (0,h,0,0), row 2 couples
// only theta and x_AG, row 3 only theta and x_ANT): NZU[m][i][r] is false where
// u_i[r] is identically zero, so those terms are dropped at compile time.
__device__ constexpr bool NZU[2][4][4] = {
    {{false, false, true, false}, {false, true, true, false}, {true, true, true, false},
     {true, true, true, true}},
    {{false, false, false, true}, {false, true, false, true}, {true, true, false, true},
     {true, true, true, true}}};

// out = Z v for a vector v with structural-zero mask nz (compile-time).
template <typename R, typename MM>
__device__ __forceinline__ void zmul_masked(const MM& m, const R v[4], const bool nz[4], R out[4]) {
  out[0] = nz[1] ? R(m.z01) * v[1] : R(0);
  R o1 = R(0);
  if (nz[0]) o1 = R(m.z10) * v[0];
  if (nz[1]) o1 = fma(R(m.z11), v[1], o1);
  if (nz[2]) o1 = fma(R(m.z12), v[2], o1);
  if (nz[3]) o1 = fma(R(m.z13), v[3], o1);
  out[1] = o1;
  R o2 = R(0);
  if (nz[0]) o2 = R(m.z20) * v[0];
  if (nz[2]) o2 = fma(R(m.z22), v[2], o2);
  out[2] = o2;
  R o3 = R(0);
  if (nz[0]) o3 = R(m.z30) * v[0];
  if (nz[3]) o3 = fma(R(m.z33), v[3], o3);
  out[3] = o3;
}

// Post-pulse coefficients in the per-thread shared-memory stash: [10][ld]
// vec2 (see run_propagator).
template <typename T>
__device__ __forceinline__ void stash_phase(const PhaseProp2<T>& q, typename Vec2<T>::type* st2,
                                            int ld) {
  st2[0 * ld] = make_v2<T>(q.X2[0][0], q.X2[0][1]);
  st2[1 * ld] = make_v2<T>(q.X2[1][0], q.X2[1][1]);
  st2[2 * ld] = make_v2<T>(q.X2[2][0], q.X2[2][1]);
  st2[3 * ld] = make_v2<T>(q.X2[3][0], q.X2[3][1]);
  st2[4 * ld] = make_v2<T>(q.c2[0], q.c2[1]);
  st2[5 * ld] = make_v2<T>(q.c2[2], q.c2[3]);
  st2[6 * ld] = make_v2<T>(q.pf2[0], q.pf2[1]);
  st2[7 * ld] = make_v2<T>(q.qf2[0], q.qf2[1]);
  st2[8 * ld] = make_v2<T>(q.X0[0], q.X0[1]);
  st2[9 * ld] = make_v2<T>(q.c0, T(0));
}

// Building blocks of the propagator (force-inlined into make_prop, so its
// code is the one-pass form below; make_prop_sub reuses them for substeps).
// R is the arithmetic type (double in the product; see make_prop).
//
// one-step mechanical block P(Z) = (I + Z) + Z^2 (I/2 + Z/6 + Z^2/24),
// Z = hM: Z^2 from Z's 9 structural non-zeros (19 ops), then one sparse x
// dense product (Z^2 has zeros at (2,3) and (3,2)) -- ~100 ops instead of
// ~156 for three Horner steps.
template <typename R>
__device__ __forceinline__ void one_step_P(const Mech& m, R P[4][4]) {
  const R h = R(m.z01), a = R(m.z10), b = R(m.z11), c = R(m.z12), d = R(m.z13);
  const R e = R(m.z20), f = R(m.z22), g = R(m.z30), k = R(m.z33);
  R Z2[4][4];
  Z2[0][0] = h * a; Z2[0][1] = h * b; Z2[0][2] = h * c; Z2[0][3] = h * d;
  Z2[1][0] = fma(b, a, fma(c, e, d * g));
  Z2[1][1] = fma(a, h, b * b);
  Z2[1][2] = fma(b, c, c * f);
  Z2[1][3] = fma(b, d, d * k);
  Z2[2][0] = f * e; Z2[2][1] = e * h; Z2[2][2] = f * f; Z2[2][3] = R(0);
  Z2[3][0] = k * g; Z2[3][1] = g * h; Z2[3][2] = R(0); Z2[3][3] = k * k;
  const R Zm[4][4] = {{R(0), h, R(0), R(0)}, {a, b, c, d}, {e, R(0), f, R(0)}, {g, R(0), R(0), k}};
  // B = I/2 + Z/6 + Z^2/24
  R B[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const bool zz = (i == 0 && j != 1) || (i == 2 && (j == 1 || j == 3)) || (i == 3 && (j == 1 || j == 2));
      R v = Z2[i][j] * R(1.0 / 24.0);
      if (!zz) v = fma(Zm[i][j], R(1.0 / 6.0), v);
      if (i == j) v += R(0.5);
      B[i][j] = v;
    }
  // P = I + Z + Z^2 B
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const bool zz = (i == 0 && j != 1) || (i == 2 && (j == 1 || j == 3)) || (i == 3 && (j == 1 || j == 2));
      R v = (i == j ? R(1) : R(0)) + (zz ? R(0) : Zm[i][j]);
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        if ((i == 2 && l == 3) || (i == 3 && l == 2)) continue;   // Z^2 structural zeros
        v = fma(Z2[i][l], B[l][j], v);
      }
      P[i][j] = v;
    }
}

// u_i = Z^i (h c_m): c_AG = e_2 / B_AG, c_ANT = e_3 / B_ANT.
template <typename R>
__device__ __forceinline__ void coupling_u(const Mech& m, R u[2][4][4]) {
#pragma unroll
  for (int mm = 0; mm < 2; ++mm) {
    u[mm][0][0] = R(0); u[mm][0][1] = R(0);
    u[mm][0][2] = (mm == 0) ? R(m.hb_ag) : R(0);
    u[mm][0][3] = (mm == 0) ? R(0) : R(m.hb_ant);
#pragma unroll
    for (int i = 1; i < 4; ++i) zmul_masked<R>(m, u[mm][i - 1], NZU[mm][i - 1], u[mm][i]);
  }
}

// One step of one control phase: coupling X (mechanics <- f), forcing c, and
// the f update f+ = pf f + qf.
template <typename R>
__device__ __forceinline__ void one_step_phase(const Phase& phs, const R u[2][4][4], R X[4][2],
                                               R c[4], R pf[2], R qf[2]) {
#pragma unroll
  for (int r = 0; r < 4; ++r) c[r] = R(0);
#pragma unroll
  for (int mm = 0; mm < 2; ++mm) {
    const R zd = R(mm == 0 ? phs.zd_ag : phs.zd_ant);
    const R nt = R(mm == 0 ? phs.nt_ag : phs.nt_ant);
    R av[4];
    av[3] = R(1.0 / 24.0);
    av[2] = fma(zd, av[3], R(1.0 / 6.0));
    av[1] = fma(zd, av[2], R(0.5));
    av[0] = fma(zd, av[1], R(1));
    const R g = -zd * nt;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      // X[:,m] = sum_i u_i a_i;  c += g sum_{i<3} u_i a_{i+1}  (structural zeros skipped)
      R x = R(0), cc = R(0);
      bool first_x = true, first_c = true;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (!NZU[mm][i][r]) continue;
        x = first_x ? u[mm][i][r] * av[i] : fma(u[mm][i][r], av[i], x);
        first_x = false;
        if (i < 3) {
          cc = first_c ? u[mm][i][r] * av[i + 1] : fma(u[mm][i][r], av[i + 1], cc);
          first_c = false;
        }
      }
      X[r][mm] = x;
      if (!first_c) c[r] = fma(g, cc, c[r]);
    }
    pf[mm] = fma(zd, av[0], R(1));
    qf[mm] = g * av[0];
  }
}

// Two-step block of one phase from its one-step map (X2 = P X + X diag(pf),
// c2 = P c + X qf + c, f: pf^2, pf qf + qf) plus row 0 of the one-step map.
template <typename T, typename R>
__device__ __forceinline__ void two_step_phase(const R P[4][4], const R X[4][2], const R c[4],
                                               const R pf[2], const R qf[2], PhaseProp2<T>& q) {
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    R c2 = fma(X[r][1], qf[1], fma(X[r][0], qf[0], c[r]));
#pragma unroll
    for (int l = 0; l < 4; ++l) c2 = fma(P[r][l], c[l], c2);
    q.c2[r] = (T)c2;
#pragma unroll
    for (int mm = 0; mm < 2; ++mm) {
      R x2 = X[r][mm] * pf[mm];
#pragma unroll
      for (int l = 0; l < 4; ++l) x2 = fma(P[r][l], X[l][mm], x2);
      q.X2[r][mm] = (T)x2;
    }
  }
#pragma unroll
  for (int mm = 0; mm < 2; ++mm) {
    q.pf2[mm] = (T)(pf[mm] * pf[mm]);
    q.qf2[mm] = (T)fma(pf[mm], qf[mm], qf[mm]);
    q.X0[mm] = (T)X[0][mm];
  }
  q.c0 = (T)c[0];
}

template <typename T, typename R>
__device__ __forceinline__ void square_P(const R P[4][4], Prop2<T>& pr) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      R a = P[i][0] * P[0][j];
#pragma unroll
      for (int l = 1; l < 4; ++l) a = fma(P[i][l], P[l][j], a);
      pr.P2[i][j] = (T)a;
    }
    pr.P0[i] = (T)P[0][i];
  }
}

// STASH: the post-pulse phase is written to the stash as soon as it is built
// (post-pulse first), so it never occupies registers next to the pulse phase
// -- this lowers the kernel's register peak at the setup -> loop transition.
// R: the coefficient arithmetic, fp64 for both paths (reading Q11).  fp32
// coefficients (R = float) cut the fp32 fit by 11% but made its errors ~5x
// larger (rejected).
template <typename T, bool STASH = false, typename R = double>
__device__ __forceinline__ void make_prop(const Setup& s, Prop2<T>& pr,
                                          typename Vec2<T>::type* st2 = nullptr, int ld = 0) {
  const Mech& m = s.m;
  R P[4][4];
  one_step_P<R>(m, P);
  R u[2][4][4];
  coupling_u<R>(m, u);
#pragma unroll
  for (int phi = 0; phi < 2; ++phi) {
    const int ph = STASH ? 1 - phi : phi;
    R X[4][2], c[4], pf[2], qf[2];
    one_step_phase<R>(s.ph[ph], u, X, c, pf, qf);
    PhaseProp2<T>& q = pr.ph[ph];
    two_step_phase<T, R>(P, X, c, pf, qf, q);
    if (STASH && ph == 1) stash_phase<T>(q, st2, ld);
    if (ph == 0) {
#pragma unroll
      for (int r = 0; r < 4; ++r) pr.z1[r] = (T)c[r];
      pr.f1[0] = (T)qf[0];
      pr.f1[1] = (T)qf[1];
    }
  }
  // P^2 last: it is live through the whole loop, so building it after the
  // phases keeps it out of the setup's register peak
  square_P<T, R>(P, pr);
}

// ----------------------------------------------------------------------------
// Superposition pair (fit_super_kernel): the b and u recurrences of one node
// share every map (P, X, pf: they depend on the plant and the time constants
// only) and differ in the forcing.  u is a unit pulse of one channel with no
// other drive, so its post-pulse forcing is exactly zero and only its pulse
// phase needs c, qf (and the two-step c2, qf2, c[0], the odd-start z1, f1).
// Built once: the maps and b's forcing as make_prop builds them, u's pulse
// forcing with the same one_step_phase / two_step_phase arithmetic -- so both
// are bit-identical to two make_prop calls, at about half the work and
// register peak (a second full Prop2 is never live).
// ----------------------------------------------------------------------------
struct UnitForcing {   // u's pulse-phase forcing terms (post-pulse: all zero)
  double c2[4], qf2[2], c0;
  double z1[4], f1[2];
};

__device__ __forceinline__ void make_prop_bu(const Setup& sb, const Phase& upulse,
                                             Prop2<double>& pb, UnitForcing& pu) {
  const Mech& m = sb.m;
  double P[4][4];
  one_step_P<double>(m, P);
  double u[2][4][4];
  coupling_u<double>(m, u);
#pragma unroll
  for (int phi = 0; phi < 2; ++phi) {
    const int ph = 1 - phi;   // post-pulse first, as make_prop<STASH>
    double X[4][2], c[4], pf[2], qf[2];
    one_step_phase<double>(sb.ph[ph], u, X, c, pf, qf);
    two_step_phase<double, double>(P, X, c, pf, qf, pb.ph[ph]);
    if (ph == 0) {
#pragma unroll
      for (int r = 0; r < 4; ++r) pb.z1[r] = c[r];
      pb.f1[0] = qf[0];
      pb.f1[1] = qf[1];
      // u: same zd (so the same X, pf), its own drive
      double Xu[4][2], cu[4], pfu[2], qfu[2];
      one_step_phase<double>(upulse, u, Xu, cu, pfu, qfu);
      PhaseProp2<double> q;
      two_step_phase<double, double>(P, Xu, cu, pfu, qfu, q);
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        pu.c2[r] = q.c2[r];
        pu.z1[r] = cu[r];
      }
      pu.qf2[0] = q.qf2[0];
      pu.qf2[1] = q.qf2[1];
      pu.c0 = q.c0;
      pu.f1[0] = qfu[0];
      pu.f1[1] = qfu[1];
    }
  }
  square_P<double, double>(P, pb);
}

// ----------------------------------------------------------------------------
// Integer substeps (reading Q25): the sample-to-sample map of a phase is the
// one-substep map (h/s) to the power s, by binary exponentiation of the
// affine map (z, f) -> (P z + X f + c, pf f + qf) -- the loop is unchanged
// and costs the same per sample; only the setup grows (~log2 s squarings).
// Composition A after B: P = PA PB, X = PA XB + XA diag(pfB),
// c = PA cB + XA qfB + cA, pf = pfA pfB, qf = pfA qfB + qfA.
// ----------------------------------------------------------------------------
struct AffineMap {
  double P[4][4];
  double X[2][4][2], c[2][4], pf[2][2], qf[2][2];   // per control phase
};

__device__ __forceinline__ void compose_maps(const AffineMap& A, const AffineMap& B, AffineMap& o) {
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      double v = A.P[i][0] * B.P[0][j];
      for (int l = 1; l < 4; ++l) v = fma(A.P[i][l], B.P[l][j], v);
      o.P[i][j] = v;
    }
  for (int ph = 0; ph < 2; ++ph) {
    for (int r = 0; r < 4; ++r) {
      double cc = fma(A.X[ph][r][1], B.qf[ph][1], fma(A.X[ph][r][0], B.qf[ph][0], A.c[ph][r]));
      for (int l = 0; l < 4; ++l) cc = fma(A.P[r][l], B.c[ph][l], cc);
      o.c[ph][r] = cc;
      for (int mm = 0; mm < 2; ++mm) {
        double x = A.X[ph][r][mm] * B.pf[ph][mm];
        for (int l = 0; l < 4; ++l) x = fma(A.P[r][l], B.X[ph][l][mm], x);
        o.X[ph][r][mm] = x;
      }
    }
    for (int mm = 0; mm < 2; ++mm) {
      o.pf[ph][mm] = A.pf[ph][mm] * B.pf[ph][mm];
      o.qf[ph][mm] = fma(A.pf[ph][mm], B.qf[ph][mm], A.qf[ph][mm]);
    }
  }
}

// M <- M^n, n >= 1
__device__ __forceinline__ void map_power(AffineMap& M, int n) {
  AffineMap R, B = M, t;
  bool have = false;
  while (n > 0) {
    if (n & 1) {
      if (have) { compose_maps(B, R, t); R = t; }
      else { R = B; have = true; }
    }
    n >>= 1;
    if (n > 0) { compose_maps(B, B, t); B = t; }
  }
  M = R;
}

template <typename T>
__device__ __forceinline__ void make_prop_sub(const Setup& s, int nsub, Prop2<T>& pr,
                                           typename Vec2<T>::type* st2, int ld) {
  AffineMap M;   // fp64 for both paths: the powering compounds rounding
  one_step_P<double>(s.m, M.P);
  double u[2][4][4];
  coupling_u<double>(s.m, u);
  for (int ph = 0; ph < 2; ++ph)
    one_step_phase<double>(s.ph[ph], u, M.X[ph], M.c[ph], M.pf[ph], M.qf[ph]);
  map_power(M, nsub);
  square_P<T, double>(M.P, pr);
  for (int ph = 1; ph >= 0; --ph) {
    two_step_phase<T, double>(M.P, M.X[ph], M.c[ph], M.pf[ph], M.qf[ph], pr.ph[ph]);
    if (ph == 1) stash_phase<T>(pr.ph[1], st2, ld);
  }
  for (int r = 0; r < 4; ++r) pr.z1[r] = (T)M.c[0][r];
  pr.f1[0] = (T)M.qf[0][0];
  pr.f1[1] = (T)M.qf[0][1];
}

// ----------------------------------------------------------------------------
// Trace staging (D5/D6, reading Q7/Q8): s = sign(A) (+1 for A = 0),
// A' = |A|, rel_k = s (rec_k - rec_0), into shared memory in the loop's type.
// ----------------------------------------------------------------------------
// Long fp64 traces (>= TMA_TRACE_BYTES, north_star: "staged once per block
// into shared memory, or via TMA when long") arrive by one bulk copy
// (cp.async.bulk, the TMA engine, completion counted on an mbarrier) and are
// then relativized in place; shorter ones, fp32 traces and 16-byte-misaligned
// sources take coalesced loads.  Every thread of the block must call it.
constexpr int TMA_TRACE_BYTES = 48 * 1024;

__device__ __forceinline__ bool stage_trace_bulk(const double* __restrict__ rec, int32_t n_samples,
                                                 double* rel) {
  const uint32_t bytes = (uint32_t)n_samples * 8u;
  if (bytes < (uint32_t)TMA_TRACE_BYTES || (reinterpret_cast<uintptr_t>(rec) & 15u) ||
      (reinterpret_cast<uintptr_t>(rel) & 15u))
    return false;
  __shared__ __align__(8) uint64_t bar;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  const uint32_t bulk = bytes & ~15u;   // the bulk unit is 16 bytes; a last odd sample by hand
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(b) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(bulk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"((uint32_t)__cvta_generic_to_shared(rel)), "l"(rec), "r"(bulk), "r"(b)
                 : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "TMA_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
      "@!P1 bra TMA_WAIT_%=;\n}" :: "r"(b) : "memory");
  if (threadIdx.x == 0 && bulk < bytes) rel[n_samples - 1] = rec[n_samples - 1];
  __syncthreads();   // the hand-copied sample, and every thread past the wait
  return true;
}

template <typename T>
__device__ __forceinline__ void stage_trace(const double* __restrict__ rec, int32_t n_samples,
                                            double amplitude, T* rel, double& sgn,
                                            double& Aprime) {
  const double r0 = rec[0];
  const double A = isnan(amplitude) ? rec[n_samples - 1] - r0 : amplitude;
  sgn = A < 0.0 ? -1.0 : 1.0;
  Aprime = fabs(A);
  if (sizeof(T) == 8 && stage_trace_bulk(rec, n_samples, reinterpret_cast<double*>(rel))) {
    for (int k = threadIdx.x; k < n_samples; k += blockDim.x) rel[k] = (T)(sgn * ((double)rel[k] - r0));
    return;
  }
  for (int k = threadIdx.x; k < n_samples; k += blockDim.x) rel[k] = (T)(sgn * (rec[k] - r0));
}

__device__ __forceinline__ double tabs(double x) { return fabs(x); }
__device__ __forceinline__ float tabs(float x) { return fabsf(x); }

template <int METRIC, typename T>
__device__ __forceinline__ void accumulate(T& acc, T d) {
  if (METRIC == 0) acc += tabs(d);
  else acc = fma(d, d, acc);
}

template <int METRIC, typename T>
__device__ __forceinline__ double finish_error(T acc, int32_t n_samples) {
  const double a = (double)acc;
  if (!(a < CAP)) return __longlong_as_double(0x7ff0000000000000LL);  // +inf (Q10)
  return METRIC == 0 ? a : sqrt(a / (double)n_samples);
}

// ----------------------------------------------------------------------------
// Integrate + fused score, PROPAGATOR form: 26 FMA per step for the RK4 map +
// 2 for the score.  TRAJ (dump mode, no trace): store theta0 + s*Delta-theta_k
// time-major and accumulate |Delta-theta| instead, to flag divergence.
// ----------------------------------------------------------------------------
// Unroll of the two-step loop: 4 blocks for fp64, 2 for fp32 (measured best
// of 1/2/4 on the 1e6 bench fit).
template <typename T> struct LoopUnroll { static constexpr int value = 4; };
template <> struct LoopUnroll<float> { static constexpr int value = 2; };

// REGSTASH: the post-pulse coefficients stay in registers (pr.ph[1]) and no
// stash is touched -- for kernels with registers to spare and no shared
// memory to spare (fit_super_kernel).
template <typename T, int METRIC, bool TRAJ, bool STASHED = false, int RL = 1,
          bool REGSTASH = false>
__device__ __forceinline__ T run_propagator(const Prop2<T>& pr, int32_t n_pulse, int32_t n_steps,
                                            const T* __restrict__ rel, T* __restrict__ traj,
                                            int64_t ld_out, T theta0, T sgn,
                                            T* __restrict__ stash, int stash_ld) {
  using V2 = typename Vec2<T>::type;
  // Post-pulse coefficients wait in a per-thread shared-memory stash
  // ([10][stash_ld] of vec2, conflict-free); the phase-independent P2 and
  // P[0] stay in registers for the whole loop.  STASHED: make_prop already
  // wrote them.
  V2* st2 = reinterpret_cast<V2*>(stash) + threadIdx.x;
  if (!STASHED && !REGSTASH) stash_phase<T>(pr.ph[1], st2, stash_ld);
  const PhaseProp2<T>& q0 = pr.ph[0];
  T A00 = q0.X2[0][0], A01 = q0.X2[0][1], A10 = q0.X2[1][0], A11 = q0.X2[1][1];
  T A20 = q0.X2[2][0], A21 = q0.X2[2][1], A30 = q0.X2[3][0], A31 = q0.X2[3][1];
  T c0 = q0.c2[0], c1 = q0.c2[1], c2 = q0.c2[2], c3 = q0.c2[3];
  T pa = q0.pf2[0], pn = q0.pf2[1], qa = q0.qf2[0], qn = q0.qf2[1];
  T x0a = q0.X0[0], x0n = q0.X0[1], d0 = q0.c0;
  const T Q00 = pr.P2[0][0], Q01 = pr.P2[0][1], Q02 = pr.P2[0][2], Q03 = pr.P2[0][3];
  const T Q10 = pr.P2[1][0], Q11 = pr.P2[1][1], Q12 = pr.P2[1][2], Q13 = pr.P2[1][3];
  const T Q20 = pr.P2[2][0], Q21 = pr.P2[2][1], Q22 = pr.P2[2][2], Q23 = pr.P2[2][3];
  const T Q30 = pr.P2[3][0], Q31 = pr.P2[3][1], Q32 = pr.P2[3][2], Q33 = pr.P2[3][3];
  const T R0 = pr.P0[0], R1 = pr.P0[1], R2 = pr.P0[2], R3 = pr.P0[3];
  auto swap_in = [&]() {
    if (REGSTASH) {
      const PhaseProp2<T>& q1 = pr.ph[1];
      A00 = q1.X2[0][0]; A01 = q1.X2[0][1]; A10 = q1.X2[1][0]; A11 = q1.X2[1][1];
      A20 = q1.X2[2][0]; A21 = q1.X2[2][1]; A30 = q1.X2[3][0]; A31 = q1.X2[3][1];
      c0 = q1.c2[0]; c1 = q1.c2[1]; c2 = q1.c2[2]; c3 = q1.c2[3];
      pa = q1.pf2[0]; pn = q1.pf2[1]; qa = q1.qf2[0]; qn = q1.qf2[1];
      x0a = q1.X0[0]; x0n = q1.X0[1]; d0 = q1.c0;
      return;
    }
    V2 v;
    v = st2[0 * stash_ld]; A00 = v.x; A01 = v.y;
    v = st2[1 * stash_ld]; A10 = v.x; A11 = v.y;
    v = st2[2 * stash_ld]; A20 = v.x; A21 = v.y;
    v = st2[3 * stash_ld]; A30 = v.x; A31 = v.y;
    v = st2[4 * stash_ld]; c0 = v.x; c1 = v.y;
    v = st2[5 * stash_ld]; c2 = v.x; c3 = v.y;
    v = st2[6 * stash_ld]; pa = v.x; pn = v.y;
    v = st2[7 * stash_ld]; qa = v.x; qn = v.y;
    v = st2[8 * stash_ld]; x0a = v.x; x0n = v.y;
    v = st2[9 * stash_ld]; d0 = v.x;
  };
  // Lane parity: blocks start at k = o (mod 2) so the pulse end n_pulse falls
  // on a block boundary.  n_pulse == 0 or > n_steps never switches mid-run.
  const bool switches = n_pulse > 0 && n_pulse <= n_steps;
  const int32_t o = switches ? (n_pulse & 1) : 0;
  T th = T(0), om = T(0), xa = T(0), xn = T(0), fa = T(0), fn = T(0);
  T acc = T(0);
  if (TRAJ) traj[0] = theta0;
  if (n_pulse == 0) swap_in();
  if (o) {  // first pulse step from the zero deviation state: z_1 = c, f_1 = qf
    th = pr.z1[0]; om = pr.z1[1]; xa = pr.z1[2]; xn = pr.z1[3];
    fa = pr.f1[0]; fn = pr.f1[1];
    accumulate<METRIC>(acc, TRAJ ? th : th - rel[RL]);
    if (TRAJ) traj[ld_out] = fma(sgn, th, theta0);
  }
  // Block b covers steps k = o + 2b -> k + 2.  Every lane runs nb uniform
  // blocks; the last one may overrun n_steps by one step for odd lanes
  // (masked below).  The lane switches phase before block bs.
  const int32_t nb = (n_steps + 1) / 2;
  const int32_t bs = switches ? (n_pulse - o) / 2 : nb;
  if (switches && bs == 0) swap_in();   // pulse ends before the first block
  const T* __restrict__ rl = rel + o * RL;   // rl[(2b + 1) RL], rl[(2b + 2) RL]
  T* __restrict__ tr = TRAJ ? traj + (int64_t)o * ld_out : traj;
  // Segmented loop over blocks: uniform segments between consecutive lane
  // switch points (warp-min), so the inner loop is pure FMA work; at a
  // segment end only the lanes that switch there reload their coefficients.
  // The callers keep all 32 lanes active.
  int32_t b = 0;
  while (b < nb - 1) {
    const int32_t mine = bs > b ? min(bs, nb - 1) : nb - 1;
    const int32_t seg_end = __reduce_min_sync(0xffffffffu, mine);
#pragma unroll LoopUnroll<T>::value
    for (; b < seg_end; ++b) {
      // The five 6-deep FMA chains (t1 and the four state rows) written level
      // by level, so the scheduler issues them interleaved (ILP 5 against the
      // 8-cycle DFMA latency); each chain's own order -- hence every rounding
      // -- is the nested form fma(P0, th, fma(P1, om, ... fma(X1, fn, c))).
      T t1 = fma(x0n, fn, d0), nth = fma(A01, fn, c0), nom = fma(A11, fn, c1);
      T nxa = fma(A21, fn, c2), nxn = fma(A31, fn, c3);
      t1 = fma(x0a, fa, t1); nth = fma(A00, fa, nth); nom = fma(A10, fa, nom);
      nxa = fma(A20, fa, nxa); nxn = fma(A30, fa, nxn);
      fa = fma(pa, fa, qa);
      fn = fma(pn, fn, qn);
      t1 = fma(R3, xn, t1); nth = fma(Q03, xn, nth); nom = fma(Q13, xn, nom);
      nxa = fma(Q23, xn, nxa); nxn = fma(Q33, xn, nxn);
      t1 = fma(R2, xa, t1); nth = fma(Q02, xa, nth); nom = fma(Q12, xa, nom);
      nxa = fma(Q22, xa, nxa); nxn = fma(Q32, xa, nxn);
      t1 = fma(R1, om, t1); nth = fma(Q01, om, nth); nom = fma(Q11, om, nom);
      nxa = fma(Q21, om, nxa); nxn = fma(Q31, om, nxn);
      t1 = fma(R0, th, t1); nth = fma(Q00, th, nth); nom = fma(Q10, th, nom);
      nxa = fma(Q20, th, nxa); nxn = fma(Q30, th, nxn);
      th = nth; om = nom; xa = nxa; xn = nxn;
      if (TRAJ) {
        accumulate<METRIC>(acc, t1);
        accumulate<METRIC>(acc, th);
        tr[(int64_t)(2 * b + 1) * ld_out] = fma(sgn, t1, theta0);
        tr[(int64_t)(2 * b + 2) * ld_out] = fma(sgn, th, theta0);
      } else {
        accumulate<METRIC>(acc, t1 - rl[(2 * b + 1) * RL]);
        accumulate<METRIC>(acc, th - rl[(2 * b + 2) * RL]);
      }
    }
    if (b == bs) swap_in();
  }
  // last block (b = nb - 1): steps o + 2b + 1 and o + 2b + 2, either of which
  // may lie past n_steps
  if (nb >= 1) {
    const int32_t k1 = o + 2 * b + 1;
    const T t1 = fma(R0, th, fma(R1, om, fma(R2, xa, fma(R3, xn, fma(x0a, fa, fma(x0n, fn, d0))))));
    const T t2 = fma(Q00, th, fma(Q01, om, fma(Q02, xa, fma(Q03, xn, fma(A00, fa, fma(A01, fn, c0))))));
    if (k1 <= n_steps) {
      accumulate<METRIC>(acc, TRAJ ? t1 : t1 - rel[k1 * RL]);
      if (TRAJ) traj[(int64_t)k1 * ld_out] = fma(sgn, t1, theta0);
    }
    if (k1 + 1 <= n_steps) {
      accumulate<METRIC>(acc, TRAJ ? t2 : t2 - rel[(k1 + 1) * RL]);
      if (TRAJ) traj[(int64_t)(k1 + 1) * ld_out] = fma(sgn, t2, theta0);
    }
  }
  return acc;
}

// ----------------------------------------------------------------------------
// Superposition pair (fit_super_kernel): the trajectories b (pulse height 0)
// and u (unit pulse of one channel) of ONE candidate, advanced together.  Both
// use the same maps P2, P[0], X2, X[0], pf2 (they depend on the plant and the
// time constants only); they differ in the forcing terms c2, c[0], qf2 and
// the odd-start state, taken from their own Prop2 (pu's post-pulse forcing is
// zero).  Each recurrence is exactly run_propagator's (same FMA order, so b
// and u are bit-identical to two separate TRAJ runs); the pair gives the
// scheduler 10 independent chains instead of 5.  Every sample k = 0..n_steps
// goes to sink.put(k, b_k, u_k); sink.after_block(b) runs (warp-uniformly)
// after each loop block, when every lane has put all samples <= 2b + 2, and
// sink.finish() at the end.  Returns sum |b_k| and sum |u_k|.
// ----------------------------------------------------------------------------
template <typename Sink>
__device__ __forceinline__ void run_propagator_bu(const Prop2<double>& pb, const UnitForcing& pu,
                                                  int32_t n_pulse, int32_t n_steps, Sink& sink,
                                                  double& Sb, double& Su) {
  const PhaseProp2<double>& q0 = pb.ph[0];
  double A00 = q0.X2[0][0], A01 = q0.X2[0][1], A10 = q0.X2[1][0], A11 = q0.X2[1][1];
  double A20 = q0.X2[2][0], A21 = q0.X2[2][1], A30 = q0.X2[3][0], A31 = q0.X2[3][1];
  double pa = q0.pf2[0], pn = q0.pf2[1];
  double x0a = q0.X0[0], x0n = q0.X0[1];
  // forcing of b and of u
  double c0 = q0.c2[0], c1 = q0.c2[1], c2 = q0.c2[2], c3 = q0.c2[3];
  double qa = q0.qf2[0], qn = q0.qf2[1], d0 = q0.c0;
  double e0 = pu.c2[0], e1 = pu.c2[1], e2 = pu.c2[2], e3 = pu.c2[3];
  double ra = pu.qf2[0], rn = pu.qf2[1], g0 = pu.c0;
  const double Q00 = pb.P2[0][0], Q01 = pb.P2[0][1], Q02 = pb.P2[0][2], Q03 = pb.P2[0][3];
  const double Q10 = pb.P2[1][0], Q11 = pb.P2[1][1], Q12 = pb.P2[1][2], Q13 = pb.P2[1][3];
  const double Q20 = pb.P2[2][0], Q21 = pb.P2[2][1], Q22 = pb.P2[2][2], Q23 = pb.P2[2][3];
  const double Q30 = pb.P2[3][0], Q31 = pb.P2[3][1], Q32 = pb.P2[3][2], Q33 = pb.P2[3][3];
  const double R0 = pb.P0[0], R1 = pb.P0[1], R2 = pb.P0[2], R3 = pb.P0[3];
  auto swap_in = [&]() {
    const PhaseProp2<double>& q1 = pb.ph[1];
    A00 = q1.X2[0][0]; A01 = q1.X2[0][1]; A10 = q1.X2[1][0]; A11 = q1.X2[1][1];
    A20 = q1.X2[2][0]; A21 = q1.X2[2][1]; A30 = q1.X2[3][0]; A31 = q1.X2[3][1];
    pa = q1.pf2[0]; pn = q1.pf2[1];
    x0a = q1.X0[0]; x0n = q1.X0[1];
    c0 = q1.c2[0]; c1 = q1.c2[1]; c2 = q1.c2[2]; c3 = q1.c2[3];
    qa = q1.qf2[0]; qn = q1.qf2[1]; d0 = q1.c0;
    e0 = 0.0; e1 = 0.0; e2 = 0.0; e3 = 0.0;   // u: no post-pulse drive
    ra = 0.0; rn = 0.0; g0 = 0.0;
  };
  const bool switches = n_pulse > 0 && n_pulse <= n_steps;
  const int32_t o = switches ? (n_pulse & 1) : 0;
  double th = 0.0, om = 0.0, xa = 0.0, xn = 0.0, fa = 0.0, fn = 0.0;
  double uth = 0.0, uom = 0.0, uxa = 0.0, uxn = 0.0, ufa = 0.0, ufn = 0.0;
  double sb = 0.0, su = 0.0;
  sink.put(0, 0.0, 0.0);
  if (n_pulse == 0) swap_in();
  if (o) {
    th = pb.z1[0]; om = pb.z1[1]; xa = pb.z1[2]; xn = pb.z1[3]; fa = pb.f1[0]; fn = pb.f1[1];
    uth = pu.z1[0]; uom = pu.z1[1]; uxa = pu.z1[2]; uxn = pu.z1[3]; ufa = pu.f1[0]; ufn = pu.f1[1];
    sb += fabs(th);
    su += fabs(uth);
    sink.put(1, th, uth);
  }
  const int32_t nb = (n_steps + 1) / 2;
  const int32_t bs = switches ? (n_pulse - o) / 2 : nb;
  if (switches && bs == 0) swap_in();
  int32_t b = 0;
  while (b < nb - 1) {
    const int32_t mine = bs > b ? min(bs, nb - 1) : nb - 1;
    const int32_t seg_end = __reduce_min_sync(0xffffffffu, mine);
#pragma unroll 2
    for (; b < seg_end; ++b) {
      double t1 = fma(x0n, fn, d0), nth = fma(A01, fn, c0), nom = fma(A11, fn, c1);
      double nxa = fma(A21, fn, c2), nxn = fma(A31, fn, c3);
      double v1 = fma(x0n, ufn, g0), vth = fma(A01, ufn, e0), vom = fma(A11, ufn, e1);
      double vxa = fma(A21, ufn, e2), vxn = fma(A31, ufn, e3);
      t1 = fma(x0a, fa, t1); nth = fma(A00, fa, nth); nom = fma(A10, fa, nom);
      nxa = fma(A20, fa, nxa); nxn = fma(A30, fa, nxn);
      v1 = fma(x0a, ufa, v1); vth = fma(A00, ufa, vth); vom = fma(A10, ufa, vom);
      vxa = fma(A20, ufa, vxa); vxn = fma(A30, ufa, vxn);
      fa = fma(pa, fa, qa);
      fn = fma(pn, fn, qn);
      ufa = fma(pa, ufa, ra);
      ufn = fma(pn, ufn, rn);
      t1 = fma(R3, xn, t1); nth = fma(Q03, xn, nth); nom = fma(Q13, xn, nom);
      nxa = fma(Q23, xn, nxa); nxn = fma(Q33, xn, nxn);
      v1 = fma(R3, uxn, v1); vth = fma(Q03, uxn, vth); vom = fma(Q13, uxn, vom);
      vxa = fma(Q23, uxn, vxa); vxn = fma(Q33, uxn, vxn);
      t1 = fma(R2, xa, t1); nth = fma(Q02, xa, nth); nom = fma(Q12, xa, nom);
      nxa = fma(Q22, xa, nxa); nxn = fma(Q32, xa, nxn);
      v1 = fma(R2, uxa, v1); vth = fma(Q02, uxa, vth); vom = fma(Q12, uxa, vom);
      vxa = fma(Q22, uxa, vxa); vxn = fma(Q32, uxa, vxn);
      t1 = fma(R1, om, t1); nth = fma(Q01, om, nth); nom = fma(Q11, om, nom);
      nxa = fma(Q21, om, nxa); nxn = fma(Q31, om, nxn);
      v1 = fma(R1, uom, v1); vth = fma(Q01, uom, vth); vom = fma(Q11, uom, vom);
      vxa = fma(Q21, uom, vxa); vxn = fma(Q31, uom, vxn);
      t1 = fma(R0, th, t1); nth = fma(Q00, th, nth); nom = fma(Q10, th, nom);
      nxa = fma(Q20, th, nxa); nxn = fma(Q30, th, nxn);
      v1 = fma(R0, uth, v1); vth = fma(Q00, uth, vth); vom = fma(Q10, uth, vom);
      vxa = fma(Q20, uth, vxa); vxn = fma(Q30, uth, vxn);
      th = nth; om = nom; xa = nxa; xn = nxn;
      uth = vth; uom = vom; uxa = vxa; uxn = vxn;
      sb += fabs(t1);
      sb += fabs(th);
      su += fabs(v1);
      su += fabs(uth);
      sink.put(o + 2 * b + 1, t1, v1);
      sink.put(o + 2 * b + 2, th, uth);
      sink.after_block(b);
    }
    if (b == bs) swap_in();
  }
  if (nb >= 1) {
    const int32_t k1 = o + 2 * b + 1;
    const double t1 = fma(R0, th, fma(R1, om, fma(R2, xa, fma(R3, xn, fma(x0a, fa, fma(x0n, fn, d0))))));
    const double t2 = fma(Q00, th, fma(Q01, om, fma(Q02, xa, fma(Q03, xn, fma(A00, fa, fma(A01, fn, c0))))));
    const double v1 = fma(R0, uth, fma(R1, uom, fma(R2, uxa, fma(R3, uxn, fma(x0a, ufa, fma(x0n, ufn, g0))))));
    const double v2 = fma(Q00, uth, fma(Q01, uom, fma(Q02, uxa, fma(Q03, uxn, fma(A00, ufa, fma(A01, ufn, e0))))));
    if (k1 <= n_steps) {
      sb += fabs(t1);
      su += fabs(v1);
      sink.put(k1, t1, v1);
    }
    if (k1 + 1 <= n_steps) {
      sb += fabs(t2);
      su += fabs(v2);
      sink.put(k1 + 1, t2, v2);
    }
  }
  sink.finish();
  Sb = sb;
  Su = su;
}

// ----------------------------------------------------------------------------
// Fit mode, C candidates per thread (C = 2): the same two-step recurrence as
// run_propagator for C independent candidates interleaved in one thread, so
// the scheduler sees 5C independent FMA chains per block (the fit kernel runs
// 2 warps per scheduler with 255 registers; see fit2_kernel).  Each
// candidate keeps its own lane parity, switch block and trace offset; the
// warp's segments end at the minimum over all its lanes' candidates.
// ----------------------------------------------------------------------------
template <typename T, int METRIC, int C>
__device__ __forceinline__ void run_propagator_multi(const Prop2<T> (&pr)[C],
                                                     const int32_t (&n_pulse)[C], int32_t n_steps,
                                                     const T* __restrict__ rel,
                                                     T* __restrict__ stash, int stash_ld,
                                                     T (&acc)[C]) {
  using V2 = typename Vec2<T>::type;
  V2* st2 = reinterpret_cast<V2*>(stash) + threadIdx.x;
  T Q[C][4][4], R[C][4], A[C][4][2], cc[C][4], pa[C], pn[C], qa[C], qn[C], x0a[C], x0n[C], d0[C];
  T th[C], om[C], xa[C], xn[C], fa[C], fn[C];
  int32_t o[C], bs[C];
  bool sw[C];
  const int32_t nb = (n_steps + 1) / 2;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const PhaseProp2<T>& q = pr[c].ph[1];
    V2* s = st2 + (c * 10) * stash_ld;
    s[0 * stash_ld] = make_v2<T>(q.X2[0][0], q.X2[0][1]);
    s[1 * stash_ld] = make_v2<T>(q.X2[1][0], q.X2[1][1]);
    s[2 * stash_ld] = make_v2<T>(q.X2[2][0], q.X2[2][1]);
    s[3 * stash_ld] = make_v2<T>(q.X2[3][0], q.X2[3][1]);
    s[4 * stash_ld] = make_v2<T>(q.c2[0], q.c2[1]);
    s[5 * stash_ld] = make_v2<T>(q.c2[2], q.c2[3]);
    s[6 * stash_ld] = make_v2<T>(q.pf2[0], q.pf2[1]);
    s[7 * stash_ld] = make_v2<T>(q.qf2[0], q.qf2[1]);
    s[8 * stash_ld] = make_v2<T>(q.X0[0], q.X0[1]);
    s[9 * stash_ld] = make_v2<T>(q.c0, T(0));
    const PhaseProp2<T>& q0 = pr[c].ph[0];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
      for (int j = 0; j < 4; ++j) Q[c][r][j] = pr[c].P2[r][j];
      R[c][r] = pr[c].P0[r];
      A[c][r][0] = q0.X2[r][0];
      A[c][r][1] = q0.X2[r][1];
      cc[c][r] = q0.c2[r];
    }
    pa[c] = q0.pf2[0]; pn[c] = q0.pf2[1]; qa[c] = q0.qf2[0]; qn[c] = q0.qf2[1];
    x0a[c] = q0.X0[0]; x0n[c] = q0.X0[1]; d0[c] = q0.c0;
    sw[c] = n_pulse[c] > 0 && n_pulse[c] <= n_steps;
    o[c] = sw[c] ? (n_pulse[c] & 1) : 0;
    bs[c] = sw[c] ? (n_pulse[c] - o[c]) / 2 : nb;
    th[c] = T(0); om[c] = T(0); xa[c] = T(0); xn[c] = T(0); fa[c] = T(0); fn[c] = T(0);
    acc[c] = T(0);
  }
  auto swap_in = [&](int c) {
    const V2* s = st2 + (c * 10) * stash_ld;
    V2 v;
    v = s[0 * stash_ld]; A[c][0][0] = v.x; A[c][0][1] = v.y;
    v = s[1 * stash_ld]; A[c][1][0] = v.x; A[c][1][1] = v.y;
    v = s[2 * stash_ld]; A[c][2][0] = v.x; A[c][2][1] = v.y;
    v = s[3 * stash_ld]; A[c][3][0] = v.x; A[c][3][1] = v.y;
    v = s[4 * stash_ld]; cc[c][0] = v.x; cc[c][1] = v.y;
    v = s[5 * stash_ld]; cc[c][2] = v.x; cc[c][3] = v.y;
    v = s[6 * stash_ld]; pa[c] = v.x; pn[c] = v.y;
    v = s[7 * stash_ld]; qa[c] = v.x; qn[c] = v.y;
    v = s[8 * stash_ld]; x0a[c] = v.x; x0n[c] = v.y;
    v = s[9 * stash_ld]; d0[c] = v.x;
  };
#pragma unroll
  for (int c = 0; c < C; ++c) {
    if (n_pulse[c] == 0 || (sw[c] && bs[c] == 0)) swap_in(c);
    if (o[c]) {  // first pulse step from the zero deviation state
      th[c] = pr[c].z1[0]; om[c] = pr[c].z1[1]; xa[c] = pr[c].z1[2]; xn[c] = pr[c].z1[3];
      fa[c] = pr[c].f1[0]; fn[c] = pr[c].f1[1];
      accumulate<METRIC>(acc[c], th[c] - rel[1]);
    }
  }
  int32_t b = 0;
  while (b < nb - 1) {
    int32_t mine = nb - 1;
#pragma unroll
    for (int c = 0; c < C; ++c) mine = min(mine, bs[c] > b ? bs[c] : nb - 1);
    const int32_t seg_end = __reduce_min_sync(0xffffffffu, mine);
    for (; b < seg_end; ++b) {
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const T t1 = fma(R[c][0], th[c], fma(R[c][1], om[c], fma(R[c][2], xa[c], fma(R[c][3], xn[c],
                     fma(x0a[c], fa[c], fma(x0n[c], fn[c], d0[c]))))));
        T nz[4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
          nz[r] = fma(Q[c][r][0], th[c], fma(Q[c][r][1], om[c], fma(Q[c][r][2], xa[c],
                  fma(Q[c][r][3], xn[c], fma(A[c][r][0], fa[c], fma(A[c][r][1], fn[c], cc[c][r]))))));
        fa[c] = fma(pa[c], fa[c], qa[c]);
        fn[c] = fma(pn[c], fn[c], qn[c]);
        th[c] = nz[0]; om[c] = nz[1]; xa[c] = nz[2]; xn[c] = nz[3];
        const T* rl = rel + o[c] + 2 * b;
        accumulate<METRIC>(acc[c], t1 - rl[1]);
        accumulate<METRIC>(acc[c], th[c] - rl[2]);
      }
    }
#pragma unroll
    for (int c = 0; c < C; ++c)
      if (b == bs[c]) swap_in(c);
  }
  if (nb >= 1) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const int32_t k1 = o[c] + 2 * b + 1;
      const T t1 = fma(R[c][0], th[c], fma(R[c][1], om[c], fma(R[c][2], xa[c], fma(R[c][3], xn[c],
                   fma(x0a[c], fa[c], fma(x0n[c], fn[c], d0[c]))))));
      const T t2 = fma(Q[c][0][0], th[c], fma(Q[c][0][1], om[c], fma(Q[c][0][2], xa[c],
                   fma(Q[c][0][3], xn[c], fma(A[c][0][0], fa[c], fma(A[c][0][1], fn[c], cc[c][0]))))));
      if (k1 <= n_steps) accumulate<METRIC>(acc[c], t1 - rel[k1]);
      if (k1 + 1 <= n_steps) accumulate<METRIC>(acc[c], t2 - rel[k1 + 1]);
    }
  }
}

// ----------------------------------------------------------------------------
// Integrate + fused score, RK4_STAGES form: the four classical stages
// evaluated literally (SPEC D2), in deviation coordinates, K_i = h f(Y_i).
// ----------------------------------------------------------------------------
template <typename T, int METRIC, bool TRAJ, int RL = 1>
__device__ __forceinline__ T run_rk4_stages(const Setup& s, int32_t n_steps,
                                            const T* __restrict__ rel, T* __restrict__ traj,
                                            int64_t ld_out, T theta0, T sgn, int32_t substeps = 1) {
  const T z01 = (T)s.m.z01, z10 = (T)s.m.z10, z11 = (T)s.m.z11, z12 = (T)s.m.z12,
          z13 = (T)s.m.z13, z20 = (T)s.m.z20, z22 = (T)s.m.z22, z30 = (T)s.m.z30,
          z33 = (T)s.m.z33, hba = (T)s.m.hb_ag, hbn = (T)s.m.hb_ant;
  T y[6] = {T(0), T(0), T(0), T(0), T(0), T(0)};
  T acc = T(0);
  T zda = (T)s.ph[0].zd_ag, zdn = (T)s.ph[0].zd_ant;
  T zna = (T)(s.ph[0].zd_ag * s.ph[0].nt_ag), znn = (T)(s.ph[0].zd_ant * s.ph[0].nt_ant);
  if (TRAJ) traj[0] = theta0;
  const T half = T(0.5), sixth = T(1.0 / 6.0), two = T(2);
  for (int32_t k = 0; k < n_steps; ++k) {
    if (k == s.n_pulse) {
      zda = (T)s.ph[1].zd_ag; zdn = (T)s.ph[1].zd_ant;
      zna = (T)(s.ph[1].zd_ag * s.ph[1].nt_ag); znn = (T)(s.ph[1].zd_ant * s.ph[1].nt_ant);
    }
    for (int32_t sub = 0; sub < substeps; ++sub) {   // reading Q25: control held per sample
      T K[4][6];
      T Y[6];
#pragma unroll
      for (int i = 0; i < 6; ++i) Y[i] = y[i];
#pragma unroll
      for (int st = 0; st < 4; ++st) {
        K[st][0] = z01 * Y[1];
        K[st][1] = fma(z10, Y[0], fma(z11, Y[1], fma(z12, Y[2], z13 * Y[3])));
        K[st][2] = fma(z20, Y[0], fma(z22, Y[2], hba * Y[4]));
        K[st][3] = fma(z30, Y[0], fma(z33, Y[3], hbn * Y[5]));
        K[st][4] = fma(zda, Y[4], -zna);
        K[st][5] = fma(zdn, Y[5], -znn);
        if (st < 3) {
          const T w = st == 2 ? T(1) : half;
#pragma unroll
          for (int i = 0; i < 6; ++i) Y[i] = fma(w, K[st][i], y[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        const T t = fma(two, K[2][i], fma(two, K[1][i], K[0][i])) + K[3][i];
        y[i] = fma(sixth, t, y[i]);
      }
    }
    accumulate<METRIC>(acc, TRAJ ? y[0] : y[0] - rel[(k + 1) * RL]);
    if (TRAJ) traj[(int64_t)(k + 1) * ld_out] = fma(sgn, y[0], theta0);
  }
  return acc;
}

// ---------------------------------------------------------------------------
// Evaluate one candidate: physical check, setup, integrate + fused score.
// ---------------------------------------------------------------------------
template <typename T, int INTEG, int METRIC, bool TRAJ, typename RS = double, int RL = 1>
__device__ __forceinline__ double evaluate(const double p[NP], const CtlDev& c, double Aprime,
                                           double pw_default, const T* rel, T* traj,
                                           int64_t ld_out, double sgn, uint8_t* status,
                                           T* stash, bool check_physical = true,
                                           int stash_ld = -1) {
  // generated candidates skip the check when the host proved the whole
  // search space physical (SpaceDev::all_physical).  A non-physical candidate
  // still runs the (meaningless) recurrence before its penalty is returned:
  // the segmented loop's warp reductions need every lane of the warp.
  const double pen = check_physical ? physical_penalty(p) : 0.0;
  Setup s;
  // INTEG 2 = the propagator with substeps (internal; reading Q25)
  make_setup(p, c.dt_ms, c.h, c.n_steps, Aprime, pw_default, s, INTEG == 0 ? 1 : c.substeps);
  T acc;
  if (INTEG == 0 || INTEG == 2) {
    Prop2<T> pr;
    const int ld = stash_ld < 0 ? (int)blockDim.x : stash_ld;
    typename Vec2<T>::type* st2 = reinterpret_cast<typename Vec2<T>::type*>(stash) + threadIdx.x;
    if (INTEG == 2) {   // sample map = one-substep map ^ substeps (own instantiation)
      make_prop_sub<T>(s, c.substeps, pr, st2, ld);
    } else {
      make_prop<T, true, RS>(s, pr, st2, ld);
    }
    acc = run_propagator<T, METRIC, TRAJ, true, RL>(pr, s.n_pulse, c.n_steps, rel, traj, ld_out,
                                                (T)c.theta0, (T)sgn, stash, ld);
  } else {
    acc = run_rk4_stages<T, METRIC, TRAJ, RL>(s, c.n_steps, rel, traj, ld_out, (T)c.theta0, (T)sgn,
                                          c.substeps);
  }
  if (pen != 0.0) {
    if (TRAJ) {
      const T nanv = (T)__longlong_as_double(0x7ff8000000000000LL);
      for (int32_t k = 0; k <= c.n_steps; ++k) traj[(int64_t)k * ld_out] = nanv;
    }
    if (status) *status = 1;
    return pen;
  }
  const double E = finish_error<METRIC>(acc, c.n_steps + 1);
  if (status) *status = isinf(E) ? 2 : 0;
  return E;
}

// ----------------------------------------------------------------------------
// (E, index) lexicographic order (reading Q12).
// ----------------------------------------------------------------------------
__device__ __forceinline__ bool better(double e1, int64_t i1, double e2, int64_t i2) {
  return e1 < e2 || (e1 == e2 && i1 < i2);
}

__device__ __forceinline__ void warp_argmin(double& e, int64_t& i) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double oe = __shfl_xor_sync(0xffffffffu, e, off);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, i, off);
    if (better(oe, oi, e, i)) { e = oe; i = oi; }
  }
}

}  // namespace opmm
