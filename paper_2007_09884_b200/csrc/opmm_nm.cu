// opmm_nm.cu -- batched parallel Nelder-Mead OPC estimation.
//
// The paper's own estimator: "an original parallel implementation of
// Nelder-Mead based on a serial implementation by Lagarias";
// "all of the simplex transformations are calculated simultaneously"
// (PAPER.md:250), "sorted for accuracy at every iteration",
// dual tolerance exit; Alg. 1 runs one
// optimisation task per saccade.  SPEC D9/D10/D13/D14 fix the initial
// simplex, coefficients, defaults and the stable sort.
//
// B200 mapping: one warp per problem (saccade).  Each iteration the warp
// builds ALL candidate points at once -- reflection, expansion, outside and
// inside contraction and the n shrink points (n + 4 <= 22 points for the
// 18-parameter OPC) -- evaluates one point per lane in parallel, then applies
// the Lagarias decision step and a stable rank sort of the simplex in shared
// memory.  The decision uses only the values the serial algorithm would
// compute, so the iterates are the serial algorithm's; the simplex
// arithmetic uses explicitly rounded fp64 operations (no FMA contraction).
//
// Objectives: the plant error with the propagator or the literal four-stage
// integrator (the fit path's evaluate()), the plant error in the RK4
// definition's reference operation order (opmm_ref_objective, explicitly
// rounded fp64: bit-for-bit the definition's own arithmetic), and the SPEC
// test functions (sphere, Rosenbrock, Powell).
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "opmm.h"
#include "opmm_device.cuh"
#include "opmm_internal.h"

namespace opmm {

// The paper's time-boundary exit (SPEC D13 time_budget): a
// problem stops iterating once its own wall clock (from its start, read from
// %globaltimer in ns) exceeds NmArgs::time_budget_ns (0 = none); exit_reason 2.
__device__ __forceinline__ unsigned long long nm_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}


#define Mr(a, b) __dmul_rn((a), (b))
#define Ar(a, b) __dadd_rn((a), (b))
#define Sr(a, b) __dsub_rn((a), (b))
#define Dr(a, b) __ddiv_rn((a), (b))

// ---------------------------------------------------------------------------
// Plant objective in the RK4 definition's reference operation order: the
// D1 right-hand side and classical RK4 written out as the definition states
// them (absolute coordinates, every quotient an IEEE division), each operation
// explicitly rounded, so the result is the definition's exact fp64 value.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void ref_rhs(const double p[NP], const double y[6], double n_ag,
                                        double n_ant, double tau_ag_ms, double tau_ant_ms,
                                        double dy[6]) {
  const double theta = y[0], omega = y[1], x_ag = y[2], x_ant = y[3], f_ag = y[4], f_ant = y[5];
  const double th_ag = theta, th_ant = -theta;
  const double T_ag = Mr(p[KSE_AG], Sr(x_ag, th_ag));
  const double T_ant = Mr(p[KSE_ANT], Sr(x_ant, th_ant));
  const double tau_ag = Mr(1e-3, tau_ag_ms), tau_ant = Mr(1e-3, tau_ant_ms);
  dy[0] = omega;
  dy[1] = Dr(Sr(Sr(T_ag, T_ant), Mr(p[B_P], omega)), p[J_]);
  dy[2] = Dr(Sr(Sr(Sr(f_ag, Mr(p[NC_AG], th_ag)), Mr(p[KLT_AG], x_ag)), T_ag), p[B_AG]);
  dy[3] = Dr(Sr(Sr(Sr(f_ant, Mr(p[NC_ANT], th_ant)), Mr(p[KLT_ANT], x_ant)), T_ant), p[B_ANT]);
  dy[4] = Dr(Sr(n_ag, f_ag), tau_ag);
  dy[5] = Dr(Sr(n_ant, f_ant), tau_ant);
}

__device__ double ref_objective(const double p_in[NP], const double* rel, int32_t n_steps,
                                double dt_ms, double Aprime, double pw_default, int metric,
                                int32_t substeps, int rel_ld = 1) {
  double p[NP];
#pragma unroll
  for (int d = 0; d < NP; ++d) p[d] = p_in[d];
  if (isnan(p[PW_])) p[PW_] = pw_default;
  // physical check (D8): same rule and summation order as the definition
  {
    bool bad = false;
    double amount = 0.0;
    for (int i = 0; i < NP; ++i) {
      const double v = p[i];
      const bool strict = (i == KSE_AG || i == KSE_ANT || i == B_AG || i == B_ANT || i == J_ ||
                           i == TAU_AC_AG || i == TAU_AC_ANT || i == TAU_DE_AG ||
                           i == TAU_DE_ANT || i == PW_);
      if (!isfinite(v)) { bad = true; amount = Ar(amount, 1.0); continue; }
      if (strict ? !(v > 0.0) : !(v >= 0.0)) {
        bad = true;
        if (v < 0.0) amount = Ar(amount, -v);
      }
    }
    if (!bad) {
      const double g_ag = Dr(p[KSE_AG], Ar(p[KLT_AG], p[KSE_AG]));
      const double g_ant = Dr(p[KSE_ANT], Ar(p[KLT_ANT], p[KSE_ANT]));
      const double G = Ar(Mr(g_ag, Ar(p[NC_AG], p[KLT_AG])), Mr(g_ant, Ar(p[NC_ANT], p[KLT_ANT])));
      if (!(G > 0.0)) bad = true;
    }
    if (bad) return Mr(PENALTY, Ar(1.0, amount));
  }
  const double F = p[NC_FIX];
  const double g_ag = Dr(p[KSE_AG], Ar(p[KLT_AG], p[KSE_AG]));
  const double g_ant = Dr(p[KSE_ANT], Ar(p[KLT_ANT], p[KSE_ANT]));
  const double G = Ar(Mr(g_ag, Ar(p[NC_AG], p[KLT_AG])), Mr(g_ant, Ar(p[NC_ANT], p[KLT_ANT])));
  // fixation equilibrium (n = f = N_C_FIX)
  double ystar[6];
  ystar[0] = Dr(Sr(Mr(g_ag, F), Mr(g_ant, F)), G);
  ystar[1] = 0.0;
  ystar[2] = Dr(Sr(F, Mr(Sr(p[NC_AG], p[KSE_AG]), ystar[0])), Ar(p[KLT_AG], p[KSE_AG]));
  ystar[3] = Dr(Ar(F, Mr(Sr(p[NC_ANT], p[KSE_ANT]), ystar[0])), Ar(p[KLT_ANT], p[KSE_ANT]));
  ystar[4] = F;
  ystar[5] = F;
  // post-pulse step levels (D4 generalised)
  const double delta = Dr(Mr(G, Aprime), Ar(g_ag, g_ant));
  double lv_ag = Ar(F, delta), lv_ant = Sr(F, delta);
  if (lv_ant < NANT_FLOOR) {
    const double theta_star = Dr(Sr(Mr(g_ag, F), Mr(g_ant, F)), G);
    lv_ant = NANT_FLOOR;
    lv_ag = Dr(Ar(Mr(G, Ar(theta_star, Aprime)), Mr(NANT_FLOOR, g_ant)), g_ag);
  }
  const double npd = ceil(Dr(p[PW_], dt_ms));
  const int32_t nsub = substeps > 1 ? substeps : 1;   // reading Q25
  const double h = Dr(Mr(1e-3, dt_ms), (double)nsub);
  const double h2 = Mr(0.5, h), h6 = Dr(h, 6.0);
  double y[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) y[i] = ystar[i];
  double acc = 0.0;   // k = 0 term: |0 - rel_0| = 0
  {
    const double d0 = Sr(Sr(y[0], ystar[0]), rel[0]);   // rel_ld: trace stride
    acc = metric == 0 ? Ar(acc, fabs(d0)) : Ar(acc, Mr(d0, d0));
  }
  for (int32_t k = 0; k < n_steps; ++k) {
    const bool pulse = (double)k < npd;
    const double na = pulse ? p[NSAC_AG] : lv_ag, nn = pulse ? p[NSAC_ANT] : lv_ant;
    const double ta = pulse ? p[TAU_AC_AG] : p[TAU_DE_AG];
    const double tn = pulse ? p[TAU_AC_ANT] : p[TAU_DE_ANT];
    for (int32_t sub = 0; sub < nsub; ++sub) {
      double k1[6], k2[6], k3[6], k4[6], yt[6];
      ref_rhs(p, y, na, nn, ta, tn, k1);
#pragma unroll
      for (int i = 0; i < 6; ++i) yt[i] = Ar(y[i], Mr(h2, k1[i]));
      ref_rhs(p, yt, na, nn, ta, tn, k2);
#pragma unroll
      for (int i = 0; i < 6; ++i) yt[i] = Ar(y[i], Mr(h2, k2[i]));
      ref_rhs(p, yt, na, nn, ta, tn, k3);
#pragma unroll
      for (int i = 0; i < 6; ++i) yt[i] = Ar(y[i], Mr(h, k3[i]));
      ref_rhs(p, yt, na, nn, ta, tn, k4);
#pragma unroll
      for (int i = 0; i < 6; ++i)
        y[i] = Ar(y[i], Mr(h6, Ar(Ar(Ar(k1[i], Mr(2.0, k2[i])), Mr(2.0, k3[i])), k4[i])));
    }
    const double d = Sr(Sr(y[0], ystar[0]), rel[(int64_t)(k + 1) * rel_ld]);
    acc = metric == 0 ? Ar(acc, fabs(d)) : Ar(acc, Mr(d, d));
  }
  if (!(acc < CAP)) return __longlong_as_double(0x7ff0000000000000LL);
  return metric == 0 ? acc : __dsqrt_rn(Dr(acc, (double)(n_steps + 1)));
}

// SPEC acceptance-3 test functions, in the definition's operation order.
__device__ double test_objective(int fn_id, int n, const double* x) {
  double s = 0.0;
  if (fn_id == 0) {
    for (int i = 0; i < n; ++i) s = Ar(s, Mr(x[i], x[i]));
  } else if (fn_id == 1) {
    for (int i = 0; i + 1 < n; ++i) {
      const double a = Sr(x[i + 1], Mr(x[i], x[i])), b = Sr(1.0, x[i]);
      s = Ar(s, Ar(Mr(100.0, Mr(a, a)), Mr(b, b)));
    }
  } else {
    for (int i = 0; i + 3 < n; i += 4) {
      const double a = Ar(x[i], Mr(10.0, x[i + 1])), b = Sr(x[i + 2], x[i + 3]);
      const double c = Sr(x[i + 1], Mr(2.0, x[i + 2])), d = Sr(x[i], x[i + 3]);
      s = Ar(s, Ar(Ar(Ar(Mr(a, a), Mr(5.0, Mr(b, b))), Mr(Mr(c, c), Mr(c, c))),
                   Mr(10.0, Mr(Mr(d, d), Mr(d, d)))));
    }
  }
  return s;
}

// ---------------------------------------------------------------------------
// The batched Nelder-Mead kernel: one warp per problem.
// OBJ: 0 plant/propagator, 1 plant/RK4 stages, 2 plant/reference order,
// 4 plant/propagator with substeps (reading Q25; internal, chosen by the host),
//      3 test function.
// ---------------------------------------------------------------------------
constexpr int NM_NMAX = NP;               // simplex dimension <= 18
constexpr int NM_PTS = NM_NMAX + 4;       // points evaluated per iteration
constexpr int NM_WARPS = 4;               // problems per block
constexpr int NM_THREADS = 32 * NM_WARPS;

struct NmWarpSmem {
  double S[NM_NMAX + 1][NM_NMAX];         // simplex vertices, in fixed slots
  double fs[NM_NMAX + 1];                 // objective per slot
  int ord[2][NM_NMAX + 1];                // slots in sorted order (double-buffered)
  double P[NM_PTS][NM_NMAX];              // xr, xe, xc, xcc, shrink points
  double fp[NM_PTS];
  double xbar[NM_NMAX];
};

// GREL: the relativized trace lives per problem in a global workspace (traces
// too long for shared memory); otherwise per warp in shared memory.  A
// compile-time choice, so the common path's trace loads stay shared-memory
// loads.
template <typename T, int OBJ, int METRIC, bool GREL>
__device__ __forceinline__ void nm_run(const NmArgs& a, unsigned char* smem_raw) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  NmWarpSmem* W = reinterpret_cast<NmWarpSmem*>(smem_raw) + warp;
  const int64_t prob = (int64_t)blockIdx.x * NM_WARPS + warp + a.prob_begin;
  T* rel = GREL ? reinterpret_cast<T*>(a.rel_global) + (prob - a.prob_begin) * (int64_t)(a.ctl.n_steps + 1)
                : reinterpret_cast<T*>(smem_raw + NM_WARPS * sizeof(NmWarpSmem) +
                                       (size_t)warp * rel_bytes<T>(a.ctl.n_steps + 1));
  T* stash = reinterpret_cast<T*>(smem_raw + NM_WARPS * sizeof(NmWarpSmem) +
                                  (GREL ? 0 : NM_WARPS * rel_bytes<T>(a.ctl.n_steps + 1)));
  if (prob >= a.prob_end) return;   // whole warp
  const unsigned long long t0 = __shfl_sync(0xffffffffu, nm_now(), 0);
  const int n = OBJ == 3 ? a.dim : NP;   // plant objectives: always the 18-vector
  const int32_t ns = a.ctl.n_steps + 1;
  double sgn = 1.0, Aprime = 0.0, pwd = 0.0;
  if (OBJ != 3) {
    const double amp = a.sac_ctl[2 * prob];
    pwd = a.sac_ctl[2 * prob + 1];
    const double* rec = a.rec + prob * (int64_t)ns;
    const double r0 = rec[0];
    const double A = isnan(amp) ? rec[ns - 1] - r0 : amp;
    sgn = A < 0.0 ? -1.0 : 1.0;
    Aprime = fabs(A);
    for (int k = lane; k < ns; k += 32) rel[k] = (T)(sgn * (rec[k] - r0));
  }
  __syncwarp();   // every lane reads the whole trace
  // evaluate point x (n coordinates) on every lane; returns f with NaN -> +inf (D11)
  auto evaluate_point = [&](const double* x) -> double {
    double f;
    if (OBJ == 3) {
      f = test_objective(a.fn_id, n, x);
    } else {
      double p[NP];
#pragma unroll
      for (int d = 0; d < NP; ++d) p[d] = x[d];
      if (OBJ == 2) {
        f = ref_objective(p, reinterpret_cast<const double*>(rel), a.ctl.n_steps, a.ctl.dt_ms,
                          Aprime, pwd, METRIC, a.ctl.substeps);
      } else {
        f = evaluate<T, (OBJ == 4 ? 2 : OBJ), METRIC, false>(p, a.ctl, Aprime, pwd, rel, nullptr, 0,
                                                            sgn, nullptr,
                                           stash, true);
      }
    }
    return isnan(f) ? __longlong_as_double(0x7ff0000000000000LL) : f;
  };
  const double* x0 = a.x0 + prob * (int64_t)a.x0_ld;
  // initial simplex (D9): vertex 0 = x0; vertex i = x0 with coordinate i-1
  // scaled by (1 + scale), or scale * 0.00025 when that coordinate is zero.
  int cur = 0;
  {
    const int i = lane <= n ? lane : 0;
    double x[NM_NMAX];
    for (int j = 0; j < n; ++j) {
      double v = x0[j];
      if (OBJ != 3 && j == PW_ && isnan(v)) v = pwd;
      x[j] = v;
    }
    if (i > 0) x[i - 1] = x[i - 1] != 0.0 ? Mr(Ar(1.0, a.init_scale), x[i - 1]) : Mr(a.init_scale, 0.00025);
    const double f = evaluate_point(x);
    if (lane <= n) {
      for (int j = 0; j < n; ++j) W->P[lane][j] = x[j];
      W->fp[lane] = f;
    }
  }
  __syncwarp();
  // The sorted simplex is a permutation ord of fixed vertex slots: replacing
  // the worst vertex writes one slot and re-ranks, instead of copying the
  // whole simplex every iteration.  Order, ties and arithmetic are the serial
  // algorithm's (stable rank by position, D14).
  if (lane <= n) {
    for (int j = 0; j < n; ++j) W->S[lane][j] = W->P[lane][j];
    W->fs[lane] = W->fp[lane];
    const double f = W->fp[lane];
    int rank = 0;
    for (int k = 0; k <= n; ++k) {
      const double g = W->fp[k];
      rank += (g < f || (g == f && k < lane)) ? 1 : 0;
    }
    W->ord[cur][rank] = lane;
  }
  __syncwarp();
  int32_t it = 1, evals = n + 1, gpu_evals = n + 1, reason = 1;
  const double rho = 1.0, chi = 2.0, psi = 0.5, sigma = 0.5;
  while (it < a.max_iter) {
    const int* ord = W->ord[cur];
    const int s0 = ord[0];
    // dual tolerance exit
    bool ok = true;
    if (lane >= 1 && lane <= n) ok = fabs(W->fs[ord[lane]] - W->fs[s0]) <= a.tol_f;
    if (lane < n) {
      const double v0 = W->S[s0][lane];
      for (int i = 1; i <= n; ++i) ok = ok && fabs(W->S[ord[i]][lane] - v0) <= a.tol_x;
    }
    if (__all_sync(0xffffffffu, ok)) { reason = 0; break; }
    if (a.time_budget_ns &&
        __shfl_sync(0xffffffffu, nm_now(), 0) - t0 >= a.time_budget_ns) { reason = 2; break; }
    // centroid of the n best vertices (summed in vertex order, then / n)
    if (lane < n) {
      double sum = 0.0;
      for (int i = 0; i < n; ++i) sum = Ar(sum, W->S[ord[i]][lane]);
      W->xbar[lane] = Dr(sum, (double)n);
    }
    __syncwarp();
    const int sn = ord[n];
    const double f0 = W->fs[s0], fn1 = W->fs[ord[n - 1]], fnn = W->fs[sn];
    // all transformation points at once: lane 0 xr, 1 xe,
    // 2 outside contraction, 3 inside contraction, 4.. shrink of vertex lane-3
    {
      const int L = lane < n + 4 ? lane : 0;
      // Branch-free per coordinate: the four non-shrink points are
      // fl(fl(ca xbar) + fl(cb v_n)) with per-lane (ca, cb) -- bit-identical
      // to the serial forms, since fl(x - y) = fl(x + (-y)) and negation is
      // exact -- and the shrink points fl(v_0 + fl(sigma fl(v_k - v_0))).
      double ca, cb;
      if (L == 0) { ca = Ar(1.0, rho); cb = -rho; }
      else if (L == 1) { const double rc = Mr(rho, chi); ca = Ar(1.0, rc); cb = -rc; }
      else if (L == 2) { const double pr = Mr(psi, rho); ca = Ar(1.0, pr); cb = -pr; }
      else { ca = Sr(1.0, psi); cb = psi; }   // L == 3 (unused by shrink lanes)
      const bool shrink = L >= 4;
      const int sk = ord[shrink ? L - 3 : 0];
      double x[NM_NMAX];
      for (int j = 0; j < n; ++j) {
        const double xb = W->xbar[j], vn = W->S[sn][j], v0 = W->S[s0][j], vkj = W->S[sk][j];
        const double vt = Ar(Mr(ca, xb), Mr(cb, vn));
        const double vs = Ar(v0, Mr(sigma, Sr(vkj, v0)));
        x[j] = shrink ? vs : vt;
      }
      const double f = evaluate_point(x);
      if (lane < n + 4) {
        for (int j = 0; j < n; ++j) W->P[lane][j] = x[j];
        W->fp[lane] = f;
      }
    }
    __syncwarp();
    gpu_evals += n + 4;
    // Lagarias decision step (identical on every lane)
    const double fr = W->fp[0];
    int take = -1;   // point replacing vertex n; -2 = shrink
    if (fr < f0) {
      take = W->fp[1] < fr ? 1 : 0;
      evals += 2;
    } else if (fr < fn1) {
      take = 0;
      evals += 1;
    } else if (fr < fnn) {
      take = W->fp[2] <= fr ? 2 : -2;
      evals += 2;
    } else {
      take = W->fp[3] < fnn ? 3 : -2;
      evals += 2;
    }
    const int nxt = cur ^ 1;
    if (take >= 0) {
      // vertex n (slot sn) replaced by the accepted point, then stable re-rank
      const double fnew = W->fp[take];
      if (lane <= n) {
        const double f = lane == n ? fnew : W->fs[ord[lane]];
        int rank = 0;
        for (int k = 0; k <= n; ++k) {
          const double g = k == n ? fnew : W->fs[ord[k]];
          rank += (g < f || (g == f && k < lane)) ? 1 : 0;
        }
        W->ord[nxt][rank] = lane == n ? sn : ord[lane];
      }
      __syncwarp();
      if (lane < n) W->S[sn][lane] = W->P[take][lane];
      if (lane == 0) W->fs[sn] = fnew;
    } else {
      // shrink: vertices 1..n become the precomputed shrink points
      evals += n;
      if (lane <= n) {
        const double f = lane == 0 ? f0 : W->fp[lane + 3];
        int rank = 0;
        for (int k = 0; k <= n; ++k) {
          const double g = k == 0 ? f0 : W->fp[k + 3];
          rank += (g < f || (g == f && k < lane)) ? 1 : 0;
        }
        W->ord[nxt][rank] = ord[lane];
      }
      __syncwarp();
      if (lane < n)
        for (int i = 1; i <= n; ++i) W->S[ord[i]][lane] = W->P[i + 3][lane];
      if (lane >= 1 && lane <= n) W->fs[ord[lane]] = W->fp[lane + 3];
    }
    __syncwarp();
    cur = nxt;
    ++it;
  }
  const int sb = W->ord[cur][0];
  if (lane < n) a.x_best[prob * (int64_t)a.x_ld + lane] = W->S[sb][lane];
  if (lane == 0) {
    NmOut o;
    o.f_best = W->fs[sb];
    o.iterations = it;
    o.func_evals = evals;
    o.gpu_evals = gpu_evals;
    o.exit_reason = reason;
    a.out[prob] = o;
  }
}

// GREL selects its own instantiation (nm_kernel_ptr), so each kernel holds
// one trace path.
template <typename T, int OBJ, int METRIC, bool GREL>
__global__ void __launch_bounds__(NM_THREADS) nm_kernel(NmArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  nm_run<T, OBJ, METRIC, GREL>(a, smem_raw);
}

template <typename T, int OBJ, int METRIC, bool GREL = false>
static const void* nm_fn() { return reinterpret_cast<const void*>(&nm_kernel<T, OBJ, METRIC, GREL>); }

template <bool G>
static const void* nm_ptr(int precision, int obj, int metric) {
  if (obj == 3) return nm_fn<double, 3, 0, false>();
  if (obj == 2) return metric == 0 ? nm_fn<double, 2, 0, G>() : nm_fn<double, 2, 1, G>();
  if (obj == 4) {
    if (precision == 0) return metric == 0 ? nm_fn<double, 4, 0, G>() : nm_fn<double, 4, 1, G>();
    return metric == 0 ? nm_fn<float, 4, 0, G>() : nm_fn<float, 4, 1, G>();
  }
  if (precision == 0) {
    if (obj == 0) return metric == 0 ? nm_fn<double, 0, 0, G>() : nm_fn<double, 0, 1, G>();
    return metric == 0 ? nm_fn<double, 1, 0, G>() : nm_fn<double, 1, 1, G>();
  }
  if (obj == 0) return metric == 0 ? nm_fn<float, 0, 0, G>() : nm_fn<float, 0, 1, G>();
  return metric == 0 ? nm_fn<float, 1, 0, G>() : nm_fn<float, 1, 1, G>();
}

// ---------------------------------------------------------------------------
// Lane schedule: one problem per LANE (32 per warp).  Each lane runs the
// serial Lagarias iteration and evaluates only the points the decision needs
// (reflection, then expansion or one contraction, shrink points one by one),
// so a lane does ~1.7 evaluations per iteration instead of the n + 4 the
// lock-step schedule spends per problem.  The warp steps its 32 problems
// together: every step each lane builds its next point, all lanes evaluate
// (the propagator loop's segment reductions need the whole warp), and each
// lane applies its own decision.  Lanes whose problem has finished evaluate
// their best vertex and drop the value.  The decisions, the explicitly
// rounded simplex arithmetic and the stable order are the lock-step kernel's,
// so the iterates are the same serial algorithm's.
//
// Shared memory, lane-interleaved ([.][32], conflict-free for any per-lane
// slot): vertex slots S[19][18], f per slot, the centroid, the sorted order;
// the relativized trace rel[k][32] (or the global workspace for long traces);
// the propagator stash.  ~100 KB + the trace per warp: one warp per block.
// ---------------------------------------------------------------------------
constexpr int NML_NV = NM_NMAX + 1;
enum { NML_INIT = 0, NML_R, NML_E, NML_OC, NML_IC, NML_SHRINK, NML_DONE };

__host__ __device__ constexpr size_t nml_fixed_bytes() {
  return (size_t)32 * (NML_NV * NM_NMAX * 8 + NML_NV * 8 + NM_NMAX * 8 + NML_NV * 4);
}

template <typename T, int OBJ, int METRIC, bool GREL>
__global__ void __launch_bounds__(32, 1) nm_lane_kernel(NmArgs a) {
  using RT = typename std::conditional<OBJ == 2, double, T>::type;   // trace type
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x;
  double* S = reinterpret_cast<double*>(smem_raw);         // [slot][j][32]
  double* FSv = S + NML_NV * NM_NMAX * 32;                  // [slot][32]
  double* XBv = FSv + NML_NV * 32;                          // [j][32]
  int* ORDv = reinterpret_cast<int*>(XBv + NM_NMAX * 32);   // [pos][32]
  unsigned char* rest = smem_raw + nml_fixed_bytes();
  T* stash = reinterpret_cast<T*>(rest);
  if (OBJ != 3 && OBJ != 2) rest += stash_bytes<T>(32);
  const int32_t ns = a.ctl.n_steps + 1;
  RT* rel = (GREL ? reinterpret_cast<RT*>(a.rel_global) + (int64_t)blockIdx.x * ns * 32
                  : reinterpret_cast<RT*>(rest)) + lane;    // rel[k * 32]
#define SV(slot, j) S[((slot) * NM_NMAX + (j)) * 32 + lane]
#define FS(slot) FSv[(slot) * 32 + lane]
#define XB(j) XBv[(j) * 32 + lane]
#define ORD(p) ORDv[(p) * 32 + lane]
  const int64_t prob_raw = (int64_t)blockIdx.x * 32 + lane + a.prob_begin;
  const bool live = prob_raw < a.prob_end;
  const int64_t prob = live ? prob_raw : a.prob_end - 1;   // pad lanes mirror the last problem
  const unsigned long long t0 = nm_now();
  const int n = OBJ == 3 ? a.dim : NP;
  double sgn = 1.0, Aprime = 0.0, pwd = 0.0;
  if (OBJ != 3) {
    const double amp = a.sac_ctl[2 * prob];
    pwd = a.sac_ctl[2 * prob + 1];
    const double* rec = a.rec + prob * (int64_t)ns;
    const double r0 = rec[0];
    const double A = isnan(amp) ? rec[ns - 1] - r0 : amp;
    sgn = A < 0.0 ? -1.0 : 1.0;
    Aprime = fabs(A);
    for (int k = 0; k < ns; ++k) rel[(int64_t)k * 32] = (RT)(sgn * (rec[k] - r0));
  }
  const double* x0 = a.x0 + prob * (int64_t)a.x0_ld;
  const double rho = 1.0, chi = 2.0, psi = 0.5, sigma = 0.5;
  // (ca, cb) of the four non-shrink points, as the lock-step kernel forms them
  auto coefs = [&](int st, double& ca, double& cb) {
    if (st == NML_R) { ca = Ar(1.0, rho); cb = -rho; }
    else if (st == NML_E) { const double rc = Mr(rho, chi); ca = Ar(1.0, rc); cb = -rc; }
    else if (st == NML_OC) { const double pr = Mr(psi, rho); ca = Ar(1.0, pr); cb = -pr; }
    else { ca = Sr(1.0, psi); cb = psi; }
  };
  int st = NML_INIT, k = 0, sn = 0, s0 = 0;
  int32_t it = 1, evals = n + 1, gpu_evals = 0, reason = 1;
  double fr = 0.0, f0 = 0.0, fn1 = 0.0, fnn = 0.0;
  // point of state (st, k); deterministic, so an accepted point is rebuilt
  // bit-identically instead of being kept across the evaluation
  auto build = [&](int s, int kk, double* x) {
    if (s == NML_INIT) {
#pragma unroll
      for (int j = 0; j < NM_NMAX; ++j) {
        if (j < n) {
          double v = x0[j];
          if (OBJ != 3 && j == PW_ && isnan(v)) v = pwd;
          if (kk > 0 && j == kk - 1) v = v != 0.0 ? Mr(Ar(1.0, a.init_scale), v) : Mr(a.init_scale, 0.00025);
          x[j] = v;
        }
      }
    } else if (s == NML_SHRINK) {
      const int sk = ORD(kk);
#pragma unroll
      for (int j = 0; j < NM_NMAX; ++j)
        if (j < n) { const double v0 = SV(s0, j); x[j] = Ar(v0, Mr(sigma, Sr(SV(sk, j), v0))); }
    } else if (s == NML_DONE) {
      const int sb = ORD(0);
#pragma unroll
      for (int j = 0; j < NM_NMAX; ++j)
        if (j < n) x[j] = SV(sb, j);
    } else {
      double ca, cb;
      coefs(s, ca, cb);
#pragma unroll
      for (int j = 0; j < NM_NMAX; ++j)
        if (j < n) x[j] = Ar(Mr(ca, XB(j)), Mr(cb, SV(sn, j)));
    }
  };
  // start an iteration: exit tests, centroid, the decision's reference values
  auto begin_iteration = [&]() {
    if (!(it < a.max_iter)) { st = NML_DONE; return; }
    // (loops ordered so each vertex's 18 loads are independent: one warp
    // per SM leaves shared-memory latency exposed otherwise)
    s0 = ORD(0);
    bool ok = true;
    {
      const double fb = FS(s0);
      for (int p = 1; p <= n; ++p) ok &= fabs(FS(ORD(p)) - fb) <= a.tol_f;
    }
    if (ok) {
      double v0[NM_NMAX];
#pragma unroll
      for (int j = 0; j < NM_NMAX; ++j) v0[j] = j < n ? SV(s0, j) : 0.0;
      for (int p = 1; p <= n; ++p) {
        const int sp = ORD(p);
#pragma unroll
        for (int j = 0; j < NM_NMAX; ++j)
          if (j < n) ok &= fabs(SV(sp, j) - v0[j]) <= a.tol_x;
      }
    }
    if (ok) { st = NML_DONE; reason = 0; return; }
    if (a.time_budget_ns && nm_now() - t0 >= a.time_budget_ns) { st = NML_DONE; reason = 2; return; }
    {
      // centroid of the n best, summed per coordinate in vertex order
      double sum[NM_NMAX];
#pragma unroll
      for (int j = 0; j < NM_NMAX; ++j) sum[j] = 0.0;
      for (int i = 0; i < n; ++i) {
        const int si = ORD(i);
#pragma unroll
        for (int j = 0; j < NM_NMAX; ++j)
          if (j < n) sum[j] = Ar(sum[j], SV(si, j));
      }
#pragma unroll
      for (int j = 0; j < NM_NMAX; ++j)
        if (j < n) XB(j) = Dr(sum[j], (double)n);
    }
    sn = ORD(n);
    f0 = FS(s0);
    fn1 = FS(ORD(n - 1));
    fnn = FS(sn);
    st = NML_R;
  };
  // stable sort of positions 0..n by f (insertion; equal values keep order)
  auto sort_all = [&]() {
    for (int p = 1; p <= n; ++p) {
      const int key = ORD(p);
      const double fk = FS(key);
      int q = p - 1;
      while (q >= 0 && FS(ORD(q)) > fk) { ORD(q + 1) = ORD(q); --q; }
      ORD(q + 1) = key;
    }
  };
  if (!live) st = NML_DONE;
  if (!live) {   // a pad lane still needs a valid point to evaluate
#pragma unroll
    for (int j = 0; j < NM_NMAX; ++j)
      if (j < n) SV(0, j) = x0[j];
    ORD(0) = 0;
  }
  while (!__all_sync(0xffffffffu, st == NML_DONE)) {
    double f;
    {
      double x[NM_NMAX];
      build(st, k, x);
      if (OBJ == 3) {
        f = test_objective(a.fn_id, n, x);
      } else {
        double p[NP];
#pragma unroll
        for (int d = 0; d < NP; ++d) p[d] = x[d];
        __syncwarp();
        if (OBJ == 2) {
          f = ref_objective(p, reinterpret_cast<const double*>(rel), a.ctl.n_steps, a.ctl.dt_ms,
                            Aprime, pwd, METRIC, a.ctl.substeps, 32);
        } else {
          f = evaluate<T, (OBJ == 4 ? 2 : OBJ), METRIC, false, double, 32>(
              p, a.ctl, Aprime, pwd, reinterpret_cast<const T*>(rel), nullptr, 0, sgn, nullptr,
              stash, true, 32);
        }
      }
      if (isnan(f)) f = __longlong_as_double(0x7ff0000000000000LL);
    }
    if (st == NML_DONE) continue;
    ++gpu_evals;
    // Decide; every write below has a single call site (one warp per SM:
    // the instruction cache is worth keeping small).
    int put_state = -1, put_k = 0, put_slot = 0;   // point to store, if any
    double put_f = f;
    bool accept = false, resort = false, next = false;
    switch (st) {
      case NML_INIT:   // vertex k of the initial simplex, in slot k
        put_state = NML_INIT; put_k = k; put_slot = k;
        ORD(k) = k;
        if (++k > n) { resort = true; next = true; }
        break;
      case NML_R:
        fr = f;
        if (fr < f0) st = NML_E;
        else if (fr < fn1) { evals += 1; accept = true; put_state = NML_R; }
        else if (fr < fnn) st = NML_OC;
        else st = NML_IC;
        break;
      case NML_E:
        evals += 2;
        accept = true;
        if (f < fr) put_state = NML_E;
        else { put_state = NML_R; put_f = fr; }
        break;
      case NML_OC:
      case NML_IC:
        evals += 2;
        if (st == NML_OC ? f <= fr : f < fnn) { accept = true; put_state = st; }
        else { st = NML_SHRINK; k = 1; }
        break;
      case NML_SHRINK:
        // shrink point k replaces the vertex at sorted position k (its old
        // coordinates feed only this point)
        put_state = NML_SHRINK; put_k = k; put_slot = ORD(k);
        if (++k > n) { evals += n; resort = true; ++it; next = true; }
        break;
      default: break;
    }
    if (accept) { put_slot = sn; ++it; next = true; }
    if (put_state >= 0) {
      double x[NM_NMAX];
      build(put_state, put_k, x);
#pragma unroll
      for (int j = 0; j < NM_NMAX; ++j)
        if (j < n) SV(put_slot, j) = x[j];
      FS(put_slot) = put_f;
    }
    if (accept) {   // vertex n replaced: stable re-rank of position n
      int q = n - 1;
      while (q >= 0 && FS(ORD(q)) > put_f) { ORD(q + 1) = ORD(q); --q; }
      ORD(q + 1) = sn;
    }
    if (resort) sort_all();
    if (next) begin_iteration();
  }
  if (live) {
    const int sb = ORD(0);
    for (int j = 0; j < n; ++j) a.x_best[prob * (int64_t)a.x_ld + j] = SV(sb, j);
    NmOut o;
    o.f_best = FS(sb);
    o.iterations = it;
    o.func_evals = evals;
    o.gpu_evals = gpu_evals;
    o.exit_reason = reason;
    a.out[prob] = o;
  }
#undef SV
#undef FS
#undef XB
#undef ORD
}

// ---------------------------------------------------------------------------
// Group schedule: 4 lanes per problem, 8 problems per warp.  The paper's
// "all transformations simultaneously" sized to what the
// decision can use: every iteration the group evaluates the reflection, the
// expansion and both contractions at once (lanes q = 0..3), so an iteration
// costs one evaluation of latency; the shrink points (rare) and the initial
// vertices go 4 at a time.  The centroid and the exit tests are split over
// the group's lanes by coordinate.  Same decisions, same explicitly rounded
// arithmetic, same stable order as the other schedules: the same runs.
// Shared memory ~40 KB per warp (problems interleaved [.][8]): ~5 warps/SM.
// ---------------------------------------------------------------------------
constexpr int NMQ_G = 4;              // lanes per problem
constexpr int NMQ_P = 32 / NMQ_G;     // problems per warp
enum { NMQ_INIT = 0, NMQ_ITER, NMQ_SHRINK, NMQ_DONE };

__host__ __device__ constexpr size_t nmq_fixed_bytes() {
  return (size_t)NMQ_P * (NML_NV * NM_NMAX * 8 + NML_NV * 8 + NM_NMAX * 8 + NML_NV * 4);
}

template <typename T, int OBJ, int METRIC, bool GREL>
__global__ void __launch_bounds__(32) nm_group_kernel(NmArgs a) {
  using RT = typename std::conditional<OBJ == 2, double, T>::type;   // trace type
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x, g = lane >> 2, q = lane & 3;
  const unsigned gmask = 0xFu << (4 * g);
  double* S = reinterpret_cast<double*>(smem_raw);           // [slot][j][8]
  double* FSv = S + NML_NV * NM_NMAX * NMQ_P;                 // [slot][8]
  double* XBv = FSv + NML_NV * NMQ_P;                         // [j][8]
  int* ORDv = reinterpret_cast<int*>(XBv + NM_NMAX * NMQ_P);  // [pos][8]
  unsigned char* rest = smem_raw + nmq_fixed_bytes();
  T* stash = reinterpret_cast<T*>(rest);
  if (OBJ != 3 && OBJ != 2) rest += stash_bytes<T>(32);
  const int32_t ns = a.ctl.n_steps + 1;
  RT* rel = (GREL ? reinterpret_cast<RT*>(a.rel_global) + (int64_t)blockIdx.x * ns * NMQ_P
                  : reinterpret_cast<RT*>(rest)) + g;         // rel[k * 8]
#define SV(slot, j) S[((slot) * NM_NMAX + (j)) * NMQ_P + g]
#define FS(slot) FSv[(slot) * NMQ_P + g]
#define XB(j) XBv[(j) * NMQ_P + g]
#define ORD(p) ORDv[(p) * NMQ_P + g]
  // Problem refill (a.nm_next != nullptr): the grid is one wave of resident
  // blocks, and a group whose problem is done takes the next unassigned one
  // from the global counter, so problems that stop early no longer leave
  // their slots idle until the whole wave ends.  Each problem's run is the
  // same whichever slot runs it.
  int64_t prob_raw = (int64_t)blockIdx.x * NMQ_P + g + a.prob_begin;
  bool live = prob_raw < a.prob_end;
  int64_t prob = live ? prob_raw : a.prob_end - 1;   // pad groups mirror the last problem
  unsigned long long t0 = 0;
  const int n = OBJ == 3 ? a.dim : NP;
  double sgn = 1.0, Aprime = 0.0, pwd = 0.0;
  const double* x0 = nullptr;
  // stage problem `prob`: its relativized trace in the group's slot, the
  // start vector, and the group-uniform start of its clock
  auto load_problem = [&]() {
    t0 = __shfl_sync(gmask, nm_now(), 4 * g);
    if (OBJ != 3) {
      const double amp = a.sac_ctl[2 * prob];
      pwd = a.sac_ctl[2 * prob + 1];
      const double* rec = a.rec + prob * (int64_t)ns;
      const double r0 = rec[0];
      const double A = isnan(amp) ? rec[ns - 1] - r0 : amp;
      sgn = A < 0.0 ? -1.0 : 1.0;
      Aprime = fabs(A);
      for (int k = q; k < ns; k += NMQ_G) rel[(int64_t)k * NMQ_P] = (RT)(sgn * (rec[k] - r0));
    }
    x0 = a.x0 + prob * (int64_t)a.x0_ld;
  };
  load_problem();
  const double rho = 1.0, chi = 2.0, psi = 0.5, sigma = 0.5;
  auto coefs = [&](int t, double& ca, double& cb) {   // t: 0 xr, 1 xe, 2 xc, 3 xcc
    if (t == 0) { ca = Ar(1.0, rho); cb = -rho; }
    else if (t == 1) { const double rc = Mr(rho, chi); ca = Ar(1.0, rc); cb = -rc; }
    else if (t == 2) { const double pr = Mr(psi, rho); ca = Ar(1.0, pr); cb = -pr; }
    else { ca = Sr(1.0, psi); cb = psi; }
  };
  auto x0_coord = [&](int v, int j) {   // coordinate j of initial vertex v
    double x = x0[j];
    if (OBJ != 3 && j == PW_ && isnan(x)) x = pwd;
    if (v > 0 && j == v - 1) x = x != 0.0 ? Mr(Ar(1.0, a.init_scale), x) : Mr(a.init_scale, 0.00025);
    return x;
  };
  // group-uniform state (every lane of the group keeps the same copy)
  int st = NMQ_INIT, k = 0, sn = 0, s0 = 0;
  int32_t it = 1, evals = n + 1, gpu_evals = 0, reason = 1;
  double f0 = 0.0, fn1 = 0.0, fnn = 0.0;
  // the finished problem's result, written as soon as it is known
  auto retire = [&]() {
    __syncwarp(gmask);
    const int sb = ORD(0);
    for (int j = q; j < n; j += NMQ_G) a.x_best[prob * (int64_t)a.x_ld + j] = SV(sb, j);
    if (q == 0) {
      NmOut o;
      o.f_best = FS(sb);
      o.iterations = it;
      o.func_evals = evals;
      o.gpu_evals = gpu_evals;
      o.exit_reason = reason;
      a.out[prob] = o;
    }
    live = false;
  };
  // refill: the next unassigned problem, if any (group-uniform)
  bool drained = a.nm_next == nullptr;
  auto take_next = [&]() {
    unsigned long long nx = 0;
    if (q == 0) nx = atomicAdd(a.nm_next, 1ull);
    nx = __shfl_sync(gmask, nx, 4 * g);
    if ((int64_t)nx >= a.prob_end) { drained = true; return; }
    prob = (int64_t)nx;
    live = true;
    __syncwarp(gmask);
    load_problem();
    __syncwarp(gmask);
    st = NMQ_INIT;
    k = 0;
    it = 1;
    evals = n + 1;
    gpu_evals = 0;
    reason = 1;
  };
  auto sort_all = [&]() {   // lane q = 0; stable insertion sort of positions 0..n by f
    for (int p = 1; p <= n; ++p) {
      const int key = ORD(p);
      const double fk = FS(key);
      int r = p - 1;
      while (r >= 0 && FS(ORD(r)) > fk) { ORD(r + 1) = ORD(r); --r; }
      ORD(r + 1) = key;
    }
  };
  // all 4 lanes of the group, group-uniform control flow.  The sorted order
  // is read once into registers so every vertex load below is independent
  // (a few warps per SM leave shared-memory latency exposed otherwise); the
  // f test runs first and the coordinate test only when it passes (the exit
  // needs both).
  auto begin_iteration = [&]() {
    if (!(it < a.max_iter)) { st = NMQ_DONE; return; }
    int o[NML_NV];
#pragma unroll
    for (int p = 0; p < NML_NV; ++p) o[p] = p <= n ? ORD(p) : 0;
    s0 = o[0];
    const double fb = FS(s0);
    bool ok = true;
#pragma unroll
    for (int p = 1; p < NML_NV; ++p)
      if (p <= n && (p & 3) == q) ok &= fabs(FS(o[p]) - fb) <= a.tol_f;
    ok = __all_sync(gmask, ok);
    if (ok) {
#pragma unroll
      for (int jj = 0; jj < (NM_NMAX + NMQ_G - 1) / NMQ_G; ++jj) {
        const int j = q + NMQ_G * jj;
        if (j < n) {
          const double v0 = SV(s0, j);
#pragma unroll
          for (int p = 1; p < NML_NV; ++p)
            if (p <= n) ok &= fabs(SV(o[p], j) - v0) <= a.tol_x;
        }
      }
      if (__all_sync(gmask, ok)) { st = NMQ_DONE; reason = 0; return; }
    }
    if (a.time_budget_ns &&
        __shfl_sync(gmask, nm_now(), 4 * g) - t0 >= a.time_budget_ns) { st = NMQ_DONE; reason = 2; return; }
#pragma unroll
    for (int jj = 0; jj < (NM_NMAX + NMQ_G - 1) / NMQ_G; ++jj) {   // centroid, in vertex order
      const int j = q + NMQ_G * jj;
      if (j < n) {
        double sum = 0.0;
#pragma unroll
        for (int i = 0; i < NM_NMAX; ++i)
          if (i < n) sum = Ar(sum, SV(o[i], j));
        XB(j) = Dr(sum, (double)n);
      }
    }
    __syncwarp(gmask);
    sn = o[n];
    f0 = fb;
    fn1 = FS(o[n - 1]);
    fnn = FS(sn);
    st = NMQ_ITER;
  };
  if (!live) {
    if (q == 0) {
      for (int j = 0; j < n; ++j) SV(0, j) = x0[j];
      ORD(0) = 0;
    }
    st = NMQ_DONE;
  }
  __syncwarp();
  for (;;) {
    if (st == NMQ_DONE) {   // group-uniform
      if (live) retire();
      if (!drained) take_next();
    }
    if (__all_sync(0xffffffffu, st == NMQ_DONE)) break;
    double f;
    {
      // this lane's point: vertex / transformation / shrink point / best vertex
      double x[NM_NMAX];
      if (st == NMQ_INIT) {
        const int v = k + q <= n ? k + q : 0;
#pragma unroll
        for (int j = 0; j < NM_NMAX; ++j)
          if (j < n) x[j] = x0_coord(v, j);
      } else if (st == NMQ_ITER) {
        double ca, cb;
        coefs(q, ca, cb);
#pragma unroll
        for (int j = 0; j < NM_NMAX; ++j)
          if (j < n) x[j] = Ar(Mr(ca, XB(j)), Mr(cb, SV(sn, j)));
      } else if (st == NMQ_SHRINK) {
        const int sk = ORD(k + q <= n ? k + q : 0);
#pragma unroll
        for (int j = 0; j < NM_NMAX; ++j)
          if (j < n) { const double v0 = SV(s0, j); x[j] = Ar(v0, Mr(sigma, Sr(SV(sk, j), v0))); }
      } else {
        const int sb = ORD(0);
#pragma unroll
        for (int j = 0; j < NM_NMAX; ++j)
          if (j < n) x[j] = SV(sb, j);
      }
      if (OBJ == 3) {
        f = test_objective(a.fn_id, n, x);
      } else {
        double p[NP];
#pragma unroll
        for (int d = 0; d < NP; ++d) p[d] = x[d];
        __syncwarp();
        if (OBJ == 2) {
          f = ref_objective(p, reinterpret_cast<const double*>(rel), a.ctl.n_steps, a.ctl.dt_ms,
                            Aprime, pwd, METRIC, a.ctl.substeps, NMQ_P);
        } else {
          f = evaluate<T, (OBJ == 4 ? 2 : OBJ), METRIC, false, double, NMQ_P>(
              p, a.ctl, Aprime, pwd, reinterpret_cast<const T*>(rel), nullptr, 0, sgn, nullptr,
              stash, true, 32);
        }
      }
      if (isnan(f)) f = __longlong_as_double(0x7ff0000000000000LL);
    }
    // the group's four values (full-warp shuffles, before any group branch)
    const double fq0 = __shfl_sync(0xffffffffu, f, g * NMQ_G + 0);
    const double fq1 = __shfl_sync(0xffffffffu, f, g * NMQ_G + 1);
    const double fq2 = __shfl_sync(0xffffffffu, f, g * NMQ_G + 2);
    const double fq3 = __shfl_sync(0xffffffffu, f, g * NMQ_G + 3);
    if (st == NMQ_DONE) continue;
    if (st == NMQ_INIT || st == NMQ_SHRINK) {
      // store this lane's point (rebuilt bit-identically) into its slot
      const int pos = k + q;
      const int m = n + 1 - k < NMQ_G ? n + 1 - k : NMQ_G;   // points this step
      gpu_evals += m;
      if (pos <= n) {
        const int slot = st == NMQ_INIT ? pos : ORD(pos);
        if (st == NMQ_INIT) {
          for (int j = 0; j < n; ++j) SV(slot, j) = x0_coord(pos, j);
          ORD(pos) = pos;
        } else {
          for (int j = 0; j < n; ++j) {
            const double v0 = SV(s0, j);
            SV(slot, j) = Ar(v0, Mr(sigma, Sr(SV(slot, j), v0)));
          }
        }
        FS(slot) = f;
      }
      k += NMQ_G;
      if (k > n) {
        const bool shrink = st == NMQ_SHRINK;
        if (shrink) { evals += n; ++it; }
        __syncwarp(gmask);
        if (q == 0) sort_all();
        __syncwarp(gmask);
        begin_iteration();
      }
      continue;
    }
    // NMQ_ITER: the Lagarias decision on (fr, fe, fc, fcc)
    gpu_evals += NMQ_G;
    const double fr = fq0;
    int take;   // 0..3 = point replacing vertex n; -1 = shrink
    double ftake = fr;
    if (fr < f0) {
      evals += 2;
      take = fq1 < fr ? 1 : 0;
      ftake = take == 1 ? fq1 : fr;
    } else if (fr < fn1) {
      evals += 1;
      take = 0;
    } else if (fr < fnn) {
      evals += 2;
      take = fq2 <= fr ? 2 : -1;
      ftake = fq2;
    } else {
      evals += 2;
      take = fq3 < fnn ? 3 : -1;
      ftake = fq3;
    }
    if (take < 0) { st = NMQ_SHRINK; k = 1; continue; }
    {
      double ca, cb;
      coefs(take, ca, cb);
      for (int j = q; j < n; j += NMQ_G) SV(sn, j) = Ar(Mr(ca, XB(j)), Mr(cb, SV(sn, j)));
    }
    // vertex n replaced: stable re-rank of position n.  Positions 0..n-1 are
    // sorted, so the new vertex goes after every f <= its own (equal values
    // keep their order), i.e. at rank = #{r < n : f_r <= f_new}; the group
    // counts in parallel and shifts positions rank..n-1 up by one.
    {
      int cnt = 0, keep[(NM_NMAX + NMQ_G - 1) / NMQ_G];
#pragma unroll
      for (int rr = 0; rr < (NM_NMAX + NMQ_G - 1) / NMQ_G; ++rr) {
        const int r = q + NMQ_G * rr;
        keep[rr] = r < n ? ORD(r) : 0;
        if (r < n) cnt += FS(keep[rr]) <= ftake ? 1 : 0;
      }
      const int rank = __reduce_add_sync(gmask, cnt);
      __syncwarp(gmask);
#pragma unroll
      for (int rr = 0; rr < (NM_NMAX + NMQ_G - 1) / NMQ_G; ++rr) {
        const int r = q + NMQ_G * rr;
        if (r < n && r >= rank) ORD(r + 1) = keep[rr];
      }
      __syncwarp(gmask);
      if (q == 0) { FS(sn) = ftake; ORD(rank) = sn; }
      __syncwarp(gmask);
    }
    ++it;
    begin_iteration();
  }
#undef SV
#undef FS
#undef XB
#undef ORD
}

template <typename T, int OBJ, int METRIC, bool GREL = false>
static const void* nmg_fn() { return reinterpret_cast<const void*>(&nm_group_kernel<T, OBJ, METRIC, GREL>); }

template <bool G>
static const void* nmg_ptr(int precision, int obj, int metric) {
  if (obj == 3) return nmg_fn<double, 3, 0, false>();
  if (obj == 2) return metric == 0 ? nmg_fn<double, 2, 0, G>() : nmg_fn<double, 2, 1, G>();
  if (obj == 4) {
    if (precision == 0) return metric == 0 ? nmg_fn<double, 4, 0, G>() : nmg_fn<double, 4, 1, G>();
    return metric == 0 ? nmg_fn<float, 4, 0, G>() : nmg_fn<float, 4, 1, G>();
  }
  if (precision == 0) {
    if (obj == 0) return metric == 0 ? nmg_fn<double, 0, 0, G>() : nmg_fn<double, 0, 1, G>();
    return metric == 0 ? nmg_fn<double, 1, 0, G>() : nmg_fn<double, 1, 1, G>();
  }
  if (obj == 0) return metric == 0 ? nmg_fn<float, 0, 0, G>() : nmg_fn<float, 0, 1, G>();
  return metric == 0 ? nmg_fn<float, 1, 0, G>() : nmg_fn<float, 1, 1, G>();
}

const void* nm_group_kernel_ptr(int precision, int obj, int metric, bool rel_global) {
  return rel_global ? nmg_ptr<true>(precision, obj, metric) : nmg_ptr<false>(precision, obj, metric);
}

size_t nm_group_smem(int precision, int obj, int32_t n_samples, bool rel_in_smem) {
  const bool f32 = precision != 0 && obj != 2 && obj != 3;
  size_t b = nmq_fixed_bytes();
  if (obj == 0 || obj == 1 || obj == 4) b += f32 ? stash_bytes<float>(32) : stash_bytes<double>(32);
  if (rel_in_smem && obj != 3) b += (size_t)n_samples * NMQ_P * (f32 ? sizeof(float) : sizeof(double));
  return b;
}

int nm_group_problems_per_block() { return NMQ_P; }

// rel_global: the instantiation that reads the trace from the global workspace
const void* nm_kernel_ptr(int precision, int obj, int metric, bool rel_global) {
  return rel_global ? nm_ptr<true>(precision, obj, metric) : nm_ptr<false>(precision, obj, metric);
}

size_t nm_smem(int precision, int obj, int32_t n_samples, bool rel_in_smem) {
  const size_t relb = !rel_in_smem ? 0
                      : (obj == 2 || precision == 0) ? rel_bytes<double>(n_samples)
                                                     : rel_bytes<float>(n_samples);
  const size_t st = precision == 0 || obj >= 2 ? stash_bytes<double>(NM_THREADS)
                                               : stash_bytes<float>(NM_THREADS);
  return NM_WARPS * sizeof(NmWarpSmem) + NM_WARPS * (obj == 3 ? 0 : relb) + (obj < 2 || obj == 4 ? st : 0);
}

template <typename T, int OBJ, int METRIC, bool GREL = false>
static const void* nml_fn() { return reinterpret_cast<const void*>(&nm_lane_kernel<T, OBJ, METRIC, GREL>); }

template <bool G>
static const void* nml_ptr(int precision, int obj, int metric) {
  if (obj == 3) return nml_fn<double, 3, 0, false>();
  if (obj == 2) return metric == 0 ? nml_fn<double, 2, 0, G>() : nml_fn<double, 2, 1, G>();
  if (obj == 4) {
    if (precision == 0) return metric == 0 ? nml_fn<double, 4, 0, G>() : nml_fn<double, 4, 1, G>();
    return metric == 0 ? nml_fn<float, 4, 0, G>() : nml_fn<float, 4, 1, G>();
  }
  if (precision == 0) {
    if (obj == 0) return metric == 0 ? nml_fn<double, 0, 0, G>() : nml_fn<double, 0, 1, G>();
    return metric == 0 ? nml_fn<double, 1, 0, G>() : nml_fn<double, 1, 1, G>();
  }
  if (obj == 0) return metric == 0 ? nml_fn<float, 0, 0, G>() : nml_fn<float, 0, 1, G>();
  return metric == 0 ? nml_fn<float, 1, 0, G>() : nml_fn<float, 1, 1, G>();
}

const void* nm_lane_kernel_ptr(int precision, int obj, int metric, bool rel_global) {
  return rel_global ? nml_ptr<true>(precision, obj, metric) : nml_ptr<false>(precision, obj, metric);
}

size_t nm_lane_smem(int precision, int obj, int32_t n_samples, bool rel_in_smem) {
  const bool f32 = precision != 0 && obj != 2 && obj != 3;
  size_t b = nml_fixed_bytes();
  if (obj == 0 || obj == 1 || obj == 4) b += f32 ? stash_bytes<float>(32) : stash_bytes<double>(32);
  if (rel_in_smem && obj != 3) b += (size_t)n_samples * 32 * (f32 ? sizeof(float) : sizeof(double));
  return b;
}

cudaError_t launch_nm_lane(const void* fn, const NmArgs& a, int grid, size_t smem, cudaStream_t st) {
  void* args[] = {const_cast<NmArgs*>(&a)};
  return cudaLaunchKernel(fn, dim3(grid), dim3(32), args, smem, st);
}

int nm_problems_per_block() { return NM_WARPS; }
int nm_threads() { return NM_THREADS; }

cudaError_t launch_nm(const void* fn, const NmArgs& a, int grid, size_t smem, cudaStream_t st) {
  void* args[] = {const_cast<NmArgs*>(&a)};
  return cudaLaunchKernel(fn, dim3(grid), dim3(NM_THREADS), args, smem, st);
}

}  // namespace opmm
