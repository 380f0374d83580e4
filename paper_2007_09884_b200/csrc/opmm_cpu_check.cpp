// opmm_cpu_check.cpp -- the paper's CPU_check column (Fig. 4, PAPER.md:352:
// "CPU_check is the optimization error computed by a serial implementation
// for validation purposes").  A serial fp64 re-score of the ONE OPC vector a
// fit returns, on the host, against the host copy of the recorded trace.
// It validates the GPU result; it is never used in place of the GPU path
// (opmm_create fails without a device, so no fit ever reaches here without
// one).  Independent of both the CUDA kernels and the test oracle: the RK4
// stages are written directly from the D1 plant equations.
#include <cmath>
#include <cstring>

#include "opmm_cpu_check.h"

namespace opmm {
namespace {

struct Plant {
  double kse[2], klt[2], b[2], nc[2];
  double bp, J;
  double inv_J, inv_b[2];   // the divisors, inverted once per call
};

// D1: T_m = K_SE_m (x_m - s_m theta); B_m x_m' = f_m - N_C_m s_m theta - K_LT_m x_m - T_m;
// f_m' = (n_m - f_m)/tau_m; J omega' = T_AG - T_ANT - B_P omega; theta' = omega.
// (s_AG = +1, s_ANT = -1; written out per muscle so the compiler keeps the
// state in registers)
inline void deriv(const Plant& P, const double y[6], const double n[2], const double inv_tau_s[2],
                  double dy[6]) {
  const double t0 = P.kse[0] * (y[2] - y[0]);
  const double t1 = P.kse[1] * (y[3] + y[0]);
  dy[0] = y[1];
  dy[1] = (t0 - t1 - P.bp * y[1]) * P.inv_J;
  dy[2] = (y[4] - P.nc[0] * y[0] - P.klt[0] * y[2] - t0) * P.inv_b[0];
  dy[3] = (y[5] + P.nc[1] * y[0] - P.klt[1] * y[3] - t1) * P.inv_b[1];
  dy[4] = (n[0] - y[4]) * inv_tau_s[0];
  dy[5] = (n[1] - y[5]) * inv_tau_s[1];
}

}  // namespace

double cpu_check_score(const double opc[OPMM_NPARAM], const double* rec, const opmm_control* ctl,
                       int metric) {
  Plant P;
  P.kse[0] = opc[OPMM_P_KSE_AG];  P.kse[1] = opc[OPMM_P_KSE_ANT];
  P.klt[0] = opc[OPMM_P_KLT_AG];  P.klt[1] = opc[OPMM_P_KLT_ANT];
  P.b[0] = opc[OPMM_P_B_AG];      P.b[1] = opc[OPMM_P_B_ANT];
  P.nc[0] = opc[OPMM_P_NC_AG];    P.nc[1] = opc[OPMM_P_NC_ANT];
  P.bp = opc[OPMM_P_B_P];         P.J = opc[OPMM_P_J];
  P.inv_J = 1.0 / P.J;
  P.inv_b[0] = 1.0 / P.b[0];
  P.inv_b[1] = 1.0 / P.b[1];
  const double F = opc[OPMM_P_NC_FIX];
  const double pw = std::isnan(opc[OPMM_P_PW]) ? ctl->pw_default_ms : opc[OPMM_P_PW];
  const int n = ctl->n_steps;
  const double A = std::isnan(ctl->amplitude_deg) ? rec[n] - rec[0] : ctl->amplitude_deg;
  const double s = A < 0.0 ? -1.0 : 1.0, Ap = std::fabs(A);
  // statics: g_m = K_SE/(K_LT+K_SE), G = sum g_m (N_C_m + K_LT_m)
  double g[2];
  for (int m = 0; m < 2; ++m) g[m] = P.kse[m] / (P.klt[m] + P.kse[m]);
  const double G = g[0] * (P.nc[0] + P.klt[0]) + g[1] * (P.nc[1] + P.klt[1]);
  const double th_star = (g[0] * F - g[1] * F) / G;
  double y[6];
  y[0] = th_star;
  y[1] = 0.0;
  y[2] = (F - (P.nc[0] - P.kse[0]) * th_star) / (P.klt[0] + P.kse[0]);
  y[3] = (F + (P.nc[1] - P.kse[1]) * th_star) / (P.klt[1] + P.kse[1]);
  y[4] = F;
  y[5] = F;
  double step_n[2] = {F + G * Ap / (g[0] + g[1]), F - G * Ap / (g[0] + g[1])};
  if (step_n[1] < 0.01) {
    step_n[1] = 0.01;
    step_n[0] = (G * (th_star + Ap) + 0.01 * g[1]) / g[0];
  }
  const double n_pulse = std::ceil(pw / ctl->dt_ms);
  const int nsub = ctl->substeps > 1 ? ctl->substeps : 1;   // reading Q25
  const double h = 1e-3 * ctl->dt_ms / (double)nsub;
  double acc = 0.0;
  for (int k = 0; k < n; ++k) {
    const bool pulse = (double)k < n_pulse;
    const double nn[2] = {pulse ? opc[OPMM_P_NSAC_AG] : step_n[0],
                          pulse ? opc[OPMM_P_NSAC_ANT] : step_n[1]};
    const double inv_tau[2] = {1.0 / (1e-3 * (pulse ? opc[OPMM_P_TAU_AC_AG] : opc[OPMM_P_TAU_DE_AG])),
                           1.0 / (1e-3 * (pulse ? opc[OPMM_P_TAU_AC_ANT] : opc[OPMM_P_TAU_DE_ANT]))};
    for (int sub = 0; sub < nsub; ++sub) {
      double k1[6], k2[6], k3[6], k4[6], t[6];
      deriv(P, y, nn, inv_tau, k1);
      for (int i = 0; i < 6; ++i) t[i] = y[i] + 0.5 * h * k1[i];
      deriv(P, t, nn, inv_tau, k2);
      for (int i = 0; i < 6; ++i) t[i] = y[i] + 0.5 * h * k2[i];
      deriv(P, t, nn, inv_tau, k3);
      for (int i = 0; i < 6; ++i) t[i] = y[i] + h * k3[i];
      deriv(P, t, nn, inv_tau, k4);
      for (int i = 0; i < 6; ++i) y[i] += h / 6.0 * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);
    }
    const double d = (y[0] - th_star) - s * (rec[k + 1] - rec[0]);
    acc += metric == 0 ? std::fabs(d) : d * d;
  }
  if (!(acc < 1e20)) return INFINITY;
  return metric == 0 ? acc : std::sqrt(acc / (double)(n + 1));
}

}  // namespace opmm
