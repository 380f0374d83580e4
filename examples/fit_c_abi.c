/* examples/fit_c_abi.c -- libopmm from plain C (no Python, no torch).
 *
 * Fits a synthetic 10-degree saccade (a hand-written pulse-step-like ramp,
 * host memory) over 10^5 random OPC candidates of the paper's bounds
 * (log-uniform [0.1x, 10x] of Table 1; PW in [1, 100] ms),
 * prints the winner and its exact top-5, then runs the asynchronous entry
 * points on HOST buffers (generate -> simulate -> score, and the fused
 * simulate_score; the library stages them on the device and waits), checks
 * that the two scores agree, and exercises the error path.  Build:
 *   gcc -O2 -I include examples/fit_c_abi.c -L paper_2007_09884_b200 -lopmm \
 *       -Wl,-rpath,'$ORIGIN/../paper_2007_09884_b200' -o build/fit_c_abi -lm
 */
#include <math.h>
#include <stdio.h>
#include <string.h>

#include "opmm.h"

int main(void) {
  static const double table1[OPMM_NPARAM] = {2.5, 2.5, 1.2, 1.2, 0.046, 0.022, 0.06, 0.8, 0.5,
                                             0.000043, 11.7, 2.4, 2.0, 1.9, 14.0, 55.0, 0.5, 40.0};
  opmm_handle* h = NULL;
  opmm_status st = opmm_create(&h, 0);
  if (st != OPMM_OK) {
    fprintf(stderr, "opmm_create: %d %s\n", (int)st, opmm_last_error());
    return 2;
  }
  opmm_control ctl;
  memset(&ctl, 0, sizeof(ctl));
  ctl.dt_ms = 1.0;
  ctl.n_steps = 100;
  ctl.amplitude_deg = 10.0;
  ctl.theta0_deg = 0.0;
  ctl.pw_default_ms = 40.0;
  double rec[101];
  for (int k = 0; k <= 100; ++k) rec[k] = 10.0 * (1.0 - exp(-k / 15.0));   /* saccade-like */
  opmm_search_space sp;
  memset(&sp, 0, sizeof(sp));
  sp.mode = 0;
  sp.seed = 9884;
  for (int d = 0; d < OPMM_NPARAM; ++d) {
    sp.lo[d] = 0.1 * table1[d];
    sp.hi[d] = 10.0 * table1[d];
    sp.log_scale[d] = 1;
    sp.levels[d] = 1;
  }
  sp.lo[OPMM_P_PW] = 1.0;
  sp.hi[OPMM_P_PW] = 100.0;
  sp.log_scale[OPMM_P_PW] = 0;
  opmm_fit_options opts;
  memset(&opts, 0, sizeof(opts));
  opts.cpu_check = 1;
  opmm_fit_result r;
  st = opmm_fit(h, rec, &ctl, &sp, 100000, &opts, &r);
  if (st != OPMM_OK) {
    fprintf(stderr, "opmm_fit: %d %s\n", (int)st, opmm_last_error());
    return 3;
  }
  printf("best_index %lld opt_err %.9f cpu_check %.9f n_finite %lld/%lld\n",
         (long long)r.best_index, r.opt_err, r.cpu_check, (long long)r.n_finite,
         (long long)r.n_evaluated);
  printf("K_SE_AG %.6f J %.8f PW %.4f\n", r.opc[OPMM_P_KSE_AG], r.opc[OPMM_P_J], r.opc[OPMM_P_PW]);
  if (!(fabs(r.cpu_check - r.opt_err) <= 1e-9 * r.opt_err)) return 4;
  /* the exact top-5 (E, index) pairs of the same fit */
  opts.top_k = 5;
  opmm_fit_result r5;
  st = opmm_fit(h, rec, &ctl, &sp, 100000, &opts, &r5);
  if (st != OPMM_OK || r5.top_k != 5 || r5.topk_index[0] != r.best_index) return 6;
  for (int k = 1; k < 5; ++k)
    if (!(r5.topk_err[k - 1] < r5.topk_err[k] ||
          (r5.topk_err[k - 1] == r5.topk_err[k] && r5.topk_index[k - 1] < r5.topk_index[k])))
      return 7;
  printf("top-5:");
  for (int k = 0; k < 5; ++k) printf(" %lld (%.6f)", (long long)r5.topk_index[k], r5.topk_err[k]);
  printf("\n");
  /* the same fit as three ranks' shares (opmm_fit_shard), merged on the host */
  {
    enum { R = 3 };
    opmm_fit_result part[R];
    double pe[R], le[R * 5];
    int64_t pi[R], li[R * 5];
    for (int k = 0; k < R; ++k) {
      if ((st = opmm_fit_shard(h, rec, &ctl, &sp, 100000, k, R, &opts, &part[k])) != OPMM_OK) return 14;
      pe[k] = part[k].opt_err;
      pi[k] = part[k].best_index;
      for (int j = 0; j < 5; ++j) {
        le[k * 5 + j] = part[k].topk_err[j];
        li[k * 5 + j] = part[k].topk_index[j];
      }
    }
    double be, me[5];
    int64_t bi, mi[5];
    if (opmm_merge_argmin(pe, pi, R, &be, &bi) != OPMM_OK || bi != r.best_index || be != r.opt_err) return 15;
    if (opmm_merge_topk(le, li, R, 5, me, mi) != OPMM_OK) return 16;
    for (int j = 0; j < 5; ++j)
      if (mi[j] != r5.topk_index[j] || me[j] != r5.topk_err[j]) return 17;
    printf("3 shards merged on the host: best %lld, top-5 identical\n", (long long)bi);
  }
  /* host buffers through the asynchronous entry points */
  enum { NC = 64 };
  static double opc[OPMM_NPARAM * NC], traj[101 * NC], e_score[NC], e_fused[NC];
  static uint8_t status[NC];
  if ((st = opmm_generate(h, &sp, 0, 0, NC, opc, NC, NULL)) != OPMM_OK) return 8;
  if ((st = opmm_simulate(h, opc, NC, NC, &ctl, OPMM_FP64, OPMM_INTEG_PROPAGATOR, traj, NC, status,
                          NULL)) != OPMM_OK) return 9;
  if ((st = opmm_score(h, traj, NC, NC, 101, rec, OPMM_FP64, OPMM_METRIC_L1, e_score, NULL)) != OPMM_OK)
    return 10;
  if ((st = opmm_simulate_score(h, opc, NC, NC, &ctl, rec, OPMM_FP64, OPMM_METRIC_L1,
                                OPMM_INTEG_PROPAGATOR, e_fused, NULL)) != OPMM_OK) return 11;
  int n_ok = 0;
  for (int i = 0; i < NC; ++i) {
    if (isinf(e_fused[i]) != isinf(e_score[i]) || (status[i] == 2) != (isinf(e_fused[i]) != 0)) return 12;
    if (!isinf(e_fused[i]) && !(fabs(e_fused[i] - e_score[i]) <= 1e-12 * e_fused[i])) return 13;
    n_ok += status[i] == 0;
  }
  printf("host buffers: %d candidates simulated + scored, %d finite, scores agree\n", NC, n_ok);
  /* the paper's own estimator: batched Nelder-Mead on 4 copies of the trace
   * (Table 1 defaults as the start, 60 iterations at most) */
  {
    enum { S = 4 };
    static double recs[S * 101];
    opmm_control ctls[S];
    opmm_nm_result nm[S];
    for (int k = 0; k < S; ++k) {
      memcpy(recs + k * 101, rec, sizeof(double) * 101);
      ctls[k] = ctl;
    }
    opmm_nm_options no;
    memset(&no, 0, sizeof(no));
    no.max_iter = 60;
    no.cpu_check = 1;
    if ((st = opmm_estimate_batch(h, recs, S, ctls, NULL, &no, nm)) != OPMM_OK) return 18;
    for (int k = 1; k < S; ++k)
      if (nm[k].f_best != nm[0].f_best || nm[k].iterations != nm[0].iterations) return 19;
    if (!(fabs(nm[0].cpu_check - nm[0].f_best) <= 1e-9 * nm[0].f_best)) return 20;
    printf("Nelder-Mead: f %.6f after %d iterations (exit %d), CPU_check agrees\n", nm[0].f_best,
           nm[0].iterations, nm[0].exit_reason);
  }
  /* invalid argument: error status + message, nothing launched */
  ctl.dt_ms = -1.0;
  st = opmm_fit(h, rec, &ctl, &sp, 10, &opts, &r);
  printf("invalid dt -> status %d (%s)\n", (int)st, opmm_last_error());
  if (st != OPMM_ERR_INVALID_ARG) return 5;
  opmm_destroy(h);
  printf("fit_c_abi ok\n");
  return 0;
}
