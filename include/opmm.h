/*
 * opmm.h -- C ABI of libopmm, the B200 (sm_100a) hot path of the parallel
 * Oculomotor Plant Mathematical Model (OPMM), arXiv 2007.09884.
 *
 * The hot path: for every candidate OPC
 * vector c_i (Table 1) simulate the
 * 18-parameter linear homeomorphic plant (Fig. 1; equations
 * = SPEC D1) under the pulse-step control signal
 * with fixed-step classical RK4 (SPEC D2),
 * score it against the recorded saccade ("absolute difference between the
 * recorded and simulated eye movement trajectories"), and reduce
 * to the best-fit OPC ("exhaustive search of potential parameter values",
 * PAPER.md:202; "solutions are sorted for accuracy").
 *
 * Conventions (all entry points):
 *  - Every function returns an opmm_status and never aborts or exits.  On a
 *    non-OK status a message is available from opmm_last_error() (thread-local).
 *  - Units: angles in degrees, time arguments in ms, forces in g; internally
 *    mechanics run in seconds (reading Q2).
 *  - OPC vectors are 18 doubles in Table-1 order (OPMM_P_* below).  Batches of
 *    OPC vectors are SoA: element (p, i) at opc[p * ld + i], ld >= n.
 *  - Trajectories are time-major: sample k of candidate i at traj[k * ld + i]
 *    (coalesced across candidates).
 *  - Ownership: the caller owns every buffer passed in or out; the handle owns
 *    its workspace (block partials, staged trace, NCCL communicator) and frees
 *    it in opmm_destroy.  A handle is not thread-safe: calls on one handle are
 *    serialised on its stream.
 *  - "device" pointers must be CUDA device (or managed) memory on the handle's
 *    device; "host" pointers are ordinary host memory; "host or device"
 *    pointers are told apart with cudaPointerGetAttributes.
 *    The entry points opmm_generate / simulate / simulate_batch / score /
 *    simulate_score are asynchronous on `stream` (NULL = the handle's own
 *    stream, which is a non-blocking stream; pass cudaStreamLegacy, (void*)1,
 *    to order the work with the legacy default stream) when every buffer is
 *    device memory: they enqueue and return.  A host input is copied into a
 *    handle-owned device buffer on that stream; a host output is produced in
 *    one (its current contents copied in first, so entries the call does not
 *    write come back unchanged) and copied back, and the call then waits for
 *    its stream, so host results are complete on return.  Staging buffers
 *    are per handle: calls with host buffers on different streams of one
 *    handle must be ordered by the caller.  opmm_fit_async is device-only.
 *  - Per-candidate numerical failure is data, not an error:
 *      non-physical OPC  -> E = 1e10 * (1 + sum of violations)  (D8)
 *      non-finite or E >= 1e20 accumulated -> E = +inf          (reading Q10)
 *  - The product never computes on the CPU in place of the GPU: without a
 *    CUDA device opmm_create fails with OPMM_ERR_CUDA.  The only host
 *    arithmetic is argument validation, search-space preprocessing, and the
 *    paper's CPU_check column (a serial re-score of the single returned
 *    winner), which is validation, not a fallback.
 */
#ifndef OPMM_H
#define OPMM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OPMM_NPARAM 18
#define OPMM_MAX_STEPS 16384
#define OPMM_MAX_SUBSTEPS 4096
#define OPMM_NCCL_ID_BYTES 128

/* Table-1 order. */
enum {
  OPMM_P_KSE_AG = 0, OPMM_P_KSE_ANT, OPMM_P_KLT_AG, OPMM_P_KLT_ANT, OPMM_P_B_AG,
  OPMM_P_B_ANT, OPMM_P_B_P, OPMM_P_NC_AG, OPMM_P_NC_ANT, OPMM_P_J,
  OPMM_P_TAU_AC_AG, OPMM_P_TAU_AC_ANT, OPMM_P_TAU_DE_AG, OPMM_P_TAU_DE_ANT,
  OPMM_P_NC_FIX, OPMM_P_NSAC_AG, OPMM_P_NSAC_ANT, OPMM_P_PW
};

typedef enum {
  OPMM_OK = 0,
  OPMM_ERR_INVALID_ARG = 1,  /* argument failed validation; nothing launched   */
  OPMM_ERR_CUDA = 2,         /* CUDA runtime error or no usable device          */
  OPMM_ERR_NCCL = 3,         /* NCCL unavailable or a collective failed         */
  OPMM_ERR_OOM = 4,          /* device allocation failed                        */
  OPMM_ERR_NO_FINITE = 5,    /* fit: every candidate scored +inf (or N == 0)    */
  OPMM_ERR_UNSUPPORTED = 6   /* option combination not implemented              */
} opmm_status;

typedef enum { OPMM_FP64 = 0, OPMM_FP32 = 1 } opmm_precision;
/* PAPER.md:366 "absolute difference" -> L1 sum over all samples (default);
 * RMS = sqrt(mean d^2) is the option north_star names (reading Q9). */
typedef enum { OPMM_METRIC_L1 = 0, OPMM_METRIC_RMS = 1 } opmm_metric;
/* Both integrators compute the same classical RK4 map (SPEC D2).  PROPAGATOR
 * applies it as y+ = P(hA) y + hQ(hA) b, built per candidate (DESIGN.md
 * "Kernels"); RK4_STAGES evaluates the four stages literally. */
typedef enum { OPMM_INTEG_PROPAGATOR = 0, OPMM_INTEG_RK4_STAGES = 1 } opmm_integrator;

/* Pulse-step control + integration grid of one saccade. */
typedef struct {
  double dt_ms;          /* sample interval, > 0 (1.0 at 1 kHz)                  */
  int32_t n_steps;       /* 1..OPMM_MAX_STEPS; trajectories have n_steps+1 samples */
  int32_t substeps;      /* RK4 steps per sample interval: 0 or 1 -> h = dt;
                            s in 2..OPMM_MAX_SUBSTEPS -> s steps of dt/s with the
                            control held over the interval (Q25).  The
                            propagator integrator composes them into one
                            sample-to-sample map: the per-sample loop cost does
                            not grow with s, only the per-candidate setup. */
  double amplitude_deg;  /* signed target amplitude A; NaN => rec[n]-rec[0] (D5) */
  double theta0_deg;     /* absolute start position (opmm_simulate output only)  */
  double pw_default_ms;  /* PW used when a candidate's PW is NaN: "saccade
                            duration - 6 ms"                      */
} opmm_control;

/* Candidate generator (PAPER.md:202 exhaustive search; reading Q14/Q15).
 * mode 0 (random): candidate i uses Philox4x32-10 with key = (seed_lo, seed_hi)
 *   and counter = (i_lo, i_hi, saccade, j), j = 0..4 -> 20 words; dimension d
 *   uses word d: u = (w + 0.5) 2^-32; log dims lo*exp(u*log(hi/lo)); linear
 *   dims lo + u*(hi-lo); lo == hi fixes the dimension.
 * mode 1 (grid): mixed-radix digits of i (dimension 0 fastest) over levels[d];
 *   log dims lo*exp(digit*(log(hi/lo)/(L-1))); linear lo + digit*((hi-lo)/(L-1)).
 *   The product of levels must equal the candidate count of the call. */
typedef struct {
  int32_t mode;
  int32_t model;   /* 0 = 18-parameter OPMM (Table 1); 1 = 9-parameter OPMM (Table 2,
                      PAPER.md:173-197): free slots K_SE_AG (= K_SE), K_LT_AG (= K_LT),
                      B_AG, B_ANT, B_P, N_C_AG, N_C_ANT, J, N_C_FIX; every generated
                      candidate is expanded per SPEC D7 (K_SE_ANT = K_SE_AG,
                      K_LT_ANT = K_LT_AG, pulse 55 / 0.5 g of width pw_default,
                      Table 1 time constants -- DESIGN.md reading Q23) */
  uint64_t seed;
  double lo[OPMM_NPARAM];
  double hi[OPMM_NPARAM];
  uint8_t log_scale[OPMM_NPARAM];  /* 1: log-uniform / geometric; requires lo > 0 */
  uint8_t pad2_[6];
  int32_t levels[OPMM_NPARAM];     /* grid mode only, each >= 1                   */
} opmm_search_space;

typedef struct {
  int32_t precision;    /* opmm_precision: arithmetic of the integrate+score loop */
  int32_t metric;       /* opmm_metric                                            */
  int32_t integrator;   /* opmm_integrator                                        */
  int32_t block_size;   /* 0 = default (384); else 64..384, multiple of 32        */
  int32_t grid_blocks;  /* 0 = default (persistent: SMs x resident blocks)        */
  int32_t cpu_check;    /* 1 = fill result.cpu_check, 0 = NaN      */
  int32_t kernel_variant; /* fit kernel: 0 = auto; 1 = one candidate per thread;
                              2 = two interleaved candidates per thread;
                              3 = warp-specialised producer/consumer.  2 and 3
                              need PROPAGATOR, a physical-by-construction space
                              and block_size = 0.
                              4 = superposition over the grid levels of a pulse
                              height (N_SAC_AG or N_SAC_ANT, the one with more
                              levels): the trajectory is affine in it (RK4 of
                              the linear plant), so each grid node is integrated
                              twice and every level scored at 2 fp64 ops per
                              sample (FP32: fp64 integration, fp32 level loop).
                              Needs grid mode, the 18-parameter model,
                              PROPAGATOR, no substeps, a physical space,
                              no certify, no top_k, block_size = 0; else
                              UNSUPPORTED.  Auto (0) picks it for such grids
                              with >= 8 levels.  Errors equal variant 1's up to
                              rounding (<= 1e-11 relative measured, DESIGN.md
                              section 7b), so where two candidates' errors tie
                              to within that rounding the returned index may
                              differ from variant 1's; exact ties still go to
                              the lowest index.
                              5 = lane refill: a lane whose error
                              has passed CAP (reading Q10: +inf) stops; once 16
                              lanes of a warp are free they take new candidates.
                              Same needs as 2/3, no certify / top_k.  Errors bit-identical to 1;
                              measured slower.          */
  int32_t certify;      /* FP32 only ("solutions are sorted for accuracy",
                           PAPER.md:251): keep the exact top-K by fp32 error
                           (K = top_k, or 8 when top_k = 0), re-score those K in
                           fp64 and return the fp64-best; result.certified says
                           whether the list provably holds the fp64 winner
                           (DESIGN.md section 6).  Works on one GPU and across the
                           ranks of an NCCL handle (the ranks' lists are merged
                           before the re-score); kernel_variant 0/1 only.        */
  int32_t top_k;        /* 0 or 1..OPMM_MAX_TOPK: also return the K best (E, index)
                           pairs of the fit, exact and in lexicographic order
                           (reading Q12), over all candidates and ranks.
                           kernel_variant 0/1 (auto never superposes then).     */
  uint32_t flags;       /* OPMM_FIT_FLAG_* (measurement / test switches)          */
  double* err_out;      /* optional DEVICE [n]: E_i of every candidate (validation);
                           a host pointer is refused (OPMM_ERR_INVALID_ARG)      */
} opmm_fit_options;

#define OPMM_MAX_TOPK 32
/* opmm_fit_options.flags.  None changes any result; they select between
 * equivalent code paths for measurement and for the tests that prove the
 * equivalence. */
#define OPMM_FIT_FLAG_NO_LANE_SORT   1u  /* fit_kernel: no pulse-end sort pre-pass    */
#define OPMM_FIT_FLAG_SUPER_SMEM     2u  /* superposition: shared-memory columns only */
#define OPMM_FIT_FLAG_NO_GRAPH       4u  /* opmm_fit: plain launches, no CUDA graph   */
#define OPMM_FIT_FLAG_NO_GRID_TABLES 8u  /* grid fits: the generic grid generator, not
                                            the shared-memory level tables           */

typedef struct {
  int64_t best_index;            /* global candidate index; -1 if no finite E     */
  double opt_err;                /* E of the winner as computed by the kernel
                                    (certify: its fp64 re-score)                  */
  double cpu_check;              /* serial host fp64 re-score (Fig. 4 CPU_check)   */
  double opc[OPMM_NPARAM];       /* winner's OPC, exactly as evaluated on device   */
  int64_t n_finite;              /* candidates with finite E (all ranks)           */
  int64_t n_evaluated;           /* candidates evaluated (all ranks)               */
  int32_t top_k;                 /* entries used below (top_k, or the certify K)   */
  int32_t certified;             /* certify: 1 if (a) every candidate whose fp32
                                    error is <= T* = E32[0] + 2 delta is in the
                                    list (delta = 1e-4 max(E32[0], s), s = sum|rel|
                                    or RMS(rel)) and (b) every listed candidate's
                                    fp32 and fp64 errors agree within delta.  Then
                                    the fp64 winner is in the list -- and returned
                                    -- unless its own fp32 error misses the budget
                                    (possible only for RK4-unstable candidates,
                                    whose rounding grows with the step; DESIGN.md
                                    section 6 bounds it for stable ones)           */
  int64_t topk_index[OPMM_MAX_TOPK]; /* kept indices in (E, index) order (certify:
                                    fp32 E); -1 = unused                           */
  double topk_err[OPMM_MAX_TOPK];    /* their errors (certify: fp64 re-scores)     */
} opmm_fit_result;

typedef struct opmm_handle opmm_handle;

/* ---- library / handle --------------------------------------------------- */
const char* opmm_version(void);
const char* opmm_last_error(void);

/* Create a handle on CUDA device `device` (single GPU, world = 1). */
opmm_status opmm_create(opmm_handle** h, int device);
/* Multi-GPU: one process per GPU.  `nccl_id` is OPMM_NCCL_ID_BYTES produced by
 * opmm_nccl_unique_id on rank 0 and broadcast by the caller (e.g. through
 * torch.distributed).  Candidates are sharded disjointly per rank and the
 * per-rank results are merged with one ncclAllGather per fit: 32 bytes per
 * rank (E, index, n_finite, n_evaluated), 544 with top_k / certify (the
 * rank's top-32 list).  world = 1 still creates a
 * one-rank communicator, so the gather + merge path also runs on one GPU.
 * NCCL is loaded at run time (libnccl.so.2). */
opmm_status opmm_nccl_unique_id(uint8_t* nccl_id /* host, 128 B */);
opmm_status opmm_create_nccl(opmm_handle** h, int device, const uint8_t* nccl_id,
                             int rank, int world);
opmm_status opmm_destroy(opmm_handle* h);
/* The handle's own stream (cudaStream_t), for callers that want to order work. */
opmm_status opmm_get_stream(opmm_handle* h, void** stream);
/* Kernel timing, off by default: when on, every launch through the handle is
 * bracketed by a pair of CUDA events on its stream (~6 us of stream time per
 * call on a B200), and opmm_last_kernel_ms reads them. */
opmm_status opmm_set_kernel_timing(opmm_handle* h, int32_t on);
/* Device time (ms, CUDA events on the launching stream) of the most recent
 * launch through this handle while timing was on: the kernels of one fit /
 * simulate / score / estimate call (a synchronous opmm_fit: its H2D copy and
 * kernel).  Synchronises with that launch.  INVALID_ARG when timing is off or
 * nothing has been launched since it was turned on. */
opmm_status opmm_last_kernel_ms(opmm_handle* h, float* ms);

/* ---- host-only helpers (no GPU needed) ----------------------------------- */
/* Rank r of R owns global candidate indices [floor(rN/R), floor((r+1)N/R)). */
opmm_status opmm_shard_range(int64_t n, int rank, int world, int64_t* begin, int64_t* end);
/* Lexicographic (E, index) minimum of `count` partial results (err[i], idx[i]);
 * idx -1 entries are ignored; +inf never beats a finite E (reading Q12). */
opmm_status opmm_merge_argmin(const double* err, const int64_t* idx, int count,
                              double* best_err, int64_t* best_idx);
/* Merge `lists` sorted (E, index) lists of K entries each (list l at
 * err/idx + l * K; index -1 marks unused entries) into the K lexicographically
 * smallest pairs out_err/out_idx [K] (-1 / +inf where fewer exist).  The same
 * function the merge kernel applies to the ranks' top-K lists (reading Q12). */
opmm_status opmm_merge_topk(const double* err, const int64_t* idx, int lists, int K,
                            double* out_err, int64_t* out_idx);
/* The fp32 certificate (opmm_fit_result.certified) of one
 * merged list: e32 [K] its fp32 errors (sorted), e64 [K] their fp64
 * re-scores, idx [K] (-1 unused), scale s = sum |rel| (L1) or RMS(rel) (RMS).
 * Returns certified and the fp64-best entry (lowest index on ties). */
opmm_status opmm_certify_topk(const double* e32, const double* e64, const int64_t* idx, int K,
                              double scale, int32_t* certified, int64_t* best_index,
                              double* best_err);
/* Validate a control / search space (the same checks every entry point runs). */
opmm_status opmm_validate(const opmm_control* ctl, const opmm_search_space* space,
                          int64_t n_candidates);

/* ---- hot path ------------------------------------------------------------- */
/* Candidates [begin, begin+count) of `space` for saccade `saccade`, written
 * SoA to host-or-device opc_out[18][ld].  Bit-identical to what the fit
 * kernel evaluates for the same indices. */
opmm_status opmm_generate(opmm_handle* h, const opmm_search_space* space, uint32_t saccade,
                          int64_t begin, int64_t count, double* opc_out, int64_t ld,
                          void* stream);

/* Simulate n explicit OPC vectors (host-or-device SoA opc[18][ld]) under
 * `ctl`: host-or-device traj[(n_steps+1) x ld_out] of `precision` (double or
 * float) receives absolute positions theta0 + s * Delta-theta_k (s = sign(A),
 * D6 mirroring); optional host-or-device status[n]: 0 ok, 1 non-physical
 * (trajectory NaN), 2 diverged (non-finite sample).  SPEC simulate
 * (SPEC.md:108-116); the model is opmm_simulate(opc_batch, control, dt,
 * n_steps) -> trajectories of BASELINE.json's north_star. */
opmm_status opmm_simulate(opmm_handle* h, const double* opc, int64_t n, int64_t ld,
                          const opmm_control* ctl, int32_t precision, int32_t integrator,
                          void* traj, int64_t ld_out, uint8_t* status, void* stream);

/* opmm_simulate with one control per candidate (host-or-device opc, traj,
 * status as opmm_simulate): candidate i (column i) is
 * simulated under HOST ctl[i] -- its own amplitude_deg, theta0_deg and
 * pw_default_ms; dt_ms and n_steps must be equal for all i (INVALID_ARG
 * otherwise).  Identical outputs to n single-candidate opmm_simulate calls;
 * used to synthesize a population of saccades in one launch.  The controls
 * are staged in a handle-owned device buffer (calls on different streams
 * must be ordered by the caller). */
opmm_status opmm_simulate_batch(opmm_handle* h, const double* opc, int64_t n, int64_t ld,
                                const opmm_control* ctl, int32_t precision, int32_t integrator,
                                void* traj, int64_t ld_out, uint8_t* status, void* stream);

/* Score n stored trajectories (host-or-device traj[n_samples x ld] of
 * `precision`) against host-or-device recorded[n_samples] (fp64):  E_i =
 * sum_k |traj_k,i - rec_k| (L1, "absolute difference") or
 * sqrt(mean d^2) (RMS); accumulated >= 1e20 or non-finite -> +inf.
 * host-or-device err[n] (fp64).  The only HBM-bound entry point. */
opmm_status opmm_score(opmm_handle* h, const void* traj, int64_t n, int64_t ld,
                       int32_t n_samples, const double* recorded, int32_t precision,
                       int32_t metric, double* err, void* stream);

/* Fused simulate + score of n explicit OPC vectors (host-or-device opc)
 * against host-or-device recorded[n_steps+1] (a host trace must be finite:
 * INVALID_ARG otherwise); no trajectory reaches HBM.  E_i as in opmm_fit
 * (penalty for non-physical).  host-or-device err[n] (fp64). */
opmm_status opmm_simulate_score(opmm_handle* h, const double* opc, int64_t n, int64_t ld,
                                const opmm_control* ctl, const double* recorded,
                                int32_t precision, int32_t metric, int32_t integrator,
                                double* err, void* stream);

/* Exhaustive fit of one saccade over candidates [0, n_candidates) of `space`:
 * generate -> simulate -> score -> argmin, in one kernel (plus, for world > 1,
 * one ncclAllGather and a merge kernel).  `recorded` is HOST or DEVICE
 * (n_steps+1 fp64 samples, auto-detected); `out` is HOST.  Synchronous.
 * Returns OPMM_ERR_NO_FINITE (best_index = -1) if no candidate is finite. */
opmm_status opmm_fit(opmm_handle* h, const double* recorded, const opmm_control* ctl,
                     const opmm_search_space* space, int64_t n_candidates,
                     const opmm_fit_options* opts, opmm_fit_result* out);

/* Asynchronous fit for device-resident inputs: DEVICE recorded, DEVICE
 * out_dev (one opmm_fit_result; cpu_check is NaN).  Enqueues on the handle's
 * stream; nothing is copied to or from the host. */
opmm_status opmm_fit_async(opmm_handle* h, const double* recorded_dev, const opmm_control* ctl,
                           const opmm_search_space* space, int64_t n_candidates,
                           const opmm_fit_options* opts, opmm_fit_result* out_dev);

/* One rank's share of a fit, on a PLAIN handle, for callers that launch the
 * ranks themselves (their own launcher or communicator) and merge on the
 * host: the same evaluation as opmm_fit for rank `rank` of `world` (SURVEY
 * 8(e)) -- candidates [floor(rN/R), floor((r+1)N/R)), or, when the
 * superposition kernel is chosen, that range of grid nodes with all their
 * levels -- with out (HOST) describing the shard: its lexicographic best
 * (global index), n_finite, n_evaluated, its exact top-K when asked, CPU_check
 * of its winner.  The shards partition the candidates, so the fit's winner is
 * opmm_merge_argmin over the shards' (opt_err, best_index), its n_finite the
 * sum, its top-K opmm_merge_topk over their lists; with FP32 certify each
 * shard re-scores its own list in fp64, and the merged winner is certified
 * when every shard is (each certified shard returns its fp64-best).  An
 * NCCL handle is refused (it shards by itself). */
opmm_status opmm_fit_shard(opmm_handle* h, const double* recorded, const opmm_control* ctl,
                           const opmm_search_space* space, int64_t n_candidates, int rank,
                           int world, const opmm_fit_options* opts, opmm_fit_result* out);

/* Population batch: S independent saccades, each
 * fitted over candidates [0, n_per) of `space` with Philox counter word 2 =
 * saccade index.  recorded: HOST or DEVICE [S][n_steps+1] (same n_steps and
 * dt for all, from ctl[0]); ctl: HOST [S] (per-saccade amplitude /
 * pw_default); out: HOST [S].  On an NCCL handle rank r fits only saccades
 * [floor(rS/R), floor((r+1)S/R)) and fills only those entries of out: the
 * saccades are independent problems, so there is no collective.
 * opts->err_out (optional): DEVICE [S][n_per], row s = saccade s's errors
 * (on an NCCL handle only this rank's rows are written). */
opmm_status opmm_fit_batch(opmm_handle* h, const double* recorded, int64_t S,
                           const opmm_control* ctl, const opmm_search_space* space,
                           int64_t n_per, const opmm_fit_options* opts, opmm_fit_result* out);

/* ---- Nelder-Mead estimator ------------------------------ */
/* The paper's own estimator (Alg. 1): a
 * parallel Nelder-Mead after Lagarias -- all simplex
 * transformations evaluated simultaneously, the simplex sorted
 * every iteration, exit when BOTH the max coordinate distance
 * to the best vertex <= tol_x AND the max |f_i - f_best| <= tol_f
 * (PAPER.md:252-255), or after max_iter iterations, or at the time boundary
 * (opmm_nm_options.time_budget_ms).  Coefficients rho = 1,
 * chi = 2, gamma = 0.5, sigma = 0.5 (SPEC D10); initial simplex: each
 * coordinate scaled by (1 + init_scale), zero coordinates set to
 * init_scale * 0.00025 (SPEC D9); stable sort (SPEC D14).  Scheduled one
 * warp per problem or one lane per problem (opmm_nm_schedule); either way the
 * iterates are the serial algorithm's. */
typedef enum {
  OPMM_NM_OBJ_PROPAGATOR = 0,   /* plant error, fit-path propagator (fast)          */
  OPMM_NM_OBJ_RK4_STAGES = 1,   /* plant error, literal four-stage RK4              */
  OPMM_NM_OBJ_REFERENCE = 2     /* plant error in the RK4 definition's operation
                                   order, explicitly rounded fp64 (reproducible)    */
} opmm_nm_objective;

/* How problems map onto the GPU.  Both give the serial algorithm's iterates
 * (same decisions, same explicitly rounded simplex arithmetic, same order);
 * they differ in which points are evaluated and in the gpu_evals count.
 *   LOCKSTEP: the paper's schedule -- one warp per problem
 *     evaluates every transformation point of an iteration at once (n + 4
 *     points, one per lane): the lowest latency per problem.
 *   LANE: one problem per lane, only the points the decision needs (~1.7 per
 *     iteration): the fewest evaluations.
 *   GROUP: 4 lanes per problem evaluate the reflection, expansion and both
 *     contractions at once (shrink and initial points 4 at a time): one
 *     evaluation of latency per iteration at 8 problems per warp.
 *     With more problems than one wave of resident blocks, the grid is one
 *     wave and a group whose problem has finished takes the next one (refill),
 *     so slots are not held idle until the slowest problem of their block ends.
 *   AUTO: GROUP from 1024 problems (per rank) on, LOCKSTEP below (measured on
 *     one B200: GROUP is the fastest from ~1000 problems on, LOCKSTEP below;
 *     LANE does the least work but has the longest latency per iteration). */
typedef enum {
  OPMM_NM_SCHEDULE_AUTO = 0,
  OPMM_NM_SCHEDULE_LOCKSTEP = 1,
  OPMM_NM_SCHEDULE_LANE = 2,
  OPMM_NM_SCHEDULE_GROUP = 3
} opmm_nm_schedule;

typedef struct {
  int32_t precision;     /* OPMM_FP64 / OPMM_FP32 (REFERENCE is always fp64)       */
  int32_t objective;     /* opmm_nm_objective                                      */
  int32_t metric;        /* opmm_metric                                            */
  int32_t max_iter;      /* 0 = 200 * dim (SPEC D13)                                */
  double tol_x;          /* 0 = 1e-4 (SPEC D13)                                     */
  double tol_f;          /* 0 = 1e-4                                                */
  double init_scale;     /* 0 = 0.05 (SPEC D9)                                      */
  int32_t cpu_check;     /* 1 = fill cpu_check (plant objectives)                  */
  int32_t schedule;      /* opmm_nm_schedule (0 = auto)                             */
  double time_budget_ms; /* the paper's time boundary (SPEC D13
                            time_budget): a problem stops once its own wall
                            clock, from its start on the GPU (%globaltimer),
                            exceeds this; exit_reason 2.  0 = none.  Checked
                            once per iteration, after the tolerance test, so a
                            converged problem still reports 0; max_iter is the
                            deterministic equivalent                        */
} opmm_nm_options;

typedef struct {
  double x[OPMM_NPARAM]; /* best vertex (first dim entries used)                   */
  double f_best;         /* objective at x                                          */
  double cpu_check;      /* serial host fp64 re-score of x (plant objectives)      */
  int32_t iterations;    /* iterations, counted as the serial algorithm counts them */
  int32_t func_evals;    /* objective evaluations the serial algorithm needs        */
  int32_t gpu_evals;     /* evaluations performed (LOCKSTEP: n + 4 per iteration;
                            LANE: the serial algorithm's own, = func_evals;
                            GROUP: 4 per iteration, n per shrink)                 */
  int32_t exit_reason;   /* 0 = tolerances met, 1 = max_iter, 2 = time budget      */
} opmm_nm_result;

/* Estimate the 18-parameter OPC of S saccades independently (SPEC
 * estimate_batch).  recorded: HOST or DEVICE [S][n_steps+1];
 * ctl: HOST [S] (shared dt/n_steps); x0: HOST [18] start vector or NULL for
 * the Table 1 defaults; a NaN PW starts at the saccade's
 * pw_default_ms.  out: HOST [S].  On an NCCL handle rank r estimates only
 * saccades [floor(rS/R), floor((r+1)S/R)) (independent problems, no
 * collective) and fills only those entries.  Synchronous.  Each problem keeps
 * its trace in shared memory, or, for traces too long for it (beyond ~5000
 * samples in fp64), in a handle-owned global workspace; n_steps up to
 * OPMM_MAX_STEPS. */
opmm_status opmm_estimate_batch(opmm_handle* h, const double* recorded, int64_t S,
                                const opmm_control* ctl, const double* x0,
                                const opmm_nm_options* opts, opmm_nm_result* out);

/* The same Nelder-Mead engine on the SPEC acceptance-3 test functions
 * (fn_id 0 sphere, 1 Rosenbrock, 2 Powell quartic; dim 1..18): S problems
 * with start points HOST x0[S][dim]; out HOST [S].  Synchronous. */
opmm_status opmm_nm_minimize_test(opmm_handle* h, int32_t fn_id, int32_t dim, const double* x0,
                                  int64_t S, const opmm_nm_options* opts, opmm_nm_result* out);

#ifdef __cplusplus
}
#endif
#endif /* OPMM_H */
