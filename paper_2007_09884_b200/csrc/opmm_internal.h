// opmm_internal.h -- launch-argument structs shared by opmm_api.cu (host) and
// opmm_kernels.cu (device).  Not part of the public ABI.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "opmm.h"
#include "opmm_device.cuh"

namespace opmm {

// Dynamic shared memory of the simulate kernels: the relativized trace
// (rel_bytes) followed by the per-thread phase-coefficient stash [16][block].
template <typename T>
__host__ __device__ constexpr size_t rel_bytes(int32_t n_samples) {
  return ((size_t)n_samples * sizeof(T) + 15) & ~(size_t)15;
}
template <typename T>
__host__ __device__ constexpr size_t stash_bytes(int block, int cand_per_thread = 1) {
  return (size_t)20 * cand_per_thread * block * sizeof(T);   // [C][10][block] vec2<T>
}
// fit kernel: trace, then the exp table (double2[EXP_TAB_N]), then the stash
__host__ __device__ constexpr size_t exp_tab_bytes() { return (size_t)EXP_TAB_N * 16; }

// Per-block / per-rank (E, index) partial: 32 bytes.
struct Partial {
  double e;
  int64_t i;
  int64_t nf;     // finite candidates
  int64_t neval;  // evaluated candidates (rank partials only)
};

// fit_kernel launch bounds: 384 threads x 168 registers, one block per SM
// (3 warps per scheduler); the default block size of the fit entry points
#ifndef OPMM_FIT_LB_THREADS
#define OPMM_FIT_LB_THREADS 384
#endif
#ifndef OPMM_FIT_LB_BLOCKS
#define OPMM_FIT_LB_BLOCKS 1
#endif

// fit_kernel super-tile: a block sorts up to SUPER_MAX candidates at once
// (per candidate in shared memory: permutation uint16 for the whole pass,
// key/rank uint32 during the pre-pass only -- aliased onto the coefficient
// stash when that is large enough)
constexpr int SUPER_MAX = 8192;
__host__ __device__ constexpr size_t perm_bytes(int64_t s) { return (size_t)((s * 2 + 15) / 16 * 16); }
__host__ __device__ constexpr size_t tmp_bytes(int64_t s) { return (size_t)((s * 4 + 15) / 16 * 16); }

// Exact top-K lists (top_k / certify): one sorted list of TOPK (E, index)
// pairs per warp, lane l = rank l (K <= TOPK used).
constexpr int TOPK = OPMM_MAX_TOPK;
// certify scratch of the finishing block: the fp64 trace and a [10][32]
// double2 stash for the one-warp fp64 re-score
__host__ __device__ constexpr size_t cert_scratch_bytes(int32_t n_samples) {
  return (((size_t)n_samples + 1) & ~(size_t)1) * 8 + (size_t)20 * 32 * 8;
}
// Per-rank result (world > 1): the rank's (E, index, n_finite, n_evaluated)
// and, with top_k / certify, its top-32 list.  The all-gather moves the first
// 32 bytes, or all 544 with a list.
struct RankPartial {
  Partial p;
  double e[TOPK];
  int64_t i[TOPK];
};

struct FitArgs {
  const double* rec;        // device [S][n_steps+1]
  const double2* exp_tab;   // device [EXP_TAB_N] (handle-owned)
  CtlDev ctl;
  SpaceDev space;
  double amplitude;         // single fit: signed A (NaN => rec[n]-rec[0])
  double pw_default;
  const double* sac_ctl;    // batch: device [S][2] = (amplitude, pw_default); else nullptr
  int64_t sac_begin;        // first saccade of this launch (blockIdx.y offset)
  int64_t begin, end;       // candidate range of this rank
  double* err_out;          // optional device, candidate i at [sac * err_ld + i - err_base]
  int64_t err_ld;
  int64_t err_base;
  int32_t sort_lanes;       // counting-sort tiles by pulse end (see fit_kernel)
  int32_t certify;          // fp32: top-K by fp32 E + fp64 re-score (fit_kernel only)
  int32_t topk;             // K of the exact top-K (0 = none; certify sets it): topk_kernel
  int32_t metric_;          // opmm_metric (host side: the merge kernel's instantiation)
  int32_t fit_grid;         // topk_kernel: the fit kernel's gridDim.x (its Partials per saccade)
  int32_t pad1_;
  double* tk_e;             // topk_kernel: [S][gridDim.x * TOPK] key buffer
  int64_t* tk_i;
  unsigned int* tk_counters;   // topk_kernel: tickets [S] + fill counts at tk_fill_off, zero at rest
  int64_t tk_fill_off;
  int64_t super_tile;       // fit_kernel: candidates per block pass (multiple of 32, <= SUPER_MAX)
  int64_t perm_off;         // fit_kernel: byte offset of the super-tile permutation in smem
  int64_t tmp_off;          // fit_kernel: byte offset of the pre-pass key/rank scratch
  int64_t gt_off;           // fit_kernel<GT>: byte offset of the grid level tables in smem
  Partial* partials;        // [S][gridDim.x]
  unsigned int* counters;   // [S], zero between launches
  RankPartial* rank_out;    // optional [S]: per-rank result (world > 1)
  opmm_fit_result* final_out;  // optional: final result of saccade s at [s - out_base]
  int64_t out_base;
  // kernel_variant 4 (fit_super_kernel): superposition over the grid levels of
  // one pulse height; a "node" is a grid point with that dimension's digit 0
  int32_t sup_dim;          // NSAC_AG (15) or NSAC_ANT (16)
  int32_t sup_L;            // its grid levels
  int32_t sup_J;            // register chunk width (8, 12, ..., 32)
  int32_t sup_gt_n;         // entries of the per-dimension level tables
  int32_t sup_tab;          // 1: nodes from the tables; 0: generic generator (too many levels)
  int32_t sup_tm_warps;     // warps 0..T-1 keep their columns in tensor memory (0: none)
  int32_t sup_tm_cols;      // TMEM columns the block allocates (power of two, 32..512)
  int32_t pad2_;
  int64_t sup_st;           // its mixed-radix stride (product of the lower levels)
  int64_t node_begin, node_end;   // this rank's nodes
  unsigned long long* sup_next;   // [S]: next 32-node group to take (zero at rest)
};

struct ExplicitArgs {
  const double* opc;        // device SoA [18][ld]
  int64_t n, ld;
  CtlDev ctl;
  double amplitude, pw_default;
  const double* rec;        // simscore: device [n_steps+1]
  double* err;              // simscore: device [n]
  void* traj;               // simulate: device [(n_steps+1) x ld_out]
  int64_t ld_out;
  uint8_t* status;          // simulate: optional device [n]
  const double* cand_ctl;   // simulate_batch: device [n][3] = (amplitude, theta0, pw_default)
};

struct ScoreArgs {
  const void* traj;
  int64_t n, ld;
  int32_t n_samples;
  const double* rec;
  double* err;
};

// Batched Nelder-Mead (opmm_nm.cu)
struct NmOut {
  double f_best;
  int32_t iterations, func_evals, gpu_evals, exit_reason;
};

struct NmArgs {
  const double* rec;        // device [S][n_steps+1] (plant objectives)
  const double* sac_ctl;    // device [S][2] = (amplitude, pw_default)
  CtlDev ctl;
  const double* x0;         // device, problem p at x0 + p * x0_ld
  int64_t x0_ld;
  double* x_best;           // device [S][x_ld]
  int64_t x_ld;
  NmOut* out;               // device [S]
  int64_t prob_begin, prob_end;
  int32_t dim, fn_id, max_iter, pad_;
  double tol_x, tol_f, init_scale;
  unsigned long long time_budget_ns;   // per-problem wall-clock limit (0 = none)
  unsigned long long* nm_next;        // group schedule: next unassigned problem (refill; null = off)
  void* rel_global;         // long traces: device [S][n_steps+1] of the loop type; else null
};

const void* nm_kernel_ptr(int precision, int obj, int metric, bool rel_global = false);
size_t nm_smem(int precision, int obj, int32_t n_samples, bool rel_in_smem = true);
int nm_problems_per_block();
int nm_threads();
cudaError_t launch_nm(const void* fn, const NmArgs& a, int grid, size_t smem, cudaStream_t st);
// lane schedule: one problem per lane, 32 per block (opmm_nm.cu)
const void* nm_lane_kernel_ptr(int precision, int obj, int metric, bool rel_global);
size_t nm_lane_smem(int precision, int obj, int32_t n_samples, bool rel_in_smem);
cudaError_t launch_nm_lane(const void* fn, const NmArgs& a, int grid, size_t smem, cudaStream_t st);
// group schedule: 4 lanes per problem, 8 problems per 32-thread block (launch_nm_lane)
const void* nm_group_kernel_ptr(int precision, int obj, int metric, bool rel_global);
size_t nm_group_smem(int precision, int obj, int32_t n_samples, bool rel_in_smem);
int nm_group_problems_per_block();

const void* fit_kernel_ptr(int precision, int integrator, int metric, bool grid_tables = false);
// superposition over one pulse-height grid dimension (kernel_variant 4, fp64)
const void* fit_super_kernel_ptr(int metric, bool tmem, bool fp32);
constexpr int SUPER_MAX_WARPS = 8;   // per block: TMEM warps (<= 4, one per quadrant) + smem warps
constexpr int SUPER_TMEM_MAX_STEPS = 120;   // 4 TMEM columns per sample, groups of 4, 512 columns
constexpr int SUPER_MAX_L = 4096;    // levels of the superposed dimension
size_t super_smem(int32_t n_samples, int32_t levels, int32_t gt_n, int smem_warps, int tm_warps,
                  bool fp32 = false);
constexpr int32_t SUPER_MAX_GT = 2048;   // level-table entries kept in shared memory (also fit_kernel<GT>)
const void* fit2_kernel_ptr(int precision, int metric);   // 2 candidates/thread, 256 threads
constexpr int FIT2_BLOCK = 256;
const void* fit_refill_kernel_ptr(int precision, int metric);   // lane refill (f2), default block
const void* fit3_kernel_ptr(int precision, int metric);   // warp-specialised, 384 threads
constexpr int FIT3_BLOCK = 384;
size_t fit3_smem(int precision, int32_t n_samples);
const void* simscore_kernel_ptr(int precision, int integrator, int metric);
const void* simulate_kernel_ptr(int precision, int integrator);
const void* score_kernel_ptr(int precision, int metric);

cudaError_t launch_fit(const void* fn, const FitArgs& a, dim3 grid, int block, size_t smem,
                       cudaStream_t st);
// world > 1: merge the gathered rank results of saccade `sac` (rank r's at
// gathered + r * stride bytes; the lists only when a.topk) and write its final
// result; certify re-scores the merged list in fp64 (dynamic smem: the
// certify scratch)
cudaError_t launch_merge(const FitArgs& a, const void* gathered, int world, size_t stride,
                         int64_t sac, opmm_fit_result* out, int metric, size_t smem,
                         cudaStream_t st);
const void* merge_kernel_ptr(int metric);
// exact top-K of a fit from its err_out (after the fit kernel, same stream):
// grid (blocks, S), dynamic smem topk_smem(blocks, n_samples, certify)
constexpr int TOPK_BLOCK = 256;
const void* topk_kernel_ptr(int metric);
__host__ __device__ constexpr size_t topk_smem(int) { return (size_t)512 * 16; }   // TOPK_MAXFG minima
cudaError_t launch_topk(const FitArgs& a, int blocks, int S, size_t smem, int metric, cudaStream_t st);
// fp32 certification after topk_kernel (one rank): one warp per saccade,
// dynamic smem cert_scratch_bytes(n_samples)
const void* cert_kernel_ptr(int metric);
cudaError_t launch_cert(const FitArgs& a, int S, size_t smem, int metric, cudaStream_t st);
cudaError_t launch_explicit(const void* fn, const ExplicitArgs& a, dim3 grid, int block, size_t smem,
                            cudaStream_t st);
cudaError_t launch_score(const ScoreArgs& a, int precision, int metric, dim3 grid, int block,
                         size_t smem, cudaStream_t st);
cudaError_t launch_generate(const SpaceDev& sp, uint32_t saccade, int64_t begin, int64_t count,
                            double* out, int64_t ld, const double2* tab, int grid, cudaStream_t st);

}  // namespace opmm
