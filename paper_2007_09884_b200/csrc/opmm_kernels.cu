// opmm_kernels.cu -- sm_100a kernels of the libopmm hot path and their
// host-side launchers (called only from opmm_api.cu).
//
//   fit_kernel         generate -> setup -> integrate+score -> argmin, fused;
//                      warp shuffle -> shared -> per-block partial -> the last
//                      block reduces the partials.
//   merge_kernel       world > 1: lexicographic min of the gathered per-rank
//                      partials + winner regeneration (a8).
//   simscore_kernel    explicit OPC batch -> E per candidate (no trajectories).
//   simulate_kernel    explicit OPC batch -> time-major trajectories (dump mode).
//   score_kernel       stored trajectories -> E per candidate (HBM-bound).
//   generate_kernel    candidate dump (SoA), bit-identical to fit_kernel's.
#include <cstdint>
#include <cuda_runtime.h>

#include "opmm.h"
#include "opmm_device.cuh"
#include "opmm_internal.h"

namespace opmm {

// ---------------------------------------------------------------------------
// Evaluate one candidate: physical check, setup, integrate + fused score.
// ---------------------------------------------------------------------------
template <typename T, int INTEG, int METRIC, bool TRAJ>
__device__ __forceinline__ double evaluate(const double p[NP], const CtlDev& c, double Aprime,
                                           double pw_default, const T* rel, T* traj,
                                           int64_t ld_out, double sgn, uint8_t* status,
                                           T* stash, bool check_physical = true) {
  // generated candidates skip the check when the host proved the whole
  // search space physical (SpaceDev::all_physical)
  const double pen = check_physical ? physical_penalty(p) : 0.0;
  if (pen != 0.0) {
    if (TRAJ) {
      const T nanv = (T)__longlong_as_double(0x7ff8000000000000LL);
      for (int32_t k = 0; k <= c.n_steps; ++k) traj[(int64_t)k * ld_out] = nanv;
    }
    if (status) *status = 1;
    return pen;
  }
  Setup s;
  make_setup(p, c.dt_ms, c.h, c.n_steps, Aprime, pw_default, s);
  T acc;
  if (INTEG == 0) {
    Prop2<T> pr;
    make_prop<T>(s, pr);
    acc = run_propagator<T, METRIC, TRAJ>(pr, s.n_pulse, c.n_steps, rel, traj, ld_out,
                                          (T)c.theta0, (T)sgn, stash, blockDim.x);
  } else {
    acc = run_rk4_stages<T, METRIC, TRAJ>(s, c.n_steps, rel, traj, ld_out, (T)c.theta0, (T)sgn);
  }
  const double E = finish_error<METRIC>(acc, c.n_steps + 1);
  if (status) *status = isinf(E) ? 2 : 0;
  return E;
}

// ---------------------------------------------------------------------------
// Block-level (E, idx, n_finite) reduction; returns true in thread 0.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void block_argmin(double& e, int64_t& i, int64_t& nf) {
  __shared__ double se[32];
  __shared__ int64_t si[32];
  __shared__ int64_t sn[32];
  warp_argmin(e, i);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) nf += __shfl_xor_sync(0xffffffffu, nf, off);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if (lane == 0) { se[wid] = e; si[wid] = i; sn[wid] = nf; }
  __syncthreads();
  if (wid == 0) {
    e = lane < nw ? se[lane] : __longlong_as_double(0x7ff0000000000000LL);
    i = lane < nw ? si[lane] : INT64_MAX;
    nf = lane < nw ? sn[lane] : 0;
    warp_argmin(e, i);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) nf += __shfl_xor_sync(0xffffffffu, nf, off);
  }
}

// Write the final result struct (one thread) and the winner's OPC.
__device__ void write_result(const SpaceDev& sp, uint32_t saccade, double e, int64_t i,
                             int64_t nf, int64_t neval, opmm_fit_result* out,
                             const double2* tab) {
  const bool ok = i != INT64_MAX && e < __longlong_as_double(0x7ff0000000000000LL);
  out->best_index = ok ? i : -1;
  out->opt_err = ok ? e : __longlong_as_double(0x7ff0000000000000LL);
  out->cpu_check = __longlong_as_double(0x7ff8000000000000LL);
  out->n_finite = nf;
  out->n_evaluated = neval;
  double p[NP];
  if (ok) generate_opc(sp, saccade, i, p, tab);
#pragma unroll
  for (int d = 0; d < NP; ++d) out->opc[d] = ok ? p[d] : __longlong_as_double(0x7ff8000000000000LL);
}

// ---------------------------------------------------------------------------
// The fused fit kernel.  gridDim.y = saccades of this launch (1 for a single
// fit); blockIdx.x strides over the candidate range [begin, end) of each.
// ---------------------------------------------------------------------------
// The simulate kernels are register-heavy (per-candidate setup peaks near
// 240 live registers): 384 threads x 168 registers, 3 warps per scheduler,
// measured best among 128/168/238-register budgets.
#ifndef OPMM_FIT_LB_THREADS
#define OPMM_FIT_LB_THREADS 384
#endif
#ifndef OPMM_FIT_LB_BLOCKS
#define OPMM_FIT_LB_BLOCKS 1
#endif

template <typename T, int INTEG, int METRIC>
__global__ void __launch_bounds__(OPMM_FIT_LB_THREADS, OPMM_FIT_LB_BLOCKS) fit_kernel(FitArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int32_t ns = a.ctl.n_steps + 1;
  T* rel = reinterpret_cast<T*>(smem_raw);
  double2* tab = reinterpret_cast<double2*>(smem_raw + rel_bytes<T>(ns));
  T* stash = reinterpret_cast<T*>(smem_raw + rel_bytes<T>(ns) + exp_tab_bytes());  // [8][block] vec2
  for (int j = threadIdx.x; j < EXP_TAB_N; j += blockDim.x) tab[j] = a.exp_tab[j];
  const int64_t sac = (int64_t)blockIdx.y + a.sac_begin;
  const double amp = a.sac_ctl ? a.sac_ctl[2 * sac] : a.amplitude;
  const double pwd = a.sac_ctl ? a.sac_ctl[2 * sac + 1] : a.pw_default;
  double sgn, Aprime;
  stage_trace<T>(a.rec + sac * (int64_t)ns, ns, amp, rel, sgn, Aprime);
  __syncthreads();
#ifdef OPMM_STAGGER
  if ((threadIdx.x >> 5) & 1) {
    const long long t0 = clock64();
    while (clock64() - t0 < OPMM_STAGGER) {
    }
  }
#endif

  double best_e = __longlong_as_double(0x7ff0000000000000LL);
  int64_t best_i = INT64_MAX;
  int64_t nf = 0;
  // Warp-uniform trip count: every lane of a warp runs every iteration (lanes
  // past `end` evaluate the last candidate again and discard it), so the
  // per-step warp vote in run_propagator always sees a full warp.
  // Lane sort: each tile of blockDim candidates is counting-sorted by the
  // block index at which its pulse ends (n_pulse / 2, 256 bins), so a warp's
  // lanes share few phase-switch points and run_propagator's segmented loop
  // has few segments.  Only the candidate->thread assignment changes; every
  // result is per candidate, so outputs are identical (and deterministic).
  __shared__ int s_hist[256];
  __shared__ int s_wsum[32];
  __shared__ int s_perm[OPMM_FIT_LB_THREADS];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = a.begin + (int64_t)blockIdx.x * blockDim.x; base < a.end; base += stride) {
    int src = tid;
    if (a.sort_lanes) {
      const int nbins = blockDim.x < 256 ? (int)blockDim.x : 256;   // multiple of 32
      const int64_t j0 = base + tid;
      int key = nbins - 1;                                          // padding lanes last
      if (j0 < a.end) {
        const double pw = generate_pw(a.space, (uint32_t)sac, j0, tab);
        const double npd = ceil(pw / a.ctl.dt_ms);
        const int np = npd > (double)a.ctl.n_steps ? a.ctl.n_steps + 1 : (int)npd;
        key = min(np >> 1, nbins - 2);
      }
      if (tid < nbins) s_hist[tid] = 0;
      __syncthreads();
      const int rank = atomicAdd(&s_hist[key], 1);
      __syncthreads();
      int v = 0, incl = 0;
      if (tid < nbins) {
        v = s_hist[tid];
        incl = v;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, incl, off);
          if (lane >= off) incl += t;
        }
        if (lane == 31) s_wsum[wid] = incl;
      }
      __syncthreads();
      if (tid < 32) {
        const int nw = nbins >> 5;
        const int w = tid < nw ? s_wsum[tid] : 0;
        int inc = w;
#pragma unroll
        for (int off = 1; off < 8; off <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, inc, off);
          if (lane >= off) inc += t;
        }
        if (tid < nw) s_wsum[tid] = inc - w;
      }
      __syncthreads();
      if (tid < nbins) s_hist[tid] = incl - v + s_wsum[wid];
      __syncthreads();
      s_perm[s_hist[key] + rank] = tid;
      __syncthreads();
      src = s_perm[tid];
    }
    // Warp-uniform trip count: every lane of a warp runs every iteration
    // (lanes past `end` evaluate the last candidate again and discard it), so
    // the warp-level reductions in run_propagator always see a full warp.
    const int64_t i0 = base + src;
    const bool valid = i0 < a.end;
    const int64_t i = valid ? i0 : a.end - 1;
    double p[NP];
    generate_opc(a.space, (uint32_t)sac, i, p, tab);
    const double E = evaluate<T, INTEG, METRIC, false>(p, a.ctl, Aprime, pwd, rel, nullptr, 0,
                                                       sgn, nullptr, stash, !a.space.all_physical);
    if (valid) {
      if (a.err_out) a.err_out[sac * a.err_ld + i] = E;
      nf += E < __longlong_as_double(0x7ff0000000000000LL) ? 1 : 0;
      if (better(E, i, best_e, best_i)) { best_e = E; best_i = i; }
    }
  }
  block_argmin(best_e, best_i, nf);

  // per-block partial, then the last block of this saccade reduces them
  __shared__ bool is_last;
  Partial* parts = a.partials + sac * (int64_t)gridDim.x;
  if (threadIdx.x == 0) {
    parts[blockIdx.x] = Partial{best_e, best_i, nf, 0};
    __threadfence();
    const unsigned int t = atomicAdd(a.counters + sac, 1u);
    is_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  double e = __longlong_as_double(0x7ff0000000000000LL);
  int64_t i = INT64_MAX, n = 0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
    // L2-coherent loads: the partials were written by other blocks
    const double qe = __ldcg(&parts[b].e);
    const int64_t qi = __ldcg(reinterpret_cast<const long long*>(&parts[b].i));
    const int64_t qn = __ldcg(reinterpret_cast<const long long*>(&parts[b].nf));
    if (better(qe, qi, e, i)) { e = qe; i = qi; }
    n += qn;
  }
  __syncthreads();
  block_argmin(e, i, n);
  if (threadIdx.x == 0) {
    a.counters[sac] = 0;  // re-arm for the next launch (graph-replay safe)
    const int64_t neval = a.end - a.begin;
    if (a.rank_out) a.rank_out[sac] = Partial{e, i, n, neval};
    if (a.final_out)
      write_result(a.space, (uint32_t)sac, e, i, n, neval, a.final_out + (sac - a.out_base),
                   a.exp_tab);
  }
}

// ---------------------------------------------------------------------------
// world > 1: merge the gathered per-rank partials (lexicographic) and write
// the final result with the regenerated winner OPC.  One warp.
// ---------------------------------------------------------------------------
__global__ void merge_kernel(const Partial* gathered, int world, SpaceDev sp, uint32_t saccade,
                             opmm_fit_result* out, const double2* tab) {
  double e = __longlong_as_double(0x7ff0000000000000LL);
  int64_t i = INT64_MAX, n = 0, ne = 0;
  for (int r = threadIdx.x; r < world; r += 32) {
    const Partial q = gathered[r];
    if (better(q.e, q.i, e, i)) { e = q.e; i = q.i; }
    n += q.nf;
    ne += q.neval;
  }
  warp_argmin(e, i);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    n += __shfl_xor_sync(0xffffffffu, n, off);
    ne += __shfl_xor_sync(0xffffffffu, ne, off);
  }
  if (threadIdx.x == 0) write_result(sp, saccade, e, i, n, ne, out, tab);
}

// ---------------------------------------------------------------------------
// Explicit OPC batch kernels.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void load_opc(const double* __restrict__ opc, int64_t ld, int64_t i,
                                         double p[NP]) {
#pragma unroll
  for (int d = 0; d < NP; ++d) p[d] = __ldg(opc + (int64_t)d * ld + i);
}

template <typename T, int INTEG, int METRIC>
__global__ void __launch_bounds__(OPMM_FIT_LB_THREADS, OPMM_FIT_LB_BLOCKS) simscore_kernel(ExplicitArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int32_t ns = a.ctl.n_steps + 1;
  T* rel = reinterpret_cast<T*>(smem_raw);
  T* stash = reinterpret_cast<T*>(smem_raw + rel_bytes<T>(ns));  // [8][block] vec2
  double sgn, Aprime;
  stage_trace<T>(a.rec, ns, a.amplitude, rel, sgn, Aprime);
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < a.n; base += stride) {
    const int64_t i0 = base + threadIdx.x;
    const bool valid = i0 < a.n;
    const int64_t i = valid ? i0 : a.n - 1;
    double p[NP];
    load_opc(a.opc, a.ld, i, p);
    const double E = evaluate<T, INTEG, METRIC, false>(p, a.ctl, Aprime, a.pw_default, rel, nullptr,
                                                       0, sgn, nullptr, stash);
    if (valid) a.err[i] = E;
  }
}

template <typename T, int INTEG>
__global__ void __launch_bounds__(OPMM_FIT_LB_THREADS, OPMM_FIT_LB_BLOCKS) simulate_kernel(ExplicitArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* stash = reinterpret_cast<T*>(smem_raw);  // [8][block] vec2
  const double A = a.amplitude;  // explicit simulate: A given (NaN rejected on host)
  const double sgn = A < 0.0 ? -1.0 : 1.0, Aprime = fabs(A);
  T* traj = reinterpret_cast<T*>(a.traj);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < a.n; base += stride) {
    const int64_t i0 = base + threadIdx.x;
    const bool valid = i0 < a.n;
    // invalid lanes re-integrate candidate n-1 and store the identical values
    // into its column (benign duplicate writes)
    const int64_t i = valid ? i0 : a.n - 1;
    double p[NP];
    load_opc(a.opc, a.ld, i, p);
    uint8_t st = 0;
    // no trace: the accumulator sums |Delta-theta| so that a non-finite (or
    // >= 1e20) trajectory is flagged as diverged (status 2)
    (void)evaluate<T, INTEG, 0, true>(p, a.ctl, Aprime, a.pw_default, nullptr, traj + i,
                                      a.ld_out, sgn, &st, stash);
    if (valid && a.status) a.status[i] = st;
  }
}

// Stored-trajectory score: one candidate per thread, samples streamed
// time-major (coalesced across the warp), 8 loads in flight per thread.
template <typename T, int METRIC>
__global__ void __launch_bounds__(256) score_kernel(ScoreArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* rec = reinterpret_cast<double*>(smem_raw);
  for (int k = threadIdx.x; k < a.n_samples; k += blockDim.x) rec[k] = a.rec[k];
  __syncthreads();
  const T* traj = reinterpret_cast<const T*>(a.traj);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {
    double acc = 0.0;
    int32_t k = 0;
    for (; k + 8 <= a.n_samples; k += 8) {
      T v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcs(traj + (int64_t)(k + u) * a.ld + i);
#pragma unroll
      for (int u = 0; u < 8; ++u) accumulate<METRIC>(acc, (double)v[u] - rec[k + u]);
    }
    for (; k < a.n_samples; ++k) accumulate<METRIC>(acc, (double)__ldcs(traj + (int64_t)k * a.ld + i) - rec[k]);
    a.err[i] = finish_error<METRIC>(acc, a.n_samples);
  }
}

__global__ void generate_kernel(SpaceDev sp, uint32_t saccade, int64_t begin, int64_t count,
                                double* out, int64_t ld, const double2* tab) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += stride) {
    double p[NP];
    generate_opc(sp, saccade, begin + j, p, tab);
#pragma unroll
    for (int d = 0; d < NP; ++d) out[(int64_t)d * ld + j] = p[d];
  }
}

// ---------------------------------------------------------------------------
// Launchers.
// ---------------------------------------------------------------------------
template <typename T, int INTEG, int METRIC>
static const void* fit_fn() { return reinterpret_cast<const void*>(&fit_kernel<T, INTEG, METRIC>); }

const void* fit_kernel_ptr(int precision, int integrator, int metric) {
  if (precision == 0) {
    if (integrator == 0) return metric == 0 ? fit_fn<double, 0, 0>() : fit_fn<double, 0, 1>();
    return metric == 0 ? fit_fn<double, 1, 0>() : fit_fn<double, 1, 1>();
  }
  if (integrator == 0) return metric == 0 ? fit_fn<float, 0, 0>() : fit_fn<float, 0, 1>();
  return metric == 0 ? fit_fn<float, 1, 0>() : fit_fn<float, 1, 1>();
}

cudaError_t launch_fit(const FitArgs& a, int precision, int integrator, int metric, dim3 grid,
                       int block, size_t smem, cudaStream_t st) {
  void* args[] = {const_cast<FitArgs*>(&a)};
  return cudaLaunchKernel(fit_kernel_ptr(precision, integrator, metric), grid, dim3(block), args,
                          smem, st);
}

cudaError_t launch_merge(const Partial* gathered, int world, const SpaceDev& sp, uint32_t saccade,
                         opmm_fit_result* out, const double2* tab, cudaStream_t st) {
  merge_kernel<<<1, 32, 0, st>>>(gathered, world, sp, saccade, out, tab);
  return cudaGetLastError();
}

template <typename T, int INTEG, int METRIC>
static const void* ss_fn() { return reinterpret_cast<const void*>(&simscore_kernel<T, INTEG, METRIC>); }

const void* simscore_kernel_ptr(int precision, int integrator, int metric) {
  if (precision == 0) {
    if (integrator == 0) return metric == 0 ? ss_fn<double, 0, 0>() : ss_fn<double, 0, 1>();
    return metric == 0 ? ss_fn<double, 1, 0>() : ss_fn<double, 1, 1>();
  }
  if (integrator == 0) return metric == 0 ? ss_fn<float, 0, 0>() : ss_fn<float, 0, 1>();
  return metric == 0 ? ss_fn<float, 1, 0>() : ss_fn<float, 1, 1>();
}

const void* simulate_kernel_ptr(int precision, int integrator) {
  if (precision == 0)
    return integrator == 0 ? reinterpret_cast<const void*>(&simulate_kernel<double, 0>)
                           : reinterpret_cast<const void*>(&simulate_kernel<double, 1>);
  return integrator == 0 ? reinterpret_cast<const void*>(&simulate_kernel<float, 0>)
                         : reinterpret_cast<const void*>(&simulate_kernel<float, 1>);
}

const void* score_kernel_ptr(int precision, int metric) {
  if (precision == 0)
    return metric == 0 ? reinterpret_cast<const void*>(&score_kernel<double, 0>)
                       : reinterpret_cast<const void*>(&score_kernel<double, 1>);
  return metric == 0 ? reinterpret_cast<const void*>(&score_kernel<float, 0>)
                     : reinterpret_cast<const void*>(&score_kernel<float, 1>);
}

cudaError_t launch_explicit(const void* fn, const ExplicitArgs& a, dim3 grid, int block, size_t smem,
                            cudaStream_t st) {
  void* args[] = {const_cast<ExplicitArgs*>(&a)};
  return cudaLaunchKernel(fn, grid, dim3(block), args, smem, st);
}

cudaError_t launch_score(const ScoreArgs& a, int precision, int metric, dim3 grid, int block,
                         size_t smem, cudaStream_t st) {
  void* args[] = {const_cast<ScoreArgs*>(&a)};
  return cudaLaunchKernel(score_kernel_ptr(precision, metric), grid, dim3(block), args, smem, st);
}

cudaError_t launch_generate(const SpaceDev& sp, uint32_t saccade, int64_t begin, int64_t count,
                            double* out, int64_t ld, const double2* tab, int grid, cudaStream_t st) {
  generate_kernel<<<grid, 256, 0, st>>>(sp, saccade, begin, count, out, ld, tab);
  return cudaGetLastError();
}

}  // namespace opmm
