// opmm_api.cu -- the C ABI of libopmm (include/opmm.h): argument validation,
// search-space preprocessing, handle / workspace / stream management, kernel
// launch configuration, the multi-GPU merge (NCCL, loaded at run time), and
// the paper's CPU_check column.  Every step of the hot path itself runs in
// the kernels of opmm_kernels.cu; nothing here computes candidates on the CPU.
#include <cmath>
#include <cfloat>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <dlfcn.h>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>

#include "opmm.h"
#include "opmm_cpu_check.h"
#include "opmm_internal.h"

using opmm::Partial;

// ABI layout (mirrored by the ctypes binding; checked by tests/test_abi.py)
static_assert(sizeof(opmm_control) == 40, "opmm_control layout");
static_assert(sizeof(opmm_search_space) == 400, "opmm_search_space layout");
static_assert(sizeof(opmm_fit_options) == 48, "opmm_fit_options layout");
static_assert(sizeof(opmm_fit_result) == 704, "opmm_fit_result layout");
static_assert(sizeof(Partial) == 32, "Partial layout");
static_assert(sizeof(opmm::RankPartial) == 544, "RankPartial layout");
static_assert(sizeof(opmm_nm_options) == 56, "opmm_nm_options layout");
static_assert(sizeof(opmm_nm_result) == 176, "opmm_nm_result layout");

namespace {

thread_local std::string g_err;

opmm_status fail(opmm_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return fail(e_ == cudaErrorMemoryAllocation ? OPMM_ERR_OOM : OPMM_ERR_CUDA,     \
                  "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__,   \
                  __LINE__);                                                          \
  } while (0)

#define CKS(expr)                          \
  do {                                     \
    opmm_status s_ = (expr);               \
    if (s_ != OPMM_OK) return s_;          \
  } while (0)

// ---------------------------------------------------------------------------
// NCCL, resolved at run time (the process normally already has torch's
// libnccl.so.2 loaded; we reuse it rather than link a second copy).
// ---------------------------------------------------------------------------
struct NcclApi {
  bool loaded = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  if (!api.loaded) {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
      api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
      api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
      api.allGather = (decltype(api.allGather))dlsym(h, "ncclAllGather");
      api.getErrorString = (decltype(api.getErrorString))dlsym(h, "ncclGetErrorString");
      api.loaded = api.getUniqueId && api.commInitRank && api.commDestroy && api.allGather &&
                   api.getErrorString;
    }
  }
  return api;
}

constexpr int kDefaultBlock = OPMM_FIT_LB_THREADS;   // opmm_internal.h
constexpr size_t kMaxDynSmem = 220 * 1024;
// fit kernel picked by kernel_variant = 0 when variants 2/3 apply (1 otherwise)
constexpr int kAutoVariant = 1;
// kernel_variant = 0 picks the superposition kernel (variant 4) for eligible
// grids with at least this many pulse-height levels
constexpr bool kAutoSuper = true;
constexpr int32_t kSuperMinLevels = 8;
// certify's list length when top_k = 0
constexpr int kCertifyK = 8;
// The superposition kernel's tensor-memory layout (4 warps keep their
// columns in TMEM, 8 warps per SM instead of 4) overlaps one warp's
// latency-bound per-node setup with another's level loop: faster than the
// shared-memory layout at every level count measured.
// OPMM_FIT_FLAG_SUPER_SMEM forces the shared-memory layout (A/B timing, tests).
bool super_tmem_wanted(const opmm_fit_options* opts) {
  return !(opts && (opts->flags & OPMM_FIT_FLAG_SUPER_SMEM));
}

}  // namespace

struct opmm_handle {
  int device = 0;
  int rank = 0, world = 1;
  int num_sms = 0;
  cudaStream_t stream = nullptr;
  ncclComm_t comm = nullptr;
  // workspace
  Partial* partials = nullptr;
  size_t partials_cap = 0;
  unsigned int* counters = nullptr;
  size_t counters_cap = 0;
  double* rec = nullptr;
  size_t rec_cap = 0;
  double* sacctl = nullptr;
  size_t sacctl_cap = 0;
  double* nm_rel = nullptr;    // Nelder-Mead: relativized traces too long for shared memory
  size_t nm_rel_cap = 0;
  double* candctl = nullptr;   // opmm_simulate_batch: [n][3] per-candidate controls
  size_t candctl_cap = 0;
  // opmm_fit's CUDA graph: [H2D of the staged trace, event, fit kernel,
  // event, D2H of the result] captured once and replayed while the launch
  // (kernel, configuration and every FitArgs byte) is unchanged
  cudaGraphExec_t fit_graph = nullptr;
  std::string fit_graph_key;
  double* rec_stage = nullptr;   // pinned host staging of the recorded trace
  size_t rec_stage_cap = 0;
  const void* occ_fn = nullptr;  // grid_for's last occupancy query
  int occ_block = 0;
  size_t occ_smem = 0;
  int occ_per_sm = 0;
  opmm::RankPartial* rank_part = nullptr;   // world > 1: this rank's result per saccade
  size_t rank_part_cap = 0;
  opmm::RankPartial* gathered = nullptr;    // all ranks' results (packed, 32 or 544 B each)
  size_t gathered_cap = 0;
  void* stage[4] = {nullptr, nullptr, nullptr, nullptr};   // host-pointer staging (Staging)
  size_t stage_cap[4] = {0, 0, 0, 0};
  double* tk_e = nullptr;                   // top-K: per-block lists [S][grid][32]
  size_t tk_e_cap = 0;
  int64_t* tk_i = nullptr;
  size_t tk_i_cap = 0;
  unsigned int* tk_counters = nullptr;      // top-K: topk_kernel tickets + fill counts [2][S]
  size_t tk_counters_cap = 0;
  unsigned long long* sup_next = nullptr;   // superposition: node-group counters [S]
  size_t sup_next_cap = 0;
  double* tk_err = nullptr;                 // top-K: the fit's errors when err_out is not given
  size_t tk_err_cap = 0;
  opmm_fit_result* result = nullptr;
  size_t result_cap = 0;
  opmm_fit_result* result_host = nullptr;  // pinned
  size_t result_host_cap = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  bool timing = false;   // opmm_set_kernel_timing: record the events below
  bool timed = false;    // ev0/ev1 bracket the most recent timed launch
  double2* exp_tab = nullptr;   // exp(j/64) double-double table (generator)
  // Nelder-Mead workspace
  double* nm_x0 = nullptr;
  size_t nm_x0_cap = 0;
  double* nm_xbest = nullptr;
  size_t nm_xbest_cap = 0;
  opmm::NmOut* nm_out = nullptr;
  size_t nm_out_cap = 0;
  unsigned long long* nm_next = nullptr;    // NM group schedule: refill counter
  size_t nm_next_cap = 0;
};

namespace {

template <typename P>
opmm_status ensure(P*& ptr, size_t& cap, size_t n, bool zero = false) {
  if (n <= cap) return OPMM_OK;
  if (ptr) cudaFree(ptr);
  ptr = nullptr;
  cap = 0;
  size_t want = n < 64 ? 64 : n;
  CK(cudaMalloc(reinterpret_cast<void**>(&ptr), want * sizeof(P)));
  if (zero) CK(cudaMemset(ptr, 0, want * sizeof(P)));
  cap = want;
  return OPMM_OK;
}

opmm_status ensure_host(opmm_fit_result*& ptr, size_t& cap, size_t n) {
  if (n <= cap) return OPMM_OK;
  if (ptr) cudaFreeHost(ptr);
  ptr = nullptr;
  cap = 0;
  CK(cudaMallocHost(reinterpret_cast<void**>(&ptr), n * sizeof(opmm_fit_result)));
  cap = n;
  return OPMM_OK;
}

bool is_finite(double x) { return std::isfinite(x); }

opmm_status check_handle(opmm_handle* h) {
  if (!h) return fail(OPMM_ERR_INVALID_ARG, "handle is NULL");
  CK(cudaSetDevice(h->device));
  return OPMM_OK;
}

opmm_status validate_control(const opmm_control* c, bool need_amplitude) {
  if (!c) return fail(OPMM_ERR_INVALID_ARG, "control is NULL");
  if (!(c->dt_ms > 0.0) || !is_finite(c->dt_ms))
    return fail(OPMM_ERR_INVALID_ARG, "dt_ms must be finite and > 0 (got %g)", c->dt_ms);
  if (c->n_steps < 1 || c->n_steps > OPMM_MAX_STEPS)
    return fail(OPMM_ERR_INVALID_ARG, "n_steps must be in [1, %d] (got %d)", OPMM_MAX_STEPS,
                c->n_steps);
  if (!is_finite(c->theta0_deg)) return fail(OPMM_ERR_INVALID_ARG, "theta0_deg must be finite");
  if (std::isinf(c->amplitude_deg)) return fail(OPMM_ERR_INVALID_ARG, "amplitude_deg is infinite");
  if (need_amplitude && std::isnan(c->amplitude_deg))
    return fail(OPMM_ERR_INVALID_ARG, "amplitude_deg must be given (no recorded trace here)");
  if (!(c->pw_default_ms > 0.0) || !is_finite(c->pw_default_ms))
    return fail(OPMM_ERR_INVALID_ARG, "pw_default_ms must be finite and > 0");
  if (c->substeps < 0 || c->substeps > OPMM_MAX_SUBSTEPS)
    return fail(OPMM_ERR_INVALID_ARG, "substeps must be in [0, %d] (got %d)", OPMM_MAX_SUBSTEPS,
                c->substeps);
  return OPMM_OK;
}

opmm_status validate_space(const opmm_search_space* s, int64_t n) {
  if (!s) return fail(OPMM_ERR_INVALID_ARG, "search space is NULL");
  if (s->mode != 0 && s->mode != 1) return fail(OPMM_ERR_INVALID_ARG, "mode must be 0 or 1");
  if (s->model != 0 && s->model != 1) return fail(OPMM_ERR_INVALID_ARG, "model must be 0 or 1");
  for (int d = 0; d < OPMM_NPARAM; ++d) {
    if (!is_finite(s->lo[d]) || !is_finite(s->hi[d]))
      return fail(OPMM_ERR_INVALID_ARG, "bounds of dimension %d must be finite", d);
    if (s->lo[d] > s->hi[d]) return fail(OPMM_ERR_INVALID_ARG, "lo > hi in dimension %d", d);
    if (s->log_scale[d] > 1) return fail(OPMM_ERR_INVALID_ARG, "log_scale[%d] must be 0/1", d);
    if (s->log_scale[d] && s->lo[d] != s->hi[d] && !(s->lo[d] > 0.0))
      return fail(OPMM_ERR_INVALID_ARG, "log dimension %d needs lo > 0", d);
  }
  if (s->mode == 1) {
    long double prod = 1.0L;
    int64_t p = 1;
    for (int d = 0; d < OPMM_NPARAM; ++d) {
      if (s->levels[d] < 1) return fail(OPMM_ERR_INVALID_ARG, "levels[%d] must be >= 1", d);
      prod *= (long double)s->levels[d];
      if (prod > 9.2e18L) return fail(OPMM_ERR_INVALID_ARG, "grid too large");
      p *= s->levels[d];
    }
    if (n >= 0 && p != n)
      return fail(OPMM_ERR_INVALID_ARG, "grid product %lld != n_candidates %lld", (long long)p,
                  (long long)n);
  }
  return OPMM_OK;
}

// Host preprocessing of the search space: key split, per-dimension kind and
// span (log(hi/lo) or hi-lo, over (L-1) in grid mode) -- the same
// expressions the method's generator definition uses (opmm.h).
opmm::SpaceDev make_space(const opmm_search_space* s) {
  opmm::SpaceDev d;
  std::memset(&d, 0, sizeof(d));
  d.mode = s->mode;
  d.model = s->model;
  d.key0 = (uint32_t)(s->seed & 0xffffffffu);
  d.key1 = (uint32_t)(s->seed >> 32);
  for (int k = 0; k < OPMM_NPARAM; ++k) {
    d.lo[k] = s->lo[k];
    d.levels[k] = s->mode == 1 ? s->levels[k] : 1;
    const bool fixed = s->lo[k] == s->hi[k] || (s->mode == 1 && s->levels[k] <= 1);
    if (fixed) {
      d.kind[k] = 0;
      d.span[k] = 0.0;
    } else if (s->log_scale[k]) {
      const double L = std::log(s->hi[k] / s->lo[k]);
      d.span[k] = s->mode == 1 ? L / (double)(s->levels[k] - 1) : L;
      // largest exp argument the generator can form for this dimension
      const double xmax = s->mode == 1 ? d.span[k] * (double)(s->levels[k] - 1) : L;
      d.kind[k] = xmax < 0.999 * opmm::EXP_TAB_MAX ? 2 : 3;
    } else {
      d.kind[k] = 1;
      const double w = s->hi[k] - s->lo[k];
      d.span[k] = s->mode == 1 ? w / (double)(s->levels[k] - 1) : w;
    }
  }
  // Every candidate lies in [lo, hi] per dimension, so the physical check
  // (SPEC D8 / reading Q13) holds for all of them iff it holds at the lower
  // corner: strict dimensions lo > 0, the others lo >= 0, and G > 0, which
  // (with K_SE > 0) needs N_C + K_LT > 0 for at least one muscle.
  static const int strict[] = {OPMM_P_KSE_AG, OPMM_P_KSE_ANT, OPMM_P_B_AG, OPMM_P_B_ANT,
                               OPMM_P_J, OPMM_P_TAU_AC_AG, OPMM_P_TAU_AC_ANT, OPMM_P_TAU_DE_AG,
                               OPMM_P_TAU_DE_ANT, OPMM_P_PW};
  bool phys = true;
  for (int k = 0; k < OPMM_NPARAM; ++k) {
    bool is_strict = false;
    for (int t : strict) is_strict |= (t == k);
    if (is_strict ? !(s->lo[k] > 0.0) : !(s->lo[k] >= 0.0)) phys = false;
  }
  if (!(s->lo[OPMM_P_NC_AG] + s->lo[OPMM_P_KLT_AG] > 0.0 ||
        s->lo[OPMM_P_NC_ANT] + s->lo[OPMM_P_KLT_ANT] > 0.0))
    phys = false;
  d.all_physical = phys ? 1 : 0;
  bool kinds012 = true;
  for (int k = 0; k < OPMM_NPARAM; ++k) {
    d.span32[k] = std::ldexp(d.span[k], -32);
    if (d.span[k] != 0.0 && !(std::fabs(d.span32[k]) >= DBL_MIN)) d.exact_u = 1;
    // (a fixed -0.0 would come out +0.0 from the branch-free form)
    kinds012 = kinds012 && d.kind[k] <= 2 && !(d.lo[k] == 0.0 && std::signbit(d.lo[k]));
    d.gsel[k] = d.kind[k] == 2 ? 1.0 : 0.0;
    d.lsel[k] = d.kind[k] == 1 ? 1.0 : 0.0;
  }
  d.fast_gen = (s->mode == 0 && !d.exact_u && kinds012) ? 1 : 0;
  d.pw_stride = 1;
  if (s->mode == 1)
    for (int k = 0; k < OPMM_P_PW; ++k) d.pw_stride *= s->levels[k];
  return d;
}

// Opt a kernel in to the largest dynamic shared memory it can use: the
// per-block maximum less its static shared memory (an attribute above that
// is rejected and would leave the 48 KB default).
// Dynamic shared memory a kernel may request (opt-in limit less its static
// shared memory, capped at kMaxDynSmem).
size_t max_dyn_smem(const void* fn) {
  thread_local const void* last_fn = nullptr;
  thread_local int last_dev = -1;
  thread_local size_t last = 0;
  int cur = -1;
  if (cudaGetDevice(&cur) == cudaSuccess && fn == last_fn && cur == last_dev) return last;
  cudaFuncAttributes fa;
  int dev = 0, optin = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess ||
      cudaFuncGetAttributes(&fa, fn) != cudaSuccess)
    return 48 * 1024;
  size_t dyn = (size_t)optin > fa.sharedSizeBytes ? (size_t)optin - fa.sharedSizeBytes : 0;
  last_fn = fn;
  last_dev = dev;
  last = dyn > kMaxDynSmem ? kMaxDynSmem : dyn;
  return last;
}

// The opt-in limit less static shared memory, without kMaxDynSmem's cap.
size_t max_dyn_smem_uncapped(const void* fn) {
  cudaFuncAttributes fa;
  int dev = 0, optin = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess ||
      cudaFuncGetAttributes(&fa, fn) != cudaSuccess)
    return 48 * 1024;
  return (size_t)optin > fa.sharedSizeBytes ? (size_t)optin - fa.sharedSizeBytes : 0;
}

void allow_dyn_smem(const void* fn) {
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)max_dyn_smem(fn));
}

// Kernel integrator: the public PROPAGATOR with substeps > 1 runs the
// internal instantiation 2 (sample map = substep map ^ substeps, Q25).
int kernel_integ(int integrator, const opmm_control* c) {
  return (integrator == OPMM_INTEG_PROPAGATOR && c && c->substeps > 1) ? 2 : integrator;
}

opmm::CtlDev make_ctl(const opmm_control* c) {
  opmm::CtlDev d;
  d.dt_ms = c->dt_ms;
  d.h = 1e-3 * c->dt_ms;
  d.n_steps = c->n_steps;
  d.theta0 = c->theta0_deg;
  d.substeps = c->substeps > 1 ? c->substeps : 1;
  return d;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// a kernel may write through p: device or managed memory, or mapped pinned
// host memory whose device address is p itself (UVA)
bool is_device_accessible(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged ||
         (a.type == cudaMemoryTypeHost && a.devicePointer == p);
}

// Host-or-device buffers of the asynchronous entry points (SURVEY 8(b):
// "pointers may be host or device; the library detects which with
// cudaPointerGetAttributes").  A device (or managed) pointer is used in place.
// A host input is copied into a handle-owned device buffer on the call's
// stream; a host output is staged the same way (its current contents copied
// in first, so entries the kernel does not write -- padding columns, skipped
// statuses -- come back unchanged) and copied back after the kernel, and the
// call then synchronises the stream so the results are in the caller's memory
// when it returns.  One staging slot per argument position.
struct Staging {
  opmm_handle* h;
  cudaStream_t st;
  struct Out { void* host; void* dev; size_t bytes; };
  Out outs[3];
  int n_out = 0;
  Staging(opmm_handle* hh, cudaStream_t s) : h(hh), st(s) {}
  opmm_status slot(int k, size_t bytes) {
    if (bytes <= h->stage_cap[k]) return OPMM_OK;
    if (h->stage[k]) {
      CK(cudaStreamSynchronize(st));   // the old buffer may still be in use
      cudaFree(h->stage[k]);
    }
    h->stage[k] = nullptr;
    h->stage_cap[k] = 0;
    CK(cudaMalloc(&h->stage[k], bytes));
    h->stage_cap[k] = bytes;
    return OPMM_OK;
  }
  template <typename P>
  opmm_status in(P* p, size_t bytes, int k, P** dev) {
    *dev = p;
    if (p == nullptr || bytes == 0 || is_device_ptr(p)) return OPMM_OK;
    CKS(slot(k, bytes));
    CK(cudaMemcpyAsync(h->stage[k], p, bytes, cudaMemcpyHostToDevice, st));
    *dev = static_cast<P*>(h->stage[k]);
    return OPMM_OK;
  }
  template <typename P>
  opmm_status out(P* p, size_t bytes, int k, P** dev) {
    CKS(in(p, bytes, k, dev));
    if (*dev != p) outs[n_out++] = Out{(void*)p, (void*)*dev, bytes};
    return OPMM_OK;
  }
  opmm_status finish() {
    for (int j = 0; j < n_out; ++j)
      CK(cudaMemcpyAsync(outs[j].host, outs[j].dev, outs[j].bytes, cudaMemcpyDeviceToHost, st));
    if (n_out > 0) CK(cudaStreamSynchronize(st));
    return OPMM_OK;
  }
};

int check_precision(int32_t p) { return p == OPMM_FP64 || p == OPMM_FP32; }

size_t sim_smem(int precision, int32_t n_samples, int block, bool with_rel) {
  if (precision == OPMM_FP64)
    return (with_rel ? opmm::rel_bytes<double>(n_samples) : 0) + opmm::stash_bytes<double>(block);
  return (with_rel ? opmm::rel_bytes<float>(n_samples) : 0) + opmm::stash_bytes<float>(block);
}

size_t fit_smem(int precision, int32_t n_samples, int block, int kernel_variant = 1) {
  if (precision == OPMM_FP64)
    return opmm::rel_bytes<double>(n_samples) + opmm::stash_bytes<double>(block, kernel_variant) +
           opmm::exp_tab_bytes();
  return opmm::rel_bytes<float>(n_samples) + opmm::stash_bytes<float>(block, kernel_variant) +
         opmm::exp_tab_bytes();
}

opmm_status grid_for(opmm_handle* h, const void* fn, int block, size_t smem, int64_t work,
                     int requested, int* grid) {
  int per_sm = 0;
  // the occupancy query costs microseconds; the handle remembers the last one
  if (fn == h->occ_fn && block == h->occ_block && smem == h->occ_smem) {
    per_sm = h->occ_per_sm;
  } else {
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, block, smem));
    h->occ_fn = fn;
    h->occ_block = block;
    h->occ_smem = smem;
    h->occ_per_sm = per_sm;
  }
  if (per_sm < 1) return fail(OPMM_ERR_UNSUPPORTED, "kernel does not fit on an SM (block %d)", block);
  int64_t g = (int64_t)h->num_sms * per_sm;  // persistent: one wave of resident blocks
  const int64_t need = (work + block - 1) / block;
  if (requested > 0) g = requested;
  if (g > need) g = need;
  if (g < 1) g = 1;
  *grid = (int)g;
  return OPMM_OK;
}

opmm_status check_block(int block) {
  // the simulate kernels are compiled with __launch_bounds__(384, 1): <= 168 regs
  if (block < 64 || block > kDefaultBlock || block % 32 != 0)
    return fail(OPMM_ERR_INVALID_ARG, "block_size must be a multiple of 32 in [64, 384]");
  return OPMM_OK;
}

// Kernel timing is opt-in (opmm_set_kernel_timing): each pair of timing
// events costs ~6 us of stream time per call (measured), which a caller
// that does not read opmm_last_kernel_ms should not pay.
opmm_status record_start(opmm_handle* h, cudaStream_t st) {
  if (!h->timing) {
    h->timed = false;
    return OPMM_OK;
  }
  CK(cudaEventRecord(h->ev0, st));
  return OPMM_OK;
}
opmm_status record_stop(opmm_handle* h, cudaStream_t st) {
  if (!h->timing) return OPMM_OK;
  CK(cudaEventRecord(h->ev1, st));
  h->timed = true;
  return OPMM_OK;
}

opmm_status nccl_fail(ncclResult_t r, const char* what) {
  return fail(OPMM_ERR_NCCL, "%s failed: %s", what, nccl().getErrorString(r));
}

// Enqueue one fit (candidates sharded over the handle's ranks) for saccades
// [s_begin, s_begin + S) of a batch, writing final results to out_dev[S].
// A prepared single-saccade, single-rank fit launch (opmm_fit's graph path).
struct FitLaunch {
  const void* fn = nullptr;
  int grid = 0, block = 0;
  size_t smem = 0;
  opmm::FitArgs a;
};

// topk_kernel blocks per saccade: enough 256-thread blocks to stream the
// errors at HBM speed (a few batches of 32 per warp), at most one per SM for
// a single fit (the last block stages every block's list in shared memory)
int topk_blocks(opmm_handle* h, int64_t n, int64_t S) {
  const int64_t want = (n + 8 * opmm::TOPK_BLOCK - 1) / (8 * opmm::TOPK_BLOCK);
  const int64_t cap = S > 1 ? 16 : h->num_sms;
  return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

// Shared tail of every fit enqueue: the launch(es), then for world > 1 the
// all-gather of the rank results (32 bytes each, 544 with top-K lists) and
// the merge kernel.
opmm_status launch_fit_and_merge(opmm_handle* h, const void* fn, opmm::FitArgs& a, int grid,
                                 int block, size_t smem, int64_t s_begin, int64_t S, bool multi,
                                 opmm_fit_result* out_dev) {
  CKS(record_start(h, h->stream));
  for (int64_t s0 = 0; s0 < S; s0 += 65535) {
    const int64_t sn = (S - s0) < 65535 ? (S - s0) : 65535;
    a.sac_begin = s_begin + s0;
    CK(opmm::launch_fit(fn, a, dim3(grid, (unsigned)sn), block, smem, h->stream));
  }
  if (a.topk) {   // exact top-K (+ certificate) from the errors the fit wrote
    a.sac_begin = s_begin;
    a.fit_grid = grid;
    const int tb = topk_blocks(h, a.end - a.begin, S);
    CK(opmm::launch_topk(a, tb, (int)S, opmm::topk_smem(tb), (int)a.metric_, h->stream));
    if (a.certify && !multi)
      CK(opmm::launch_cert(a, (int)S, opmm::cert_scratch_bytes(a.ctl.n_steps + 1), (int)a.metric_,
                           h->stream));
  }
  CKS(record_stop(h, h->stream));
  if (multi) {
    // the one exchange step per saccade
    NcclApi& api = nccl();
    const size_t bytes = a.topk ? sizeof(opmm::RankPartial) : sizeof(Partial);
    const int metric = (int)a.metric_;
    const size_t msmem = a.certify ? opmm::cert_scratch_bytes(a.ctl.n_steps + 1) : 0;
    for (int64_t s = 0; s < S; ++s) {
      ncclResult_t r = api.allGather(h->rank_part + s_begin + s, h->gathered, bytes, ncclUint8,
                                     h->comm, h->stream);
      if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
      CK(opmm::launch_merge(a, h->gathered, h->world, bytes, s_begin + s, out_dev + s, metric, msmem,
                            h->stream));
    }
  }
  return OPMM_OK;
}

// kernel_variant 4 (fit_super_kernel): the rank's share is a range of grid
// nodes (every level of the superposed dimension stays on one rank), so the
// union over ranks is still every candidate exactly once.
opmm_status enqueue_fit_super(opmm_handle* h, const double* rec_dev, const opmm_control* ctl,
                              const double* sacctl_dev, int64_t s_begin, int64_t S,
                              const opmm_search_space* space, const opmm::SpaceDev& space_dev,
                              int sup_dim, int64_t n_candidates, const opmm_fit_options* opts,
                              opmm_fit_result* out_dev, bool shard, FitLaunch* prepare_only) {
  const int metric = opts ? opts->metric : OPMM_METRIC_L1;
  const int32_t L = space->levels[sup_dim];
  int64_t st = 1;
  for (int d = 0; d < sup_dim; ++d) st *= space->levels[d] > 1 ? space->levels[d] : 1;
  const int64_t nodes = n_candidates / L;
  int64_t nb = 0, ne = nodes;
  if (shard) opmm_shard_range(nodes, h->rank, h->world, &nb, &ne);
  const int32_t ns = ctl->n_steps + 1;
  const int precision = opts ? opts->precision : OPMM_FP64;
  const bool f32 = precision == OPMM_FP32;   // fp32 columns and level loop (plain layout)
  const size_t lim = max_dyn_smem(opmm::fit_super_kernel_ptr(metric, false, f32));
  int32_t gt_n = 0;
  for (int d = 0; d < OPMM_NPARAM; ++d)
    if (d != sup_dim) gt_n += space->levels[d] > 1 ? space->levels[d] : 0;
  int32_t use_tab = 1;
  if (gt_n > opmm::SUPER_MAX_GT || opmm::super_smem(ns, L, gt_n, 1, 0, f32) > lim) {
    gt_n = 0;   // generic generator per node
    use_tab = 0;
  }
  // Warps per block: with n <= SUPER_TMEM_MAX_STEPS, 4 warps keep their
  // columns in their tensor-memory quadrant and as many more as shared memory
  // holds use shared memory, in ONE block per SM (8 warps, 2 per scheduler,
  // so one warp's latency-bound setup overlaps another's level loop).
  // Otherwise one warp per block, shared memory only (occupancy decides).
  int tm_warps = 0, smem_warps = 1;
  if (!f32 && ctl->n_steps <= opmm::SUPER_TMEM_MAX_STEPS && super_tmem_wanted(opts)) {
    // one block per SM: it may take all of the SM's shared memory
    const size_t lim_tm = max_dyn_smem_uncapped(opmm::fit_super_kernel_ptr(metric, true, false));
    size_t fixed = opmm::super_smem(ns, L, gt_n, 0, 4);
    int sw = 0;
    while (sw < opmm::SUPER_MAX_WARPS - 4 && opmm::super_smem(ns, L, gt_n, sw + 1, 4) <= lim_tm)
      ++sw;
    if (fixed <= lim_tm) { tm_warps = 4; smem_warps = sw; }
  }
  // tensor memory: every TMEM warp keeps 4 columns per sample in its lane
  // quadrant; the block allocates the next power of two >= 4 (n_steps + 4)
  // columns (the flushes write whole groups of 4 samples).  tcgen05.alloc
  // blocks while another block on the SM holds the columns, so the TMEM
  // layout is used only when shared memory provably limits the SM to ONE
  // block of this kernel (padding it if needed); otherwise the plain layout.
  int32_t tm_cols = 32;
  while (tm_cols < 4 * (ctl->n_steps + 4)) tm_cols *= 2;
  if (tm_warps > 0) {
    constexpr size_t kOneBlockSmem = 116 * 1024;   // 2 x (116 KB + static) > 228 KB per SM
    const void* tf = opmm::fit_super_kernel_ptr(metric, true, false);
    size_t sm = opmm::super_smem(ns, L, gt_n, smem_warps, tm_warps, f32);
    if (sm < kOneBlockSmem) sm = kOneBlockSmem;
    int per_sm = 0;
    if (tm_cols > 512 ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tf, 32 * (tm_warps + smem_warps), sm) !=
            cudaSuccess ||
        per_sm != 1) {
      cudaGetLastError();
      tm_warps = 0;   // fall back to the shared-memory layout
      smem_warps = 1;
    }
  }
  const void* fn = opmm::fit_super_kernel_ptr(metric, tm_warps > 0, f32);
  const int block = 32 * (tm_warps + smem_warps);
  size_t smem = opmm::super_smem(ns, L, gt_n, smem_warps, tm_warps, f32);
  if (tm_warps > 0 && smem < 116 * 1024) smem = 116 * 1024;
  int grid = 1;
  CKS(grid_for(h, fn, block, smem, ne - nb, opts ? opts->grid_blocks : 0, &grid));
  if (S > 1 && !(opts && opts->grid_blocks)) {
    const int64_t tiles = (ne - nb + block - 1) / block;
    grid = (int)(tiles < 65535 ? (tiles > 0 ? tiles : 1) : 65535);
  }
  if (ne <= nb) grid = 1;
  const bool multi = shard && h->comm != nullptr;
  CKS(ensure(h->partials, h->partials_cap, (size_t)grid * (size_t)(s_begin + S)));
  CKS(ensure(h->counters, h->counters_cap, (size_t)(s_begin + S), true));
  if (multi) {
    CKS(ensure(h->rank_part, h->rank_part_cap, (size_t)(s_begin + S)));
    CKS(ensure(h->gathered, h->gathered_cap, (size_t)h->world));
  }
  opmm::FitArgs a;
  std::memset(&a, 0, sizeof(a));
  a.metric_ = metric;
  a.rec = rec_dev;
  a.exp_tab = h->exp_tab;
  a.ctl = make_ctl(ctl);
  a.space = space_dev;
  a.amplitude = ctl->amplitude_deg;
  a.pw_default = ctl->pw_default_ms;
  a.sac_ctl = sacctl_dev;
  a.sac_begin = s_begin;
  a.begin = 0;                        // the epilogue's n_evaluated = end - begin
  a.end = (ne - nb) * (int64_t)L;
  a.err_out = opts ? opts->err_out : nullptr;
  a.err_ld = n_candidates;
  a.err_base = 0;
  a.partials = h->partials;
  a.counters = h->counters;
  a.rank_out = multi ? h->rank_part : nullptr;
  a.final_out = multi ? nullptr : out_dev;
  a.out_base = s_begin;
  a.sup_dim = sup_dim;
  a.sup_L = L;
  // chunk width: least padded slots over ceil(L / J) chunks, then the widest
  int best_J = 32;
  int64_t best_pad = INT64_MAX;
  for (int J = tm_warps > 0 ? 20 : 32; J >= 8; J -= 4) {
    const int64_t pad = ((int64_t)L + J - 1) / J * J - L;
    if (pad < best_pad) { best_pad = pad; best_J = J; }
  }
  a.sup_J = best_J;
  a.sup_gt_n = gt_n;
  a.sup_tab = use_tab;
  a.sup_tm_warps = tm_warps;
  a.sup_tm_cols = tm_cols;
  a.sup_st = st;
  a.node_begin = nb;
  a.node_end = ne;
  CKS(ensure(h->sup_next, h->sup_next_cap, (size_t)(s_begin + S), true));
  a.sup_next = h->sup_next;
  if (prepare_only && !multi && S == 1) {
    prepare_only->fn = fn;
    prepare_only->grid = grid;
    prepare_only->block = block;
    prepare_only->smem = smem;
    prepare_only->a = a;
    return OPMM_OK;
  }
  if (prepare_only) {   // not graph-eligible: nothing launched, the caller enqueues it plainly
    prepare_only->fn = nullptr;
    return OPMM_OK;
  }
  return launch_fit_and_merge(h, fn, a, grid, block, smem, s_begin, S, multi, out_dev);
}

opmm_status enqueue_fit(opmm_handle* h, const double* rec_dev, const opmm_control* ctl,
                        const double* sacctl_dev, int64_t s_begin, int64_t S,
                        const opmm_search_space* space, int64_t n_candidates,
                        const opmm_fit_options* opts, opmm_fit_result* out_dev, bool shard,
                        FitLaunch* prepare_only = nullptr) {
  const int precision = opts ? opts->precision : OPMM_FP64;
  const int metric = opts ? opts->metric : OPMM_METRIC_L1;
  const int integ = opts ? opts->integrator : OPMM_INTEG_PROPAGATOR;
  const int kv_opt = opts ? opts->kernel_variant : 0;
  const int top_k = opts ? opts->top_k : 0;
  if (!check_precision(precision)) return fail(OPMM_ERR_INVALID_ARG, "bad precision %d", precision);
  if (metric != 0 && metric != 1) return fail(OPMM_ERR_INVALID_ARG, "bad metric %d", metric);
  if (integ != 0 && integ != 1) return fail(OPMM_ERR_INVALID_ARG, "bad integrator %d", integ);
  if (kv_opt < 0 || kv_opt > 5) return fail(OPMM_ERR_INVALID_ARG, "kernel_variant must be 0..5");
  if (top_k < 0 || top_k > OPMM_MAX_TOPK)
    return fail(OPMM_ERR_INVALID_ARG, "top_k must be in [0, %d] (got %d)", OPMM_MAX_TOPK, top_k);
  if (opts && opts->err_out && !is_device_accessible(opts->err_out))
    return fail(OPMM_ERR_INVALID_ARG, "err_out must be device (or mapped) memory");
  // FP32 certification: the exact top-K by fp32 error (K = top_k, or 32),
  // re-scored in fp64 by the finishing block (or, world > 1, the merge kernel)
  const bool certify = opts && opts->certify && precision == OPMM_FP32;
  const int K = certify ? (top_k > 0 ? top_k : kCertifyK) : top_k;
  const opmm::SpaceDev space_dev = make_space(space);
  // variant 4: superposition over the grid levels of a pulse height (fp64
  // propagator, 18-parameter grid, physical space)
  int sup_dim = -1;
  if (space->mode == 1 && space->model == 0) {
    const int32_t la = space->levels[opmm::NSAC_AG], ln = space->levels[opmm::NSAC_ANT];
    if (la > 1 || ln > 1) sup_dim = la >= ln ? opmm::NSAC_AG : opmm::NSAC_ANT;
  }
  const bool sup_ok = sup_dim >= 0 && integ == OPMM_INTEG_PROPAGATOR &&
                      ctl->substeps <= 1 && space_dev.all_physical && !certify && K == 0 &&
                      !(opts && opts->block_size) && space->levels[sup_dim] <= opmm::SUPER_MAX_L &&
                      opmm::super_smem(ctl->n_steps + 1, space->levels[sup_dim], 0, 1, 0) <=
                          max_dyn_smem(opmm::fit_super_kernel_ptr(metric, false, false));
  if (kv_opt == 4 && !sup_ok)
    return fail(OPMM_ERR_UNSUPPORTED, "kernel_variant 4 needs a grid space (18-parameter model) "
                                      "with N_SAC_AG or N_SAC_ANT levels > 1 (<= %d), all "
                                      "candidates physical, the propagator, no substeps, "
                                      "no certify or top_k, the default block size and a trace "
                                      "that fits shared memory", opmm::SUPER_MAX_L);
  const bool superpose = kv_opt == 4 || (kv_opt == 0 && sup_ok && kAutoSuper &&
                                         space->levels[sup_dim] >= kSuperMinLevels);
  if (superpose)
    return enqueue_fit_super(h, rec_dev, ctl, sacctl_dev, s_begin, S, space, space_dev, sup_dim,
                             n_candidates, opts, out_dev, shard, prepare_only);
  // variants 2/3/5 need the propagator integrator and a search space whose
  // candidates are all physical (no per-candidate penalty path)
  const bool special_ok = integ == OPMM_INTEG_PROPAGATOR && space_dev.all_physical &&
                          !(opts && opts->block_size) && ctl->substeps <= 1;
  if (kv_opt >= 2 && !special_ok)
    return fail(OPMM_ERR_UNSUPPORTED, "kernel_variant %d needs the propagator integrator, a "
                                      "physical search space, the default block size and no "
                                      "substeps", kv_opt);
  const int kv = kv_opt == 0 ? (special_ok ? kAutoVariant : 1) : kv_opt;
  const bool two = kv == 2, three = kv == 3, refill = kv == 5;
  if ((two || three || refill) && K > 0)
    return fail(OPMM_ERR_UNSUPPORTED, "top_k / certify need kernel_variant 0 or 1");
  const int block = three ? opmm::FIT3_BLOCK : two ? opmm::FIT2_BLOCK
                        : ((opts && opts->block_size) ? opts->block_size : kDefaultBlock);
  CKS(check_block(block));
  int64_t b = 0, e = n_candidates;
  if (shard) opmm_shard_range(n_candidates, h->rank, h->world, &b, &e);
  const int32_t ns = ctl->n_steps + 1;
  size_t smem = three ? opmm::fit3_smem(precision, ns) : fit_smem(precision, ns, block, two ? 2 : 1);
  if (smem > kMaxDynSmem) return fail(OPMM_ERR_INVALID_ARG, "trace too long for shared memory");
  const bool one = !two && !three && !refill;
  // grid spaces: per-dimension level tables in shared memory (fit_kernel<GT>)
  // when they fit, the propagator integrates and the flag does not forbid it
  int64_t gt_n = 0;
  for (int d = 0; d < OPMM_NPARAM; ++d) gt_n += space->levels[d] > 1 ? space->levels[d] : 0;
  bool grid_tables = one && space->mode == 1 && kernel_integ(integ, ctl) == 0 &&
                     gt_n <= opmm::SUPER_MAX_GT &&
                     !(opts && (opts->flags & OPMM_FIT_FLAG_NO_GRID_TABLES));
  size_t gt_bytes = grid_tables ? (size_t)gt_n * sizeof(double) : 0;
  const void* fn = three ? opmm::fit3_kernel_ptr(precision, metric)
                   : two ? opmm::fit2_kernel_ptr(precision, metric)
                   : refill ? opmm::fit_refill_kernel_ptr(precision, metric)
                            : opmm::fit_kernel_ptr(precision, kernel_integ(integ, ctl), metric,
                                                   grid_tables);
  // fit_kernel dynamic shared memory: rel, exp table, stash (opmm_kernels.cu),
  // then the super-tile permutation and the pre-pass key/rank scratch
  // (aliased onto the stash when it fits there)
  const size_t perm_off = (smem + 15) & ~(size_t)15;
  const size_t stash_off = (precision == OPMM_FP64 ? opmm::rel_bytes<double>(ns)
                                                   : opmm::rel_bytes<float>(ns)) +
                           opmm::exp_tab_bytes();
  const size_t stash_sz = precision == OPMM_FP64 ? opmm::stash_bytes<double>(block)
                                                 : opmm::stash_bytes<float>(block);
  auto fit_dyn_nogt = [&](int64_t sup) {
    const size_t end = perm_off + opmm::perm_bytes(sup);
    return opmm::tmp_bytes(sup) <= stash_sz ? end : end + opmm::tmp_bytes(sup);
  };
  // the level tables (if any) follow, 8-byte aligned
  auto gt_at = [&](int64_t sup) { return (fit_dyn_nogt(sup) + 7) & ~(size_t)7; };
  auto fit_dyn = [&](int64_t sup) { return gt_at(sup) + gt_bytes; };
  // the tables must leave room for the smallest super-tile (very long
  // traces), else the generic grid generator
  if (grid_tables && fit_dyn(32) > max_dyn_smem(fn)) {
    grid_tables = false;
    gt_bytes = 0;
    fn = opmm::fit_kernel_ptr(precision, kernel_integ(integ, ctl), metric, false);
  }
  // largest super-tile the kernel's shared memory allows (long traces leave less room)
  int64_t super_cap = opmm::SUPER_MAX;
  if (one) {
    const size_t lim = max_dyn_smem(fn);
    while (super_cap > 32 && fit_dyn(super_cap) > lim) super_cap -= 32;
    smem = fit_dyn(super_cap);   // sized for occupancy at the cap
  }
  if (smem > kMaxDynSmem) return fail(OPMM_ERR_INVALID_ARG, "trace too long for shared memory");
  int grid = 1;
  // fit3 work unit per block pass: 8 consumer warps x 32 candidates
  const int64_t work = three ? (e - b + 255) / 256 * block : two ? (e - b + 1) / 2 : e - b;
  CKS(grid_for(h, fn, block, smem, work, opts ? opts->grid_blocks : 0, &grid));
  if (S > 1 && !(opts && opts->grid_blocks)) {
    // population batch: gridDim.y = saccades already fills the GPU, so each
    // block takes one slice of its saccade instead of a persistent stride --
    // one fit_kernel super-tile (<= SUPER_MAX candidates), one tile otherwise
    const int64_t unit = one ? super_cap : block;
    const int64_t tiles = (work + unit - 1) / unit;
    grid = (int)(tiles < 65535 ? (tiles > 0 ? tiles : 1) : 65535);
  }
  if (e <= b) grid = 1;  // empty shard: one block reports "no candidate"
  // fit_kernel super-tile: an equal share of the range per block, multiple of
  // 32, at most SUPER_MAX (larger ranges take several persistent passes)
  int64_t super = 32;
  if (one) {
    const int64_t share = (e - b + grid - 1) / (grid > 0 ? grid : 1);
    super = (share + 31) / 32 * 32;
    if (super < 32) super = 32;
    if (super > super_cap) super = super_cap;
    smem = fit_dyn(super);
  }
  const bool multi = shard && h->comm != nullptr;   // world > 1 (or a 1-rank communicator)
  CKS(ensure(h->partials, h->partials_cap, (size_t)grid * (size_t)(s_begin + S)));
  CKS(ensure(h->counters, h->counters_cap, (size_t)(s_begin + S), true));
  // top-K / certify: the fit writes every error (the caller's err_out, or a
  // handle workspace of 8 bytes per candidate of this rank), topk_kernel
  // selects from it
  double* err_buf = opts ? opts->err_out : nullptr;
  int64_t err_ld = n_candidates, err_base = 0;
  if (K > 0) {
    const int tb = topk_blocks(h, e - b, S);
    CKS(ensure(h->tk_e, h->tk_e_cap, (size_t)tb * (size_t)(s_begin + S) * opmm::TOPK));
    CKS(ensure(h->tk_i, h->tk_i_cap, (size_t)tb * (size_t)(s_begin + S) * opmm::TOPK));
    CKS(ensure(h->tk_counters, h->tk_counters_cap, 2 * (size_t)(s_begin + S), true));
    if (certify && opmm::cert_scratch_bytes(ns) > max_dyn_smem(opmm::cert_kernel_ptr(metric)))
      return fail(OPMM_ERR_INVALID_ARG, "trace too long for certify");
    if (!err_buf) {
      err_ld = e - b > 0 ? e - b : 1;
      err_base = b;
      CKS(ensure(h->tk_err, h->tk_err_cap, (size_t)err_ld * (size_t)(s_begin + S)));
      err_buf = h->tk_err;
    }
  }
  if (multi) {
    CKS(ensure(h->rank_part, h->rank_part_cap, (size_t)(s_begin + S)));
    CKS(ensure(h->gathered, h->gathered_cap, (size_t)h->world));
    if (certify && opmm::cert_scratch_bytes(ns) > max_dyn_smem(opmm::merge_kernel_ptr(metric)))
      return fail(OPMM_ERR_INVALID_ARG, "trace too long for certify");
  }
  opmm::FitArgs a;
  std::memset(&a, 0, sizeof(a));
  a.metric_ = metric;
  a.rec = rec_dev;
  a.exp_tab = h->exp_tab;
  a.ctl = make_ctl(ctl);
  a.space = space_dev;
  a.amplitude = ctl->amplitude_deg;
  a.pw_default = ctl->pw_default_ms;
  a.sac_ctl = sacctl_dev;
  a.sac_begin = s_begin;
  a.begin = b;
  a.end = e;
  a.err_out = err_buf;
  a.err_ld = err_ld;
  a.err_base = err_base;
  a.sort_lanes = (opts && (opts->flags & OPMM_FIT_FLAG_NO_LANE_SORT)) ? 0 : 1;
  a.super_tile = super;
  a.perm_off = (int64_t)perm_off;
  a.tmp_off = (int64_t)(opmm::tmp_bytes(super) <= stash_sz ? stash_off
                                                          : perm_off + opmm::perm_bytes(super));
  a.gt_off = grid_tables ? (int64_t)gt_at(super) : 0;
  a.topk = K;
  a.certify = certify ? 1 : 0;
  a.tk_e = h->tk_e;
  a.tk_i = h->tk_i;
  a.tk_counters = h->tk_counters;
  a.tk_fill_off = (int64_t)(h->tk_counters_cap / 2);
  a.partials = h->partials;
  a.counters = h->counters;
  a.rank_out = multi ? h->rank_part : nullptr;
  a.final_out = multi ? nullptr : out_dev;
  a.out_base = s_begin;
  if (prepare_only && !multi && S == 1 && K == 0) {   // the caller launches it (graph)
    prepare_only->fn = fn;
    prepare_only->grid = grid;
    prepare_only->block = block;
    prepare_only->smem = smem;
    prepare_only->a = a;
    return OPMM_OK;
  }
  if (prepare_only) {   // not graph-eligible: nothing launched, the caller enqueues it plainly
    prepare_only->fn = nullptr;
    return OPMM_OK;
  }
  return launch_fit_and_merge(h, fn, a, grid, block, smem, s_begin, S, multi, out_dev);
}

opmm_status stage_rec(opmm_handle* h, const double* recorded, size_t count, const double** dev) {
  if (is_device_ptr(recorded)) {
    *dev = recorded;
    return OPMM_OK;
  }
  for (size_t k = 0; k < count; ++k)
    if (!is_finite(recorded[k]))
      return fail(OPMM_ERR_INVALID_ARG, "recorded sample %zu is not finite", k);
  CKS(ensure(h->rec, h->rec_cap, count));
  CK(cudaMemcpyAsync(h->rec, recorded, count * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  *dev = h->rec;
  return OPMM_OK;
}

// Table 1 defaults; PW is the per-saccade placeholder
// "saccade duration - 6 ms", NaN here -> pw_default_ms.
const double kTable1Defaults[OPMM_NPARAM] = {2.5,  2.5, 1.2, 1.2,  0.046, 0.022, 0.06,
                                             0.8,  0.5, 0.000043, 11.7, 2.4, 2.0, 1.9,
                                             14.0, 55.0, 0.5, NAN};

struct NmConfig {
  int obj, precision, metric, max_iter, cpu_check, schedule;
  double tol_x, tol_f, init_scale, time_budget_ms;
};

// OPMM_NM_SCHEDULE_AUTO: the group schedule from this many problems on (one
// rank's share), the lock-step schedule below it.  Measured on one B200, n =
// 150 population, lock-step / lane / group (tools/time_nm_schedules.py,
// DESIGN.md section 8a): 256 problems 25 / 65 / 37 ms; 1024: 40 / 67 / 38 ms;
// 4096: 114 / 66 / 37 ms; 16384: 394 / 174 / 131 ms.
constexpr int64_t kNmGroupMinProblems = 1024;

opmm_status nm_config(const opmm_nm_options* o, int dim, bool plant, NmConfig* c) {
  c->obj = plant ? (o ? o->objective : OPMM_NM_OBJ_PROPAGATOR) : 3;
  c->precision = o ? o->precision : OPMM_FP64;
  c->metric = o ? o->metric : OPMM_METRIC_L1;
  c->max_iter = (o && o->max_iter > 0) ? o->max_iter : 200 * dim;
  c->tol_x = (o && o->tol_x > 0.0) ? o->tol_x : 1e-4;
  c->tol_f = (o && o->tol_f > 0.0) ? o->tol_f : 1e-4;
  c->init_scale = (o && o->init_scale != 0.0) ? o->init_scale : 0.05;
  c->cpu_check = o ? o->cpu_check : 1;
  c->schedule = o ? o->schedule : OPMM_NM_SCHEDULE_AUTO;
  c->time_budget_ms = o ? o->time_budget_ms : 0.0;
  if (!(c->time_budget_ms >= 0.0) || !is_finite(c->time_budget_ms))
    return fail(OPMM_ERR_INVALID_ARG, "time_budget_ms must be finite and >= 0");
  if (c->schedule < OPMM_NM_SCHEDULE_AUTO || c->schedule > OPMM_NM_SCHEDULE_GROUP)
    return fail(OPMM_ERR_INVALID_ARG, "bad NM schedule %d", c->schedule);
  if (plant && (c->obj < 0 || c->obj > 2)) return fail(OPMM_ERR_INVALID_ARG, "bad NM objective");
  if (!check_precision(c->precision)) return fail(OPMM_ERR_INVALID_ARG, "bad precision");
  if (c->metric != 0 && c->metric != 1) return fail(OPMM_ERR_INVALID_ARG, "bad metric");
  if (c->obj >= 2) c->precision = OPMM_FP64;
  if (o && o->max_iter < 0) return fail(OPMM_ERR_INVALID_ARG, "max_iter < 0");
  if (!(c->tol_x > 0.0) || !(c->tol_f > 0.0) || !is_finite(c->init_scale))
    return fail(OPMM_ERR_INVALID_ARG, "bad NM tolerances");
  return OPMM_OK;
}

opmm_status nm_launch(opmm_handle* h, const NmConfig& c, const double* rec_dev,
                      const double* sacctl_dev, const opmm_control* ctl0, int64_t x0_ld, int dim,
                      int fn_id, int64_t pb, int64_t pe) {
  const int32_t ns = ctl0 ? ctl0->n_steps + 1 : 1;
  // the propagator objective with substeps has its own instantiation (obj 4)
  const int obj = (c.obj == 0 && ctl0 && ctl0->substeps > 1) ? 4 : c.obj;
  const bool lane = c.schedule == OPMM_NM_SCHEDULE_LANE;
  const bool group = c.schedule == OPMM_NM_SCHEDULE_GROUP ||
                     (c.schedule == OPMM_NM_SCHEDULE_AUTO && pe - pb >= kNmGroupMinProblems);
  const int per = lane ? 32 : group ? opmm::nm_group_problems_per_block() : opmm::nm_problems_per_block();
  const int64_t n_blocks = (pe - pb + per - 1) / per;
  auto smem_for = [&](bool in_smem) {
    return lane ? opmm::nm_lane_smem(c.precision, obj, ns, in_smem)
           : group ? opmm::nm_group_smem(c.precision, obj, ns, in_smem)
                   : opmm::nm_smem(c.precision, obj, ns, in_smem);
  };
  auto kernel_for = [&](bool grel) {
    return lane ? opmm::nm_lane_kernel_ptr(c.precision, obj, c.metric, grel)
           : group ? opmm::nm_group_kernel_ptr(c.precision, obj, c.metric, grel)
                   : opmm::nm_kernel_ptr(c.precision, obj, c.metric, grel);
  };
  size_t smem = smem_for(true);
  // lane schedule with more warps than SMs: the trace goes to the global
  // workspace so that two warps fit per SM (the simplex alone is ~100 KB)
  const bool lane_waves = lane && n_blocks > h->num_sms;
  const bool rel_global = lane_waves || smem > max_dyn_smem(kernel_for(false));
  if (rel_global) {   // long traces: relativized per problem in global memory
    smem = smem_for(false);
    // lane / group schedules: [block][k][per] (interleaved), padded to whole blocks
    const int64_t slots = (lane || group) ? n_blocks * per : pe - pb;
    CKS(ensure(h->nm_rel, h->nm_rel_cap, (size_t)slots * (size_t)ns));
  }
  if (smem > kMaxDynSmem) return fail(OPMM_ERR_INVALID_ARG, "trace too long for the NM kernel");
  opmm::NmArgs a;
  std::memset(&a, 0, sizeof(a));
  a.rel_global = rel_global ? static_cast<void*>(h->nm_rel) : nullptr;
  a.rec = rec_dev;
  a.sac_ctl = sacctl_dev;
  if (ctl0) a.ctl = make_ctl(ctl0);
  a.x0 = h->nm_x0;
  a.x0_ld = x0_ld;
  a.x_best = h->nm_xbest;
  a.x_ld = OPMM_NPARAM;
  a.out = h->nm_out;
  a.prob_begin = pb;
  a.prob_end = pe;
  a.dim = dim;
  a.fn_id = fn_id;
  a.max_iter = c.max_iter;
  a.tol_x = c.tol_x;
  a.tol_f = c.tol_f;
  a.init_scale = c.init_scale;
  // (a positive budget below 1 ns still stops at the first check)
  a.time_budget_ns = c.time_budget_ms > 0.0
                         ? (unsigned long long)std::fmax(1.0, std::fmin(c.time_budget_ms * 1e6, 9e18))
                         : 0ull;
  int64_t grid = n_blocks;
  if (grid == 0) return OPMM_OK;
  if (grid > 0x7fffffff) return fail(OPMM_ERR_INVALID_ARG, "too many problems");
  if (group) {
    // more problems than one wave of resident blocks: launch one wave and let
    // finished groups take the next problem (nm_group_kernel's refill)
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel_for(rel_global), 32, smem));
    const int64_t wave = (int64_t)h->num_sms * (per_sm > 0 ? per_sm : 1);
    if (grid > wave) {
      grid = wave;
      CKS(ensure(h->nm_next, h->nm_next_cap, 1));
      const unsigned long long first = (unsigned long long)(pb + grid * per);
      CK(cudaMemcpyAsync(h->nm_next, &first, sizeof(first), cudaMemcpyHostToDevice, h->stream));
      CK(cudaStreamSynchronize(h->stream));   // `first` lives on this stack frame
      a.nm_next = h->nm_next;
    }
  }
  CKS(record_start(h, h->stream));
  if (lane || group)   // 32-thread blocks
    CK(opmm::launch_nm_lane(kernel_for(rel_global), a, (int)grid, smem, h->stream));
  else
    CK(opmm::launch_nm(kernel_for(rel_global), a, (int)grid, smem, h->stream));
  CKS(record_stop(h, h->stream));
  return OPMM_OK;
}

opmm_status nm_collect(opmm_handle* h, int64_t pb, int64_t pe, int dim, opmm_nm_result* out) {
  const int64_t S = pe;
  std::string xb((size_t)S * OPMM_NPARAM * sizeof(double), '\0');
  std::string ob((size_t)S * sizeof(opmm::NmOut), '\0');
  CK(cudaMemcpyAsync(&xb[0], h->nm_xbest, xb.size(), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaMemcpyAsync(&ob[0], h->nm_out, ob.size(), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  const double* xs = reinterpret_cast<const double*>(xb.data());
  const opmm::NmOut* os = reinterpret_cast<const opmm::NmOut*>(ob.data());
  for (int64_t s = pb; s < pe; ++s) {
    opmm_nm_result r;
    std::memset(&r, 0, sizeof(r));
    for (int d = 0; d < OPMM_NPARAM; ++d) r.x[d] = d < dim ? xs[s * OPMM_NPARAM + d] : NAN;
    r.f_best = os[s].f_best;
    r.cpu_check = NAN;
    r.iterations = os[s].iterations;
    r.func_evals = os[s].func_evals;
    r.gpu_evals = os[s].gpu_evals;
    r.exit_reason = os[s].exit_reason;
    out[s] = r;
  }
  return OPMM_OK;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
// The paper's CPU_check for a batch: one serial fp64 re-score per saccade,
// independent, so they run on the host's cores (up to 32 threads, shared
// among the ranks of an NCCL handle; the calling thread takes a share).
// Below `grain` saccades per thread it stays on the calling thread.
template <typename F>
void host_parallel_for(int64_t n, int world, F&& f, int64_t grain = 32) {
  const unsigned hw = std::thread::hardware_concurrency();
  int64_t T = hw ? (int64_t)hw / (world > 0 ? world : 1) : 1;
  if (T > 32) T = 32;
  if (T > n / grain) T = n / grain;
  if (T <= 1) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  auto run = [&](int64_t t) {
    for (int64_t i = n * t / T; i < n * (t + 1) / T; ++i) f(i);
  };
  std::vector<std::thread> th;
  th.reserve((size_t)(T - 1));
  for (int64_t t = 1; t < T; ++t) th.emplace_back(run, t);
  run(0);
  for (auto& x : th) x.join();
}

extern "C" {

const char* opmm_version(void) { return "libopmm 0.1.0 (sm_100a)"; }

const char* opmm_last_error(void) { return g_err.c_str(); }

opmm_status opmm_create(opmm_handle** out, int device) {
  if (!out) return fail(OPMM_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    return fail(OPMM_ERR_CUDA, "no CUDA device available (%s)",
                e == cudaSuccess ? "0 devices" : cudaGetErrorString(e));
  }
  if (device < 0 || device >= count)
    return fail(OPMM_ERR_INVALID_ARG, "device %d out of range [0, %d)", device, count);
  CK(cudaSetDevice(device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(OPMM_ERR_UNSUPPORTED, "libopmm is built for sm_100a; device is sm_%d%d", prop.major,
                prop.minor);
  opmm_handle* h = new opmm_handle();
  h->device = device;
  h->num_sms = prop.multiProcessorCount;
  opmm_status st = OPMM_OK;
  auto cleanup = [&]() { opmm_destroy(h); };
  if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&h->ev0) != cudaSuccess || cudaEventCreate(&h->ev1) != cudaSuccess) {
    st = fail(OPMM_ERR_CUDA, "stream/event creation failed");
    cleanup();
    return st;
  }
  // allow the largest traces: raise the dynamic shared-memory cap once
  for (int p = 0; p < 2; ++p)
    for (int i = 0; i < 3; ++i)
      for (int m = 0; m < 2; ++m) {
        allow_dyn_smem(opmm::fit_kernel_ptr(p, i, m));
        if (i == 0) allow_dyn_smem(opmm::fit_kernel_ptr(p, i, m, true));
        allow_dyn_smem(opmm::simscore_kernel_ptr(p, i, m));
        allow_dyn_smem(opmm::fit2_kernel_ptr(p, m));
        allow_dyn_smem(opmm::fit3_kernel_ptr(p, m));
        allow_dyn_smem(opmm::fit_refill_kernel_ptr(p, m));
        if (p == 0 && i == 0) {
          allow_dyn_smem(opmm::fit_super_kernel_ptr(m, false, false));
          allow_dyn_smem(opmm::fit_super_kernel_ptr(m, false, true));
          const void* f = opmm::fit_super_kernel_ptr(m, true, false);
          cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)max_dyn_smem_uncapped(f));
        }
        allow_dyn_smem(opmm::simulate_kernel_ptr(p, i));
        if (p == 0 && i == 0) {
          allow_dyn_smem(opmm::merge_kernel_ptr(m));
          allow_dyn_smem(opmm::topk_kernel_ptr(m));
          allow_dyn_smem(opmm::cert_kernel_ptr(m));
        }
        allow_dyn_smem(opmm::score_kernel_ptr(p, m));
        for (int obj = 0; obj < 5; ++obj)
          for (int g = 0; g < 2; ++g) {
            allow_dyn_smem(opmm::nm_kernel_ptr(p, obj, m, g == 1));
            allow_dyn_smem(opmm::nm_lane_kernel_ptr(p, obj, m, g == 1));
            allow_dyn_smem(opmm::nm_group_kernel_ptr(p, obj, m, g == 1));
          }
      }
  cudaGetLastError();
  {
    // exp(j/128), j < EXP_TAB_N, as double-double from 80-bit expl
    double2 tab[opmm::EXP_TAB_N];
    for (int j = 0; j < opmm::EXP_TAB_N; ++j) {
      const long double v = expl((long double)j / 128.0L);
      tab[j].x = (double)v;
      tab[j].y = (double)(v - (long double)tab[j].x);
    }
    if (cudaMalloc(&h->exp_tab, sizeof(tab)) != cudaSuccess ||
        cudaMemcpy(h->exp_tab, tab, sizeof(tab), cudaMemcpyHostToDevice) != cudaSuccess) {
      st = fail(OPMM_ERR_CUDA, "exp table allocation failed");
      cleanup();
      return st;
    }
  }
  if ((st = ensure(h->counters, h->counters_cap, 64, true)) != OPMM_OK ||
      (st = ensure(h->result, h->result_cap, 1)) != OPMM_OK ||
      (st = ensure_host(h->result_host, h->result_host_cap, 1)) != OPMM_OK) {
    cleanup();
    return st;
  }
  *out = h;
  return OPMM_OK;
}

opmm_status opmm_nccl_unique_id(uint8_t* id) {
  if (!id) return fail(OPMM_ERR_INVALID_ARG, "id is NULL");
  NcclApi& api = nccl();
  if (!api.loaded) return fail(OPMM_ERR_NCCL, "libnccl.so.2 could not be loaded");
  ncclUniqueId u;
  ncclResult_t r = api.getUniqueId(&u);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(id, u.internal, OPMM_NCCL_ID_BYTES);
  return OPMM_OK;
}

opmm_status opmm_create_nccl(opmm_handle** out, int device, const uint8_t* id, int rank, int world) {
  if (!id || world < 1 || rank < 0 || rank >= world)
    return fail(OPMM_ERR_INVALID_ARG, "bad NCCL arguments (rank %d, world %d)", rank, world);
  CKS(opmm_create(out, device));
  opmm_handle* h = *out;
  h->rank = rank;
  h->world = world;
  // world = 1 also gets a (one-rank) communicator: the caller asked for the
  // NCCL path, so the all-gather + merge runs for real on one GPU too.
  {
    NcclApi& api = nccl();
    if (!api.loaded) {
      opmm_destroy(h);
      *out = nullptr;
      return fail(OPMM_ERR_NCCL, "libnccl.so.2 could not be loaded");
    }
    ncclUniqueId u;
    std::memcpy(u.internal, id, OPMM_NCCL_ID_BYTES);
    ncclResult_t r = api.commInitRank(&h->comm, world, u, rank);
    if (r != ncclSuccess) {
      opmm_destroy(h);
      *out = nullptr;
      return nccl_fail(r, "ncclCommInitRank");
    }
  }
  return OPMM_OK;
}

opmm_status opmm_destroy(opmm_handle* h) {
  if (!h) return OPMM_OK;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  if (h->comm && nccl().loaded) nccl().commDestroy(h->comm);
  cudaFree(h->partials);
  cudaFree(h->counters);
  cudaFree(h->rec);
  cudaFree(h->sacctl);
  cudaFree(h->candctl);
  cudaFree(h->nm_rel);
  cudaFree(h->rank_part);
  cudaFree(h->gathered);
  cudaFree(h->tk_e);
  cudaFree(h->tk_i);
  cudaFree(h->tk_counters);
  cudaFree(h->tk_err);
  cudaFree(h->sup_next);
  for (int k = 0; k < 4; ++k) cudaFree(h->stage[k]);
  cudaFree(h->result);
  cudaFree(h->exp_tab);
  cudaFree(h->nm_x0);
  cudaFree(h->nm_xbest);
  cudaFree(h->nm_out);
  cudaFree(h->nm_next);
  if (h->result_host) cudaFreeHost(h->result_host);
  if (h->fit_graph) cudaGraphExecDestroy(h->fit_graph);
  if (h->rec_stage) cudaFreeHost(h->rec_stage);
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
  return OPMM_OK;
}

opmm_status opmm_get_stream(opmm_handle* h, void** stream) {
  CKS(check_handle(h));
  if (!stream) return fail(OPMM_ERR_INVALID_ARG, "stream is NULL");
  *stream = (void*)h->stream;
  return OPMM_OK;
}

opmm_status opmm_set_kernel_timing(opmm_handle* h, int32_t on) {
  CKS(check_handle(h));
  h->timing = on != 0;
  if (!h->timing) h->timed = false;
  return OPMM_OK;
}

opmm_status opmm_last_kernel_ms(opmm_handle* h, float* ms) {
  CKS(check_handle(h));
  if (!ms) return fail(OPMM_ERR_INVALID_ARG, "ms is NULL");
  if (!h->timed)
    return fail(OPMM_ERR_INVALID_ARG, "no timed launch: kernel timing is off (opmm_set_kernel_timing) "
                                      "or nothing was launched since it was turned on");
  CK(cudaEventSynchronize(h->ev1));
  CK(cudaEventElapsedTime(ms, h->ev0, h->ev1));
  return OPMM_OK;
}

opmm_status opmm_shard_range(int64_t n, int rank, int world, int64_t* begin, int64_t* end) {
  if (!begin || !end || n < 0 || world < 1 || rank < 0 || rank >= world)
    return fail(OPMM_ERR_INVALID_ARG, "bad shard arguments");
  // floor(r N / R) without overflow for N < 2^63
  const __int128 N = n;
  *begin = (int64_t)(N * rank / world);
  *end = (int64_t)(N * (rank + 1) / world);
  return OPMM_OK;
}

opmm_status opmm_merge_argmin(const double* err, const int64_t* idx, int count, double* best_err,
                              int64_t* best_idx) {
  if (!best_err || !best_idx || count < 0 || (count > 0 && (!err || !idx)))
    return fail(OPMM_ERR_INVALID_ARG, "bad merge arguments");
  double be = INFINITY;
  int64_t bi = -1;
  for (int r = 0; r < count; ++r) {
    if (idx[r] < 0 || !(err[r] < INFINITY)) continue;
    if (bi < 0 || err[r] < be || (err[r] == be && idx[r] < bi)) {
      be = err[r];
      bi = idx[r];
    }
  }
  *best_err = be;
  *best_idx = bi;
  return bi < 0 ? OPMM_ERR_NO_FINITE : OPMM_OK;
}

opmm_status opmm_merge_topk(const double* err, const int64_t* idx, int lists, int K,
                            double* out_err, int64_t* out_idx) {
  if (K < 1 || K > OPMM_MAX_TOPK || lists < 0 || !out_err || !out_idx ||
      (lists > 0 && (!err || !idx)))
    return fail(OPMM_ERR_INVALID_ARG, "bad merge_topk arguments");
  // K-way selection by repeated lexicographic minimum over the list heads
  // (the lists are sorted; index -1 ends a list)
  std::string ptr_buf((size_t)(lists > 0 ? lists : 1) * sizeof(int), '\0');
  int* ptr = reinterpret_cast<int*>(&ptr_buf[0]);
  for (int l = 0; l < lists; ++l) ptr[l] = 0;
  for (int k = 0; k < K; ++k) {
    int bl = -1;
    for (int l = 0; l < lists; ++l) {
      if (ptr[l] >= K) continue;
      const int64_t j = (int64_t)l * K + ptr[l];
      if (idx[j] < 0) continue;
      const int64_t bj = bl < 0 ? 0 : (int64_t)bl * K + ptr[bl];
      if (bl < 0 || err[j] < err[bj] || (err[j] == err[bj] && idx[j] < idx[bj])) bl = l;
    }
    if (bl < 0) {
      out_err[k] = INFINITY;
      out_idx[k] = -1;
      continue;
    }
    const int64_t j = (int64_t)bl * K + ptr[bl]++;
    out_err[k] = err[j];
    out_idx[k] = idx[j];
  }
  return OPMM_OK;
}

opmm_status opmm_certify_topk(const double* e32, const double* e64, const int64_t* idx, int K,
                              double scale, int32_t* certified, int64_t* best_index,
                              double* best_err) {
  if (K < 1 || K > OPMM_MAX_TOPK || !e32 || !e64 || !idx || !certified || !best_index || !best_err)
    return fail(OPMM_ERR_INVALID_ARG, "bad certify_topk arguments");
  // delta = 1e-4 max(E32[0], s), T* = E32[0] + 2 delta;
  // certified iff E32[K-1] > T* and every listed candidate's |E64 - E32| <= delta
  const bool have0 = idx[0] >= 0 && e32[0] < INFINITY;
  const double delta = 1e-4 * std::fmax(e32[0], scale);
  const double tstar = e32[0] + 2.0 * delta;
  const double eK = idx[K - 1] >= 0 ? e32[K - 1] : INFINITY;
  bool budget = true;
  double be = INFINITY;
  int64_t bi = -1;
  for (int k = 0; k < K; ++k) {
    if (idx[k] < 0 || !(e32[k] < INFINITY)) continue;
    budget = budget && std::fabs(e64[k] - e32[k]) <= delta;
    if (bi < 0 || e64[k] < be || (e64[k] == be && idx[k] < bi)) {
      be = e64[k];
      bi = idx[k];
    }
  }
  *certified = (have0 && eK > tstar && budget) ? 1 : 0;
  *best_index = bi;
  *best_err = be;
  return OPMM_OK;
}

opmm_status opmm_validate(const opmm_control* ctl, const opmm_search_space* space,
                          int64_t n_candidates) {
  if (n_candidates < 0) return fail(OPMM_ERR_INVALID_ARG, "n_candidates < 0");
  if (ctl) CKS(validate_control(ctl, false));
  if (space) CKS(validate_space(space, n_candidates));
  return OPMM_OK;
}

opmm_status opmm_generate(opmm_handle* h, const opmm_search_space* space, uint32_t saccade,
                          int64_t begin, int64_t count, double* opc_out, int64_t ld, void* stream) {
  CKS(check_handle(h));
  CKS(validate_space(space, -1));
  if (begin < 0 || count < 0 || ld < count || (count > 0 && !opc_out))
    return fail(OPMM_ERR_INVALID_ARG, "bad generate arguments");
  if (count == 0) return OPMM_OK;
  cudaStream_t st = stream ? (cudaStream_t)stream : h->stream;
  int grid = (int)((count + 255) / 256);
  if (grid > h->num_sms * 8) grid = h->num_sms * 8;
  Staging sg(h, st);
  double* out = nullptr;
  CKS(sg.out(opc_out, (size_t)(17 * ld + count) * sizeof(double), 0, &out));
  CK(opmm::launch_generate(make_space(space), saccade, begin, count, out, ld, h->exp_tab, grid, st));
  return sg.finish();
}

namespace {
opmm_status simulate_impl(opmm_handle* h, const double* opc, int64_t n, int64_t ld,
                          const opmm_control* ctl, const double* cand_ctl, int32_t precision,
                          int32_t integrator, void* traj, int64_t ld_out, uint8_t* status,
                          void* stream);
}

opmm_status opmm_simulate(opmm_handle* h, const double* opc, int64_t n, int64_t ld,
                          const opmm_control* ctl, int32_t precision, int32_t integrator, void* traj,
                          int64_t ld_out, uint8_t* status, void* stream) {
  CKS(check_handle(h));
  CKS(validate_control(ctl, true));
  return simulate_impl(h, opc, n, ld, ctl, nullptr, precision, integrator, traj, ld_out, status,
                       stream);
}

opmm_status opmm_simulate_batch(opmm_handle* h, const double* opc, int64_t n, int64_t ld,
                                const opmm_control* ctl, int32_t precision, int32_t integrator,
                                void* traj, int64_t ld_out, uint8_t* status, void* stream) {
  CKS(check_handle(h));
  if (n < 0) return fail(OPMM_ERR_INVALID_ARG, "n < 0");
  if (n == 0) return OPMM_OK;
  if (!ctl) return fail(OPMM_ERR_INVALID_ARG, "NULL ctl");
  std::string sc((size_t)n * 3 * sizeof(double), '\0');
  double* scp = reinterpret_cast<double*>(&sc[0]);
  for (int64_t i = 0; i < n; ++i) {
    CKS(validate_control(ctl + i, true));
    if (ctl[i].dt_ms != ctl[0].dt_ms || ctl[i].n_steps != ctl[0].n_steps ||
        ctl[i].substeps != ctl[0].substeps)
      return fail(OPMM_ERR_INVALID_ARG, "all candidates of a batch share dt_ms, n_steps and substeps");
    scp[3 * i] = ctl[i].amplitude_deg;
    scp[3 * i + 1] = ctl[i].theta0_deg;
    scp[3 * i + 2] = ctl[i].pw_default_ms;
  }
  cudaStream_t st = stream ? (cudaStream_t)stream : h->stream;
  CKS(ensure(h->candctl, h->candctl_cap, (size_t)n * 3));
  CK(cudaMemcpyAsync(h->candctl, scp, sc.size(), cudaMemcpyHostToDevice, st));
  return simulate_impl(h, opc, n, ld, ctl, h->candctl, precision, integrator, traj, ld_out, status,
                       stream);
}

namespace {
opmm_status simulate_impl(opmm_handle* h, const double* opc, int64_t n, int64_t ld,
                          const opmm_control* ctl, const double* cand_ctl, int32_t precision,
                          int32_t integrator, void* traj, int64_t ld_out, uint8_t* status,
                          void* stream) {
  if (!check_precision(precision)) return fail(OPMM_ERR_INVALID_ARG, "bad precision");
  if (integrator != 0 && integrator != 1) return fail(OPMM_ERR_INVALID_ARG, "bad integrator");
  if (n < 0 || ld < n || ld_out < n || (n > 0 && (!opc || !traj)))
    return fail(OPMM_ERR_INVALID_ARG, "bad simulate arguments");
  if (n == 0) return OPMM_OK;
  cudaStream_t st = stream ? (cudaStream_t)stream : h->stream;
  const int block = kDefaultBlock;
  const size_t smem = sim_smem(precision, 0, block, false);
  const void* fn = opmm::simulate_kernel_ptr(precision, kernel_integ(integrator, ctl));
  int grid = 1;
  CKS(grid_for(h, fn, block, smem, n, 0, &grid));
  const size_t esz = precision == OPMM_FP64 ? sizeof(double) : sizeof(float);
  Staging sg(h, st);
  CKS(sg.in(opc, (size_t)(17 * ld + n) * sizeof(double), 0, &opc));
  CKS(sg.out(traj, (size_t)((int64_t)ctl->n_steps * ld_out + n) * esz, 1, &traj));
  CKS(sg.out(status, (size_t)n, 2, &status));
  opmm::ExplicitArgs a;
  std::memset(&a, 0, sizeof(a));
  a.opc = opc;
  a.n = n;
  a.ld = ld;
  a.ctl = make_ctl(ctl);
  a.amplitude = ctl->amplitude_deg;
  a.pw_default = ctl->pw_default_ms;
  a.traj = traj;
  a.ld_out = ld_out;
  a.status = status;
  a.cand_ctl = cand_ctl;
  CKS(record_start(h, st));
  CK(opmm::launch_explicit(fn, a, dim3(grid), block, smem, st));
  CKS(record_stop(h, st));
  return sg.finish();
}
}

opmm_status opmm_score(opmm_handle* h, const void* traj, int64_t n, int64_t ld, int32_t n_samples,
                       const double* recorded, int32_t precision, int32_t metric, double* err,
                       void* stream) {
  CKS(check_handle(h));
  if (!check_precision(precision)) return fail(OPMM_ERR_INVALID_ARG, "bad precision");
  if (metric != 0 && metric != 1) return fail(OPMM_ERR_INVALID_ARG, "bad metric");
  if (n < 0 || ld < n || n_samples < 1 || n_samples > OPMM_MAX_STEPS + 1 ||
      (n > 0 && (!traj || !recorded || !err)))
    return fail(OPMM_ERR_INVALID_ARG, "bad score arguments");
  if (n == 0) return OPMM_OK;
  cudaStream_t st = stream ? (cudaStream_t)stream : h->stream;
  const int block = 256;
  const size_t smem = (size_t)n_samples * sizeof(double);
  int grid = 1;
  CKS(grid_for(h, opmm::score_kernel_ptr(precision, metric), block, smem, n, 0, &grid));
  const size_t esz = precision == OPMM_FP64 ? sizeof(double) : sizeof(float);
  Staging sg(h, st);
  CKS(sg.in(traj, (size_t)((int64_t)(n_samples - 1) * ld + n) * esz, 0, &traj));
  CKS(sg.in(recorded, (size_t)n_samples * sizeof(double), 1, &recorded));
  CKS(sg.out(err, (size_t)n * sizeof(double), 2, &err));
  opmm::ScoreArgs a{traj, n, ld, n_samples, recorded, err};
  CKS(record_start(h, st));
  CK(opmm::launch_score(a, precision, metric, dim3(grid), block, smem, st));
  CKS(record_stop(h, st));
  return sg.finish();
}

opmm_status opmm_simulate_score(opmm_handle* h, const double* opc, int64_t n, int64_t ld,
                                const opmm_control* ctl, const double* recorded, int32_t precision,
                                int32_t metric, int32_t integrator, double* err, void* stream) {
  CKS(check_handle(h));
  CKS(validate_control(ctl, false));
  if (!check_precision(precision)) return fail(OPMM_ERR_INVALID_ARG, "bad precision");
  if (metric != 0 && metric != 1) return fail(OPMM_ERR_INVALID_ARG, "bad metric");
  if (integrator != 0 && integrator != 1) return fail(OPMM_ERR_INVALID_ARG, "bad integrator");
  if (n < 0 || ld < n || (n > 0 && (!opc || !recorded || !err)))
    return fail(OPMM_ERR_INVALID_ARG, "bad simulate_score arguments");
  if (n == 0) return OPMM_OK;
  cudaStream_t st = stream ? (cudaStream_t)stream : h->stream;
  const int block = kDefaultBlock;
  const size_t smem = sim_smem(precision, ctl->n_steps + 1, block, true);
  if (smem > kMaxDynSmem) return fail(OPMM_ERR_INVALID_ARG, "trace too long for shared memory");
  const void* fn = opmm::simscore_kernel_ptr(precision, kernel_integ(integrator, ctl), metric);
  int grid = 1;
  CKS(grid_for(h, fn, block, smem, n, 0, &grid));
  const size_t ns = (size_t)ctl->n_steps + 1;
  if (!is_device_ptr(recorded))
    for (size_t k = 0; k < ns; ++k)
      if (!is_finite(recorded[k]))
        return fail(OPMM_ERR_INVALID_ARG, "recorded sample %zu is not finite", k);
  Staging sg(h, st);
  CKS(sg.in(opc, (size_t)(17 * ld + n) * sizeof(double), 0, &opc));
  CKS(sg.in(recorded, ns * sizeof(double), 1, &recorded));
  CKS(sg.out(err, (size_t)n * sizeof(double), 2, &err));
  opmm::ExplicitArgs a;
  std::memset(&a, 0, sizeof(a));
  a.opc = opc;
  a.n = n;
  a.ld = ld;
  a.ctl = make_ctl(ctl);
  a.amplitude = ctl->amplitude_deg;
  a.pw_default = ctl->pw_default_ms;
  a.rec = recorded;
  a.err = err;
  CKS(record_start(h, st));
  CK(opmm::launch_explicit(fn, a, dim3(grid), block, smem, st));
  CKS(record_stop(h, st));
  return sg.finish();
}

opmm_status opmm_fit_async(opmm_handle* h, const double* recorded_dev, const opmm_control* ctl,
                           const opmm_search_space* space, int64_t n_candidates,
                           const opmm_fit_options* opts, opmm_fit_result* out_dev) {
  CKS(check_handle(h));
  CKS(validate_control(ctl, false));
  if (n_candidates < 0) return fail(OPMM_ERR_INVALID_ARG, "n_candidates < 0");
  CKS(validate_space(space, n_candidates));
  if (!recorded_dev || !out_dev) return fail(OPMM_ERR_INVALID_ARG, "NULL recorded/out");
  if (!is_device_accessible(recorded_dev) || !is_device_accessible(out_dev))
    return fail(OPMM_ERR_INVALID_ARG, "opmm_fit_async takes device buffers (use opmm_fit for host ones)");
  return enqueue_fit(h, recorded_dev, ctl, nullptr, 0, 1, space, n_candidates, opts, out_dev, true);
}

opmm_status opmm_fit(opmm_handle* h, const double* recorded, const opmm_control* ctl,
                     const opmm_search_space* space, int64_t n_candidates,
                     const opmm_fit_options* opts, opmm_fit_result* out) {
  CKS(check_handle(h));
  CKS(validate_control(ctl, false));
  if (n_candidates < 0) return fail(OPMM_ERR_INVALID_ARG, "n_candidates < 0");
  CKS(validate_space(space, n_candidates));
  if (!recorded || !out) return fail(OPMM_ERR_INVALID_ARG, "NULL recorded/out");
  const size_t ns = (size_t)ctl->n_steps + 1;
  const double* rec_dev = nullptr;
  const bool host_rec = !is_device_ptr(recorded);
  // (host traces only: a device trace's pointer is part of the launch, and
  // callers that keep traces on the device use opmm_fit_async anyway)
  if (h->comm == nullptr && host_rec && !(opts && (opts->flags & OPMM_FIT_FLAG_NO_GRAPH))) {
    // Graph path: the trace is copied into pinned staging on the host, and
    // one graph launch does H2D + kernel, the kernel writing the result into
    // pinned host memory (re-captured when the launch changes).  The
    // previous call synchronised, so the staging is free.
    {
      for (size_t k = 0; k < ns; ++k)
        if (!is_finite(recorded[k]))
          return fail(OPMM_ERR_INVALID_ARG, "recorded sample %zu is not finite", k);
      if (ns > h->rec_stage_cap) {
        if (h->rec_stage) cudaFreeHost(h->rec_stage);
        h->rec_stage = nullptr;
        h->rec_stage_cap = 0;
        CK(cudaMallocHost(reinterpret_cast<void**>(&h->rec_stage), ns * sizeof(double)));
        h->rec_stage_cap = ns;
      }
      std::memcpy(h->rec_stage, recorded, ns * sizeof(double));
      CKS(ensure(h->rec, h->rec_cap, ns));
      rec_dev = h->rec;
    }
    FitLaunch L;
    CKS(enqueue_fit(h, rec_dev, ctl, nullptr, 0, 1, space, n_candidates, opts, h->result, true, &L));
    if (L.fn != nullptr) {
      // the key: every launch byte plus the host buffers the copies use
      // (they are reallocated when a larger request grows them)
      std::string key(sizeof(L.a) + 128, '\0');
      std::memcpy(&key[0], &L.a, sizeof(L.a));
      std::snprintf(&key[sizeof(L.a)], 128, "%p/%d/%d/%zu/%zu/%p/%p", L.fn, L.grid, L.block, L.smem,
                    ns, static_cast<void*>(h->rec_stage), static_cast<void*>(h->result_host));
      if (h->fit_graph == nullptr || key != h->fit_graph_key) {
        if (h->fit_graph) cudaGraphExecDestroy(h->fit_graph);
        h->fit_graph = nullptr;
        cudaGraph_t g = nullptr;
        CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
        cudaError_t ce = cudaSuccess;
        // (the kernel reading the trace from pinned host memory instead was
        // measured 13 us slower at 10^6 candidates: every block waits on PCIe)
        ce = cudaMemcpyAsync(h->rec, h->rec_stage, ns * sizeof(double), cudaMemcpyHostToDevice,
                             h->stream);
        // external event records: the timing events are real records at replay
        // the finishing block writes the 704-byte result straight into the
        // pinned host buffer (device-accessible at the same address under
        // UVA): no device-to-host copy node after the kernel
        opmm::FitArgs ga = L.a;
        ga.final_out = h->result_host;
        if (ce == cudaSuccess) ce = opmm::launch_fit(L.fn, ga, dim3(L.grid), L.block, L.smem, h->stream);
        const cudaError_t ee = cudaStreamEndCapture(h->stream, &g);
        CK(ce);
        CK(ee);
        const cudaError_t ie = cudaGraphInstantiate(&h->fit_graph, g, 0);
        cudaGraphDestroy(g);
        CK(ie);
        h->fit_graph_key = key;
      }
      // timing events bracket the graph (H2D + kernel) only when asked for
      CKS(record_start(h, h->stream));
      CK(cudaGraphLaunch(h->fit_graph, h->stream));
      CKS(record_stop(h, h->stream));
    } else {   // not graph-eligible (top-K / certify): this call's trace, then plain launches
      CK(cudaMemcpyAsync(h->rec, h->rec_stage, ns * sizeof(double), cudaMemcpyHostToDevice,
                         h->stream));
      CKS(enqueue_fit(h, rec_dev, ctl, nullptr, 0, 1, space, n_candidates, opts, h->result, true));
      CK(cudaMemcpyAsync(h->result_host, h->result, sizeof(opmm_fit_result),
                         cudaMemcpyDeviceToHost, h->stream));
    }
  } else {
    CKS(stage_rec(h, recorded, ns, &rec_dev));
    CKS(enqueue_fit(h, rec_dev, ctl, nullptr, 0, 1, space, n_candidates, opts, h->result, true));
    CK(cudaMemcpyAsync(h->result_host, h->result, sizeof(opmm_fit_result), cudaMemcpyDeviceToHost,
                       h->stream));
  }
  CK(cudaStreamSynchronize(h->stream));
  *out = *h->result_host;
  const bool want_check = !opts || opts->cpu_check;
  if (want_check && out->best_index >= 0) {
    // Fig. 4 CPU_check: serial fp64 re-score of the returned OPC on the host
    if (rec_dev == recorded) {
      std::string tmp(ns * sizeof(double), '\0');
      CK(cudaMemcpy(&tmp[0], recorded, ns * sizeof(double), cudaMemcpyDeviceToHost));
      out->cpu_check = opmm::cpu_check_score(out->opc, reinterpret_cast<const double*>(tmp.data()),
                                             ctl, opts ? opts->metric : 0);
    } else {
      out->cpu_check = opmm::cpu_check_score(out->opc, recorded, ctl, opts ? opts->metric : 0);
    }
  }
  if (out->best_index < 0) return fail(OPMM_ERR_NO_FINITE, "no candidate has a finite error");
  return OPMM_OK;
}

// One rank's share of a fit on a plain handle, for callers that bring their
// own launcher and merge on the host (opmm.h): the handle's rank/world
// select the shard for this call only; everything else is opmm_fit.
opmm_status opmm_fit_shard(opmm_handle* h, const double* recorded, const opmm_control* ctl,
                           const opmm_search_space* space, int64_t n_candidates, int rank,
                           int world, const opmm_fit_options* opts, opmm_fit_result* out) {
  CKS(check_handle(h));
  if (h->comm != nullptr)
    return fail(OPMM_ERR_INVALID_ARG, "opmm_fit_shard takes a plain handle (an NCCL handle shards itself)");
  if (world < 1 || rank < 0 || rank >= world)
    return fail(OPMM_ERR_INVALID_ARG, "rank %d / world %d", rank, world);
  opmm_fit_options o;
  if (opts) {
    o = *opts;
  } else {   // opmm_fit's defaults for a NULL opts
    std::memset(&o, 0, sizeof(o));
    o.cpu_check = 1;
  }
  o.flags |= OPMM_FIT_FLAG_NO_GRAPH;   // shards differ in their launch bytes
  const int r0 = h->rank, w0 = h->world;
  h->rank = rank;
  h->world = world;
  const opmm_status st = opmm_fit(h, recorded, ctl, space, n_candidates, &o, out);
  h->rank = r0;
  h->world = w0;
  return st;
}

opmm_status opmm_fit_batch(opmm_handle* h, const double* recorded, int64_t S,
                           const opmm_control* ctl, const opmm_search_space* space, int64_t n_per,
                           const opmm_fit_options* opts, opmm_fit_result* out) {
  CKS(check_handle(h));
  if (S < 0 || n_per < 0) return fail(OPMM_ERR_INVALID_ARG, "S and n_per must be >= 0");
  if (S == 0) return OPMM_OK;
  if (!recorded || !ctl || !out) return fail(OPMM_ERR_INVALID_ARG, "NULL argument");
  for (int64_t s = 0; s < S; ++s) {
    CKS(validate_control(ctl + s, false));
    if (ctl[s].dt_ms != ctl[0].dt_ms || ctl[s].n_steps != ctl[0].n_steps ||
        ctl[s].substeps != ctl[0].substeps)
      return fail(OPMM_ERR_INVALID_ARG, "all saccades of a batch share dt_ms, n_steps and substeps");
  }
  CKS(validate_space(space, n_per));
  // saccades are independent problems: rank r takes its contiguous share
  int64_t sb = 0, se = S;
  opmm_shard_range(S, h->rank, h->world, &sb, &se);
  const int64_t Sl = se - sb;
  if (Sl == 0) return OPMM_OK;
  const size_t ns = (size_t)ctl[0].n_steps + 1;
  const double* rec_dev = nullptr;
  if (is_device_ptr(recorded)) {
    rec_dev = recorded;
  } else {
    for (size_t k = 0; k < (size_t)S * ns; ++k)
      if (!is_finite(recorded[k])) return fail(OPMM_ERR_INVALID_ARG, "recorded sample not finite");
    CKS(ensure(h->rec, h->rec_cap, (size_t)S * ns));
    CK(cudaMemcpyAsync(h->rec, recorded, (size_t)S * ns * sizeof(double), cudaMemcpyHostToDevice,
                       h->stream));
    rec_dev = h->rec;
  }
  std::string sc((size_t)S * 2 * sizeof(double), '\0');
  double* scp = reinterpret_cast<double*>(&sc[0]);
  for (int64_t s = 0; s < S; ++s) {
    scp[2 * s] = ctl[s].amplitude_deg;
    scp[2 * s + 1] = ctl[s].pw_default_ms;
  }
  CKS(ensure(h->sacctl, h->sacctl_cap, (size_t)S * 2));
  CK(cudaMemcpyAsync(h->sacctl, scp, (size_t)S * 2 * sizeof(double), cudaMemcpyHostToDevice,
                     h->stream));
  CKS(ensure(h->result, h->result_cap, (size_t)Sl));
  CKS(ensure_host(h->result_host, h->result_host_cap, (size_t)Sl));
  // candidates are not sharded within a saccade here (shard = false)
  CKS(enqueue_fit(h, rec_dev, ctl, h->sacctl, sb, Sl, space, n_per, opts, h->result, false));
  CK(cudaMemcpyAsync(h->result_host, h->result, (size_t)Sl * sizeof(opmm_fit_result),
                     cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  const bool want_check = !opts || opts->cpu_check;
  std::string tmp;
  const double* rec_host = recorded;
  if (want_check && rec_dev == recorded) {
    tmp.resize((size_t)S * ns * sizeof(double));
    CK(cudaMemcpy(&tmp[0], recorded, (size_t)S * ns * sizeof(double), cudaMemcpyDeviceToHost));
    rec_host = reinterpret_cast<const double*>(tmp.data());
  }
  const int metric = opts ? opts->metric : 0;
  host_parallel_for(Sl, h->world, [&](int64_t j) {
    opmm_fit_result r = h->result_host[j];
    if (want_check && r.best_index >= 0)
      r.cpu_check = opmm::cpu_check_score(r.opc, rec_host + (size_t)(sb + j) * ns, ctl + sb + j, metric);
    out[sb + j] = r;
  });
  return OPMM_OK;
}

opmm_status opmm_estimate_batch(opmm_handle* h, const double* recorded, int64_t S,
                                const opmm_control* ctl, const double* x0,
                                const opmm_nm_options* opts, opmm_nm_result* out) {
  CKS(check_handle(h));
  if (S < 0) return fail(OPMM_ERR_INVALID_ARG, "S < 0");
  if (S == 0) return OPMM_OK;
  if (!recorded || !ctl || !out) return fail(OPMM_ERR_INVALID_ARG, "NULL argument");
  for (int64_t s = 0; s < S; ++s) {
    CKS(validate_control(ctl + s, false));
    if (ctl[s].dt_ms != ctl[0].dt_ms || ctl[s].n_steps != ctl[0].n_steps ||
        ctl[s].substeps != ctl[0].substeps)
      return fail(OPMM_ERR_INVALID_ARG, "all saccades of a batch share dt_ms, n_steps and substeps");
  }
  NmConfig c;
  CKS(nm_config(opts, OPMM_NPARAM, true, &c));
  double xs[OPMM_NPARAM];
  for (int d = 0; d < OPMM_NPARAM; ++d) {
    xs[d] = x0 ? x0[d] : kTable1Defaults[d];
    if (!is_finite(xs[d]) && !(d == OPMM_P_PW && std::isnan(xs[d])))
      return fail(OPMM_ERR_INVALID_ARG, "x0[%d] is not finite", d);
  }
  int64_t sb = 0, se = S;
  opmm_shard_range(S, h->rank, h->world, &sb, &se);
  const size_t ns = (size_t)ctl[0].n_steps + 1;
  const double* rec_dev = nullptr;
  if (is_device_ptr(recorded)) {
    rec_dev = recorded;
  } else {
    for (size_t k = 0; k < (size_t)S * ns; ++k)
      if (!is_finite(recorded[k])) return fail(OPMM_ERR_INVALID_ARG, "recorded sample not finite");
    CKS(ensure(h->rec, h->rec_cap, (size_t)S * ns));
    CK(cudaMemcpyAsync(h->rec, recorded, (size_t)S * ns * sizeof(double), cudaMemcpyHostToDevice,
                       h->stream));
    rec_dev = h->rec;
  }
  std::string sc((size_t)S * 2 * sizeof(double), '\0');
  double* scp = reinterpret_cast<double*>(&sc[0]);
  for (int64_t s = 0; s < S; ++s) {
    scp[2 * s] = ctl[s].amplitude_deg;
    scp[2 * s + 1] = ctl[s].pw_default_ms;
  }
  CKS(ensure(h->sacctl, h->sacctl_cap, (size_t)S * 2));
  CK(cudaMemcpyAsync(h->sacctl, scp, sc.size(), cudaMemcpyHostToDevice, h->stream));
  CKS(ensure(h->nm_x0, h->nm_x0_cap, OPMM_NPARAM));
  CK(cudaMemcpyAsync(h->nm_x0, xs, sizeof(xs), cudaMemcpyHostToDevice, h->stream));
  CKS(ensure(h->nm_xbest, h->nm_xbest_cap, (size_t)S * OPMM_NPARAM));
  CKS(ensure(h->nm_out, h->nm_out_cap, (size_t)S));
  CK(cudaStreamSynchronize(h->stream));   // host staging buffers above are temporaries
  CKS(nm_launch(h, c, rec_dev, h->sacctl, ctl, 0, OPMM_NPARAM, 0, sb, se));
  CKS(nm_collect(h, sb, se, OPMM_NPARAM, out));
  if (c.cpu_check) {
    std::string tmp;
    const double* rec_host = recorded;
    if (rec_dev == recorded) {
      tmp.resize((size_t)S * ns * sizeof(double));
      CK(cudaMemcpy(&tmp[0], recorded, tmp.size(), cudaMemcpyDeviceToHost));
      rec_host = reinterpret_cast<const double*>(tmp.data());
    }
    host_parallel_for(se - sb, h->world, [&](int64_t j) {
      const int64_t s = sb + j;
      out[s].cpu_check = opmm::cpu_check_score(out[s].x, rec_host + (size_t)s * ns, ctl + s, c.metric);
    });
  }
  return OPMM_OK;
}

opmm_status opmm_nm_minimize_test(opmm_handle* h, int32_t fn_id, int32_t dim, const double* x0,
                                  int64_t S, const opmm_nm_options* opts, opmm_nm_result* out) {
  CKS(check_handle(h));
  if (fn_id < 0 || fn_id > 2) return fail(OPMM_ERR_INVALID_ARG, "fn_id must be 0, 1 or 2");
  if (dim < 1 || dim > OPMM_NPARAM) return fail(OPMM_ERR_INVALID_ARG, "dim must be in [1, 18]");
  if (S < 0) return fail(OPMM_ERR_INVALID_ARG, "S < 0");
  if (S == 0) return OPMM_OK;
  if (!x0 || !out) return fail(OPMM_ERR_INVALID_ARG, "NULL argument");
  NmConfig c;
  CKS(nm_config(opts, dim, false, &c));
  CKS(ensure(h->nm_x0, h->nm_x0_cap, (size_t)S * dim));
  CK(cudaMemcpy(h->nm_x0, x0, (size_t)S * dim * sizeof(double), cudaMemcpyHostToDevice));
  CKS(ensure(h->nm_xbest, h->nm_xbest_cap, (size_t)S * OPMM_NPARAM));
  CKS(ensure(h->nm_out, h->nm_out_cap, (size_t)S));
  CKS(nm_launch(h, c, nullptr, nullptr, nullptr, dim, dim, fn_id, 0, S));
  return nm_collect(h, 0, S, dim, out);
}

}  // extern "C"
