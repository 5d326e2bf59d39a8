// fsmc.cu -- kernels and C-ABI entry points of libfsmc.so (see include/fsmc.h).
//
//   fsm_init_kernel      init_batch                     lockstep.py:175-206
//   fsm_run_kernel       run_fsm_batched tick loop      lockstep.py:308-406
//   lockstep_kernel      run_standard_batched           lockstep.py:238-305
//   prng_fill_kernel     prng.uniform/normal/_bits      prng.py:58-153
//   target_eval_kernel   TargetModel.log_density(_and_grad)
//
// Chains are independent (prng.py:84-94), so fsm_run_kernel gives every lane
// group a chain from a dynamic queue and runs it to completion with its
// state in registers: no barrier, no per-tick HBM round trip.  Only the
// lock-step baseline synchronises (a grid barrier per inner iteration).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <mutex>
#include <string>

#include "kernels.cuh"
#include "nvtx_range.h"

using namespace fsmc;

namespace {
thread_local std::string g_last_error;
fsmc_status fail(fsmc_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}
#define CUDA_TRY(expr)                                                               \
  do {                                                                               \
    cudaError_t e_ = (expr);                                                         \
    if (e_ != cudaSuccess)                                                           \
      return fail(FSMC_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// SM count of the current device (cached per device: a process may drive several)
constexpr int kMaxDevices = 64;
int num_sms() {
  static int sms[kMaxDevices] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) dev = 0;
  if (!sms[dev]) cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
  return sms[dev];
}

// Side streams of the overlapped windowed run, created once per device.  The
// launch bookkeeping (chain queues, barrier words) lives in each state
// block's own fsmc_state.work, so nothing else is shared between calls.
constexpr int kMaxParts = 16;   // windowed-run chain parts (work words 16 per part)
std::mutex g_side_mu;
cudaError_t side_streams(cudaStream_t (&out)[kMaxParts]) {
  static cudaStream_t side[kMaxDevices][kMaxParts] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  std::lock_guard<std::mutex> lk(g_side_mu);
  for (int h = 0; h < kMaxParts; h++) {   // [0]: the sample egress (device -> host) stream
    if (!side[dev][h]) {
      e = cudaStreamCreateWithFlags(&side[dev][h], cudaStreamNonBlocking);
      if (e != cudaSuccess) return e;
    }
    out[h] = side[dev][h];
  }
  return cudaSuccess;
}
}  // namespace

// --------------------------------------------------------------- utilities
__global__ void prng_fill_kernel(uint64_t seed, uint64_t stream, uint64_t counter, long long count,
                                 int kind, void* out) {
  uint64_t hsc = hash_seed_stream(seed, stream);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    uint64_t ctr = counter + (uint64_t)i;
    if (kind == 0)
      ((uint64_t*)out)[i] = bits(hsc, ctr);
    else if (kind == 1)
      ((double*)out)[i] = uniform(hsc, ctr);
    else
      ((double*)out)[i] = normal(hsc, ctr);
  }
}

template <int G, int E>
__global__ void __launch_bounds__(kThreads) target_eval_kernel(fsmc_target t, const double* X,
                                                               long long m, double* lp, double* grad) {
  extern __shared__ double smem[];
  Grp<G> grp;
  double* sm = group_scratch<G, E>(smem, group_doubles(t));
  const int d = t.dim;
  const long long groups = (long long)gridDim.x * (kThreads / G);
  for (long long j = (long long)blockIdx.x * (kThreads / G) + threadIdx.x / G; j < m; j += groups) {
    double x[E], g[E];
#pragma unroll
    for (int e = 0; e < E; e++) {
      int i = grp.idx(e);
      x[e] = i < d ? X[(size_t)j * d + i] : 0.0;
    }
    double v = grad ? target_eval<G, E, true>(t, x, g, sm, grp) : target_lp<G, E>(t, x, sm, grp);
    if (grp.lane == 0) lp[j] = v;
    if (grad) {
#pragma unroll
      for (int e = 0; e < E; e++) {
        int i = grp.idx(e);
        if (i < d) grad[(size_t)j * d + i] = g[e];
      }
    }
  }
}

// diagnostics: per-chain means and cross-chain summed autocovariances
// (analysis.py:344-352).  One block per (dim, lag tile).
__global__ void diag_mean_kernel(const double* S, long long n, long long m, long long d, long long burn,
                                 double* mean) {
  long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= m * d) return;
  long long j = idx / d, k = idx % d;
  double s = 0.0;
  for (long long i = burn; i < n; i++) s += S[((size_t)i * m + j) * d + k];
  mean[idx] = s / (double)(n - burn);
}

constexpr int kLagTile = 32;
// Thread per (chain, dim) series c_i = S[burn+i][j][k] - mean: lags
// lag0 .. lag0+31 of sum_i c_i c_{i+lag}, each series element read once.
// The lagged stream lives in a 32-entry register ring (indices fixed at
// compile time by unrolling the row loop 32-fold), so the kernel is one
// coalesced pass over the samples (rows of m*d consecutive doubles).  Sums
// over chains go through shared memory first (one global atomic per block
// and (lag, dim)); lag 0 of tile 0 also yields each chain's variance.
__global__ void __launch_bounds__(128) diag_acov_kernel(const double* __restrict__ S, long long n, long long m,
                                                        long long d, long long burn, long long lag0,
                                                        const double* __restrict__ mean, double* acov,
                                                        double* chain_var, long long cpt) {
  extern __shared__ double red[];   // [32][d] when d <= 128
  const bool smem_red = d <= 128;
  if (smem_red) {
    for (int i = threadIdx.x; i < kLagTile * d; i += blockDim.x) red[i] = 0.0;
    __syncthreads();
  }
  // cpt > 1 (wide targets, lag tiles past the first): a thread sums the lags
  // of chains jg, jg + mg, ... of its dimension k before its global atomics
  const long long mg = (m + cpt - 1) / cpt;
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool live = g < mg * d;
  const long long k = live ? g % d : 0;
  const long long N = n - burn;
  double acc[kLagTile];
#pragma unroll
  for (int t = 0; t < kLagTile; t++) acc[t] = 0.0;
  for (long long jj = live ? g / d : m; jj < m; jj += mg) {
    const long long idx = jj * d + k;
    const double mu = mean[idx];
    const size_t stride = (size_t)m * d;
    const double* col = S + (size_t)burn * stride + idx;
    auto b_at = [&](long long r) -> double {   // lagged stream c_{r + lag0}, 0 past the end
      long long rr = r + lag0;
      return rr < N ? __ldg(&col[(size_t)rr * stride]) - mu : 0.0;
    };
    double ring[kLagTile];
#pragma unroll
    for (int t = 0; t < kLagTile; t++) ring[t] = b_at(t);
    const long long imax = N - lag0;   // rows with at least one partner
    for (long long i0 = 0; i0 < imax; i0 += kLagTile) {
#pragma unroll
      for (int q = 0; q < kLagTile; q++) {
        const long long i = i0 + q;
        if (i < imax) {
          const double a = __ldg(&col[(size_t)i * stride]) - mu;
#pragma unroll
          for (int t = 0; t < kLagTile; t++) acc[t] = fma(a, ring[(q + t) & (kLagTile - 1)], acc[t]);
        }
        ring[q] = b_at(i + kLagTile);   // slot q now holds b_{i+32}
      }
    }
    if (lag0 == 0 && chain_var) chain_var[idx] = acc[0] / (double)N;   // cpt == 1 here
  }
  if (smem_red) {
    if (live) {
#pragma unroll
      for (int t = 0; t < kLagTile; t++) atomicAdd(&red[t * d + k], acc[t] / (double)N);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kLagTile * d; i += blockDim.x)
      if (lag0 + i / d < N) atomicAdd(&acov[i], red[i]);
  } else if (live) {
#pragma unroll
    for (int t = 0; t < kLagTile; t++)
      if (lag0 + t < N) atomicAdd(&acov[t * d + k], acc[t] / (double)N);
  }
}

// logistic-regression epilogue: one pass over Z [rows][N] (see fsmc.h)
constexpr int kEpiCols = 8192;
__global__ void __launch_bounds__(256) logreg_epilogue_kernel(const float* __restrict__ Z,
                                                              const float* __restrict__ y,
                                                              long long N, float* R, double* lp) {
  const long long r = blockIdx.y;
  const long long c0 = (long long)blockIdx.x * kEpiCols;
  const long long c1 = c0 + kEpiCols < N ? c0 + kEpiCols : N;
  const float* zr = Z + r * N;
  float* rr = R + r * N;
  double acc = 0.0;
  for (long long i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
    const float z = zr[i];
    const float yi = __ldg(&y[i]);
    const float e = expf(-fabsf(z));
    const float sp = fmaxf(z, 0.0f) + log1pf(e);           // log(1 + e^z), stable
    acc += (double)(yi * z - sp);
    const float sig = z >= 0.0f ? 1.0f / (1.0f + e) : e / (1.0f + e);
    rr[i] = yi - sig;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double part[8];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; w++) s += part[w];
    atomicAdd(&lp[r], s);
  }
}

// ================================================================ dispatch
namespace fsmc {
cudaError_t dispatch_drmh(int, int, int, Params&, const LaunchCtx&, cudaStream_t, uint64_t, long long,
                          const double*, double);
cudaError_t dispatch_ess(int, int, int, Params&, const LaunchCtx&, cudaStream_t, uint64_t, long long,
                         const double*, double);
cudaError_t dispatch_nuts(int, int, int, Params&, const LaunchCtx&, cudaStream_t, uint64_t, long long,
                          const double*, double);
cudaError_t dispatch_slice(int, int, int, Params&, const LaunchCtx&, cudaStream_t, uint64_t, long long,
                           const double*, double);
}  // namespace fsmc

namespace {

struct GE {
  int g, e;
};

// smallest compiled E for the requested lanes (auto: thread-per-chain for
// small d, a warp per chain beyond)
// the per-chain GP plugin keeps two n x n matrices per chain in shared
// memory (4 chains per block); larger designs use the batched evaluator
constexpr int kGpMaxRows = 56;

bool pick_config(int family, int dim, int lanes, GE& out, int kind = 0) {
  static const GE drmh[] = {
#define X(GG, EE) {GG, EE},
      FSMC_DRMH_CONFIGS(X)};
  static const GE ess[] = {FSMC_ESS_CONFIGS(X)};
  static const GE nuts[] = {FSMC_NUTS_CONFIGS(X)};
  static const GE slice[] = {FSMC_SLICE_CONFIGS(X)};
#undef X
  if (family == FSMC_SLICE) {
    if (dim != 1 || (lanes > 1)) return false;
    out = slice[0];
    return true;
  }
  const GE* list = family == FSMC_DRMH ? drmh : family == FSMC_ESS ? ess : nuts;
  int cnt = family == FSMC_DRMH ? (int)(sizeof(drmh) / sizeof(GE))
            : family == FSMC_ESS ? (int)(sizeof(ess) / sizeof(GE))
                                 : (int)(sizeof(nuts) / sizeof(GE));
  if (lanes <= 0) {
    if (kind == FSMC_T_GP_HYPER) lanes = 32;   // a warp factors the chain's kernel matrix
    else if (family == FSMC_DRMH && dim <= 16) lanes = 1;
    else if (dim <= 4) lanes = 1;
    else if (family == FSMC_NUTS && dim <= 16) lanes = 4;
    else if (family == FSMC_ESS && dim > 256) lanes = 128;
    else if (family == FSMC_NUTS && dim > 128) lanes = 128;
    else lanes = 32;
  }
  const GE* best = nullptr;
  for (int i = 0; i < cnt; i++) {
    const GE& c = list[i];
    if (c.g != lanes || c.g * c.e < dim) continue;
    if (!best || c.e < best->e) best = &c;
  }
  if (!best && lanes == 1) return pick_config(family, dim, family == FSMC_NUTS && dim <= 16 ? 4 : 32, out, kind);
  if (!best) return false;
  out = *best;
  return true;
}

int n_states(const fsmc_kernel* k) {
  if (k->family == FSMC_NUTS || k->family == FSMC_SLICE) return 5;
  return k->family == FSMC_DRMH && k->split_body ? 6 : 3;
}

LaunchCtx launch_ctx() {
  LaunchCtx lc;
  lc.num_sms = num_sms();
  return lc;
}

cudaError_t dispatch_family(int op, const GE& ge, Params& p, cudaStream_t s, uint64_t ps = 0,
                            long long off = 0, const double* x0 = nullptr, double jit = 0.0) {
  LaunchCtx lc = launch_ctx();
  switch (p.k.family) {
    case FSMC_DRMH: return dispatch_drmh(op, ge.g, ge.e, p, lc, s, ps, off, x0, jit);
    case FSMC_ESS: return dispatch_ess(op, ge.g, ge.e, p, lc, s, ps, off, x0, jit);
    case FSMC_SLICE: return dispatch_slice(op, ge.g, ge.e, p, lc, s, ps, off, x0, jit);
    default: return dispatch_nuts(op, ge.g, ge.e, p, lc, s, ps, off, x0, jit);
  }
}

fsmc_status check_args(const fsmc_kernel* k, const fsmc_target* t, const fsmc_state* st) {
  if (!k || !t || !st) return fail(FSMC_ERR_ARG, "null argument");
  if (k->family < FSMC_DRMH || k->family > FSMC_SLICE) return fail(FSMC_ERR_ARG, "unknown kernel family");
  if (t->dim < 1) return fail(FSMC_ERR_ARG, "dim must be >= 1");
  if (st->dim != t->dim) return fail(FSMC_ERR_ARG, "state dim does not match target dim");
  if (!st->work || !st->err_key) return fail(FSMC_ERR_ARG, "state needs err_key[1] and work[FSMC_WORK_WORDS]");
  if (st->m < 1 || st->m >= (1LL << 24)) return fail(FSMC_ERR_ARG, "m must be in [1, 2^24) per state block");
  if (k->family == FSMC_DRMH && (k->max_tries < 1 || !(k->proposal_scale > 0)))
    return fail(FSMC_ERR_ARG, "invalid drmh parameters");
  if (k->family == FSMC_NUTS && (k->max_depth < 1 || k->max_depth > 40 || !(k->step_size > 0)))
    return fail(FSMC_ERR_ARG, "invalid nuts parameters");
  if (k->family == FSMC_SLICE && (!(k->slice_width > 0) || k->max_expansions < 0))
    return fail(FSMC_ERR_ARG, "invalid slice parameters");
  if (k->family == FSMC_SLICE && t->dim != 1)
    return fail(FSMC_ERR_ARG, "slice sampling here is univariate");
  if (k->family == FSMC_ESS && t->prior_kind == FSMC_PRIOR_NONE)
    return fail(FSMC_ERR_ARG, "elliptical slice sampling needs a Gaussian-prior split");
  // scratch == 0: no per-chain plugin (more than kGpMaxRows observations), the
  // evaluations come from a batched evaluator (the plugin reports a TargetError)
  if (t->kind == FSMC_T_GP_HYPER &&
      (t->dim != 3 || t->n_rows < 2 || !t->data || !t->yvec ||
       (t->scratch != 0 && (t->n_rows > kGpMaxRows ||
                            t->scratch < 2 * t->n_rows * t->n_rows + 2 * t->n_rows + 4))))
    return fail(FSMC_ERR_ARG, "GP target: dim 3, n >= 2 observations; the per-chain plugin needs "
                              "n <= 56 and scratch 2n^2+2n+4 (scratch 0: batched evaluator only)");
  if (t->kind == FSMC_T_MOG && (t->n_modes < 1 || t->n_modes > FSMC_MAX_MODES))
    return fail(FSMC_ERR_ARG, "n_modes out of range");
  if (k->precision != 0 && k->precision != 1) return fail(FSMC_ERR_ARG, "precision must be 0 (fp64) or 1 (fp32)");
  return FSMC_OK;
}

// the fp32 throughput mode's compiled (family, lanes, elements, plugin) set
bool f32_compiled(const fsmc_kernel* k, const fsmc_target* t, const GE& ge) {
  bool ok = false;
#define D(GG, EE, TK) ok = ok || (k->family == FSMC_DRMH && !k->split_body && ge.g == GG && ge.e == EE && t->kind == TK && \
                                   (TK != FSMC_T_MOG || t->n_modes <= FSMC_MOG_SPECIAL_MODES));
  FSMC_DRMH_F32(D)
#undef D
#define N(GG, EE, TK) ok = ok || (k->family == FSMC_NUTS && ge.g == GG && ge.e == EE && t->kind == TK);
  FSMC_NUTS_F32(N)
#undef N
  return ok;
}
fsmc_status check_f32(const fsmc_kernel* k, const fsmc_target* t, const GE& ge) {
  if (k->precision == 1 && !f32_compiled(k, t, ge))
    return fail(FSMC_ERR_UNSUPPORTED, "the fp32 throughput mode is compiled for DRMH on the MoG / funnel "
                                      "(d <= 10, one lane per chain) and NUTS on the equicorrelated "
                                      "Gaussian (d <= 128, a warp per chain)");
  return FSMC_OK;
}

}  // namespace

// ================================================================== C ABI
extern "C" {

int32_t fsmc_abi_version(void) { return FSMC_ABI_VERSION; }

int64_t fsmc_launch_count(void) { return fsmc::launch_counter().load(); }
const char* fsmc_last_error(void) { return g_last_error.c_str(); }

fsmc_status fsmc_state_layout(const fsmc_kernel* k, int64_t dim, int32_t* n_vec, int32_t* n_scal,
                              int32_t* n_loop, int32_t* n_states) {
  if (!k) return fail(FSMC_ERR_ARG, "null kernel");
  switch (k->family) {
    case FSMC_DRMH:
      if (k->split_body) { *n_vec = 3; *n_scal = 4; *n_loop = 4; *n_states = 6; }
      else { *n_vec = 2; *n_scal = 3; *n_loop = 1; *n_states = 3; }
      break;
    case FSMC_ESS: *n_vec = 3; *n_scal = 6; *n_loop = 1; *n_states = 3; break;
    case FSMC_SLICE: *n_vec = 2; *n_scal = 8; *n_loop = 2; *n_states = 5; break;
    case FSMC_NUTS:
      *n_vec = 12 + 2 * k->max_depth; *n_scal = 3; *n_loop = 3; *n_states = 5;
      break;
    default: return fail(FSMC_ERR_ARG, "unknown kernel family");
  }
  (void)dim;
  return FSMC_OK;
}

fsmc_status fsmc_prng_fill(uint64_t seed, uint64_t stream, uint64_t counter, int64_t count, int32_t kind,
                           void* out, void* stream_) {
  FSMC_NVTX("fsmc_prng_fill");
  if (count < 0 || kind < 0 || kind > 2 || (!out && count)) return fail(FSMC_ERR_ARG, "bad prng_fill args");
  if (!count) return FSMC_OK;
  int blocks = (int)std::min<long long>((count + 255) / 256, 148LL * 16);
  fsmc::count_launch();
  prng_fill_kernel<<<blocks, 256, 0, (cudaStream_t)stream_>>>(seed, stream, counter, count, kind, out);
  CUDA_TRY(cudaGetLastError());
  return FSMC_OK;
}

static fsmc_status init_common(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st,
                               uint64_t parent_stream, int64_t chain_offset, const double* x0,
                               double init_jitter, void* stream_, bool defer) {
  fsmc_status s = check_args(k, t, st);
  if (s != FSMC_OK) return s;
  GE ge;
  if (!pick_config(k->family, t->dim, 0, ge, t->kind)) return fail(FSMC_ERR_UNSUPPORTED, "dimension not supported");
  Params p;
  memset(&p, 0, sizeof(p));
  p.k = *k; p.t = *t; p.st = *st;
  p.t.full = k->family != FSMC_ESS;
  p.b_defer = defer;
  cudaStream_t cs = (cudaStream_t)stream_;
  CUDA_TRY(cudaMemsetAsync(st->err_key, 0xff, sizeof(unsigned long long), cs));
  CUDA_TRY(dispatch_family(0, ge, p, cs, parent_stream, chain_offset, x0, init_jitter));
  return FSMC_OK;
}

fsmc_status fsmc_init(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st, uint64_t parent_stream,
                      int64_t chain_offset, const double* x0, double init_jitter, void* stream_) {
  FSMC_NVTX("fsmc_init");
  return init_common(k, t, st, parent_stream, chain_offset, x0, init_jitter, stream_, false);
}

fsmc_status fsmc_init_deferred(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st,
                               uint64_t parent_stream, int64_t chain_offset, const double* x0,
                               double init_jitter, void* stream_) {
  FSMC_NVTX("fsmc_init_deferred");
  return init_common(k, t, st, parent_stream, chain_offset, x0, init_jitter, stream_, true);
}

fsmc_status fsmc_init_finish(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st, const double* lp,
                             void* stream_) {
  FSMC_NVTX("fsmc_init_finish");
  fsmc_status s = check_args(k, t, st);
  if (s != FSMC_OK) return s;
  if (!lp) return fail(FSMC_ERR_ARG, "init_finish needs lp [m]");
  GE ge;
  if (!pick_config(k->family, t->dim, 0, ge, t->kind)) return fail(FSMC_ERR_UNSUPPORTED, "dimension not supported");
  Params p;
  memset(&p, 0, sizeof(p));
  p.k = *k; p.t = *t; p.st = *st;
  p.t.full = k->family != FSMC_ESS;
  p.b_init_lp = lp;
  CUDA_TRY(dispatch_family(8, ge, p, (cudaStream_t)stream_));
  return FSMC_OK;
}

fsmc_status fsmc_run(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st, int64_t n, int32_t variant,
                     const int32_t* order, int64_t tick_limit, int32_t mode, const fsmc_outputs* out,
                     int32_t lanes, void* stream_) {
  FSMC_NVTX("fsmc_run");
  return fsmc_run_egress(k, t, st, n, variant, order, tick_limit, mode, out, lanes, 1, nullptr, stream_);
}

fsmc_status fsmc_run_egress(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st, int64_t n,
                            int32_t variant, const int32_t* order, int64_t tick_limit, int32_t mode,
                            const fsmc_outputs* out, int32_t lanes, int32_t parts, const fsmc_egress* eg,
                            void* stream_) {
  FSMC_NVTX("fsmc_run_egress");
  fsmc_status s = check_args(k, t, st);
  if (s != FSMC_OK) return s;
  if (n < 0) return fail(FSMC_ERR_ARG, "n must be >= 0");
  if (variant < FSMC_PLAIN || variant > FSMC_AMORTIZED) return fail(FSMC_ERR_ARG, "bad step variant");
  GE ge;
  if (!pick_config(k->family, t->dim, lanes, ge, t->kind))
    return fail(FSMC_ERR_UNSUPPORTED, "no compiled (lanes, elements) configuration for this dimension");
  if ((s = check_f32(k, t, ge)) != FSMC_OK) return s;
  Params p;
  memset(&p, 0, sizeof(p));
  p.k = *k; p.t = *t; p.st = *st;
  p.t.full = k->family != FSMC_ESS;
  if (out) p.out = *out;
  p.n = n;
  p.tick_limit = tick_limit;
  p.variant = variant;
  p.mode = mode;
  int K = n_states(k);
  p.default_order = 1;
  for (int i = 0; i < K; i++) {
    p.order[i] = order ? order[i] : (i == 0 ? K : i);
    if (p.order[i] != (i == 0 ? K : i)) p.default_order = 0;
  }
  cudaStream_t cs = (cudaStream_t)stream_;
  p.j_lo = 0;
  p.j_hi = st->m;
  const bool any_egress = eg && out && n > 0 &&
                          ((eg->samples && out->samples) || (out->loop_counts64 && (eg->loop_counts || eg->iter_counts)));
  // the [lo, hi) chain columns of rows [0, n) of every output to the host
  auto send_cols = [&](long long lo, long long hi, cudaStream_t es) -> cudaError_t {
    cudaError_t e = cudaSuccess;
    if (eg->samples && out->samples) {
      const size_t row = (size_t)st->m * t->dim * sizeof(double), off = (size_t)lo * t->dim * sizeof(double);
      e = cudaMemcpy2DAsync((char*)eg->samples + off, row, (const char*)out->samples + off, row,
                            (size_t)(hi - lo) * t->dim * sizeof(double), (size_t)n, cudaMemcpyDeviceToHost, es);
    }
    if (e == cudaSuccess && out->loop_counts64) {
      const size_t row = (size_t)st->m * sizeof(int64_t), off = (size_t)lo * sizeof(int64_t);
      const size_t w = (size_t)(hi - lo) * sizeof(int64_t);
      for (int l = 0; e == cudaSuccess && eg->loop_counts && l < eg->n_loops; l++)
        e = cudaMemcpy2DAsync((char*)(eg->loop_counts + (size_t)l * n * st->m) + off, row,
                              (const char*)(out->loop_counts64 + (size_t)l * n * st->m) + off, row, w, (size_t)n,
                              cudaMemcpyDeviceToHost, es);
      if (e == cudaSuccess && eg->iter_counts)
        e = cudaMemcpy2DAsync((char*)eg->iter_counts + off, row,
                              (const char*)(out->loop_counts64 + (size_t)eg->iter_loop * n * st->m) + off, row, w,
                              (size_t)n, cudaMemcpyDeviceToHost, es);
    }
    return e;
  };
  if (!any_egress || parts <= 1 || st->m < 2 * parts) {
    p.next_chain = st->work;
    CUDA_TRY(cudaMemsetAsync(p.next_chain, 0, sizeof(unsigned), cs));
    CUDA_TRY(dispatch_family(1, ge, p, cs));
    if (any_egress) CUDA_TRY(send_cols(0, st->m, cs));
    return FSMC_OK;
  }
  // chains in `parts` contiguous parts launched back to back on two alternating
  // streams (a part's blocks backfill the SMs the previous part's tail frees);
  // each finished part's sample columns go to the host on the egress stream
  // (one pitched copy: n rows of its chains) while later parts still run
  if (parts > kMaxParts) parts = kMaxParts;
  cudaStream_t side[kMaxParts] = {};
  CUDA_TRY(side_streams(side));
  cudaStream_t comp[2] = {cs, side[1]};
  cudaEvent_t ev_fork, ev_part[kMaxParts], ev_done;
  CUDA_TRY(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming));
  for (int h = 0; h < parts; h++) CUDA_TRY(cudaEventCreateWithFlags(&ev_part[h], cudaEventDisableTiming));
  CUDA_TRY(cudaEventRecord(ev_fork, cs));
  CUDA_TRY(cudaStreamWaitEvent(side[1], ev_fork, 0));
  CUDA_TRY(cudaStreamWaitEvent(side[0], ev_fork, 0));
  for (int h = 0; h < parts; h++) {
    Params ph = p;
    ph.j_lo = st->m * h / parts;
    ph.j_hi = st->m * (h + 1) / parts;
    ph.next_chain = st->work + 16 * h;
    cudaStream_t sh = comp[h & 1];
    CUDA_TRY(cudaMemsetAsync(ph.next_chain, 0, sizeof(unsigned), sh));
    CUDA_TRY(dispatch_family(1, ge, ph, sh));
    CUDA_TRY(cudaEventRecord(ev_part[h], sh));
    CUDA_TRY(cudaStreamWaitEvent(side[0], ev_part[h], 0));
    CUDA_TRY(send_cols(ph.j_lo, ph.j_hi, side[0]));
  }
  CUDA_TRY(cudaEventRecord(ev_done, side[0]));
  CUDA_TRY(cudaStreamWaitEvent(cs, ev_done, 0));   // the egress waited on every part
  CUDA_TRY(cudaEventDestroy(ev_fork));
  CUDA_TRY(cudaEventDestroy(ev_done));
  for (int h = 0; h < parts; h++) CUDA_TRY(cudaEventDestroy(ev_part[h]));
  return FSMC_OK;
}

static fsmc_status advance_common(int op, const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st,
                                  int64_t n, int32_t variant, const int32_t* order, int64_t tick_limit,
                                  int32_t mode, const fsmc_outputs* out, const double* lp,
                                  const double* grad, double* theta, int32_t* req_chain,
                                  int32_t* req_count, int32_t lanes, void* stream_,
                                  int64_t* level = nullptr, int64_t j_lo = 0, int64_t j_hi = -1,
                                  int32_t part = -1) {
  if (j_hi < 0) j_hi = st->m;
  if (j_lo < 0 || j_lo > j_hi || j_hi > st->m || part >= 8)
    return fail(FSMC_ERR_ARG, "advance: chain range or part out of bounds");
  if (variant < FSMC_PLAIN || variant > FSMC_AMORTIZED) return fail(FSMC_ERR_ARG, "bad step variant");
  GE ge;
  if (!pick_config(k->family, t->dim, lanes, ge, t->kind))
    return fail(FSMC_ERR_UNSUPPORTED, "no compiled (lanes, elements) configuration for this dimension");
  Params p;
  memset(&p, 0, sizeof(p));
  p.k = *k; p.t = *t; p.st = *st;
  p.t.full = k->family != FSMC_ESS;
  if (out) p.out = *out;
  p.n = n;
  p.tick_limit = tick_limit;
  p.variant = variant;
  p.mode = mode;
  int K = n_states(k);
  p.default_order = 1;
  for (int i = 0; i < K; i++) {
    p.order[i] = order ? order[i] : (i == 0 ? K : i);
    if (p.order[i] != (i == 0 ? K : i)) p.default_order = 0;
  }
  p.b_lp = lp;
  p.b_grad = grad;
  p.b_theta = theta;
  p.b_req_chain = req_chain;
  p.b_req_count = req_count;
  p.b_prior = op == 7;
  p.b_level = (long long*)level;
  cudaStream_t cs = (cudaStream_t)stream_;
  if (level) {  // this round's barrier level = last round's minimum count
    CUDA_TRY(cudaMemcpyAsync(level, level + 1, sizeof(int64_t), cudaMemcpyDeviceToDevice, cs));
    CUDA_TRY(cudaMemsetAsync(level + 1, 0x7f, sizeof(int64_t), cs));
    CUDA_TRY(cudaMemsetAsync(level + 2, 0, sizeof(int64_t), cs));
  }
  p.j_lo = j_lo;
  p.j_hi = j_hi;
  p.next_chain = part < 0 ? st->work : st->work + 128 + 16 * part;
  CUDA_TRY(cudaMemsetAsync(p.next_chain, 0, sizeof(unsigned), cs));
  CUDA_TRY(cudaMemsetAsync(req_count, 0, sizeof(int32_t), cs));
  CUDA_TRY(dispatch_family(op, ge, p, cs));
  return FSMC_OK;
}

fsmc_status fsmc_advance(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st, int64_t n,
                         int32_t variant, const int32_t* order, int64_t tick_limit, int32_t mode,
                         const fsmc_outputs* out, const double* lp, const double* grad, double* theta,
                         int32_t* req_chain, int32_t* req_count, int32_t lanes, void* stream_) {
  FSMC_NVTX("fsmc_advance");
  fsmc_status s = check_args(k, t, st);
  if (s != FSMC_OK) return s;
  if (k->precision != 0) return fail(FSMC_ERR_UNSUPPORTED, "the fp32 throughput mode covers fsmc_run and the windowed DRMH runs");
  if (!theta || !req_chain || !req_count || !lp || (k->family == FSMC_NUTS && !grad))
    return fail(FSMC_ERR_ARG, "advance needs theta, req_chain, req_count, lp (and grad for NUTS)");
  return advance_common(3, k, t, st, n, variant, order, tick_limit, mode, out, lp, grad, theta,
                        req_chain, req_count, lanes, stream_);
}

fsmc_status fsmc_advance_lockstep(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st, int64_t n,
                                  const fsmc_outputs* out, const double* lp, const double* grad,
                                  double* theta, int32_t* req_chain, int32_t* req_count, int64_t* level,
                                  int32_t lanes, void* stream_) {
  FSMC_NVTX("fsmc_advance_lockstep");
  fsmc_status s = check_args(k, t, st);
  if (s != FSMC_OK) return s;
  if (k->precision != 0) return fail(FSMC_ERR_UNSUPPORTED, "the fp32 throughput mode covers fsmc_run and the windowed DRMH runs");
  if (!theta || !req_chain || !req_count || !lp || !level || (k->family == FSMC_NUTS && !grad))
    return fail(FSMC_ERR_ARG, "advance_lockstep needs theta, req_chain, req_count, lp, level (and grad for NUTS)");
  return advance_common(3, k, t, st, n, FSMC_PLAIN, nullptr, INT64_MAX, 0, out, lp, grad, theta,
                        req_chain, req_count, lanes, stream_, level);
}

fsmc_status fsmc_advance_prior(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st, int64_t n,
                               int32_t variant, const int32_t* order, int64_t tick_limit, int32_t mode,
                               const fsmc_outputs* out, double* nu, int32_t* req_chain,
                               int32_t* req_count, int32_t lanes, void* stream_) {
  FSMC_NVTX("fsmc_advance_prior");
  fsmc_status s = check_args(k, t, st);
  if (s != FSMC_OK) return s;
  if (k->precision != 0) return fail(FSMC_ERR_UNSUPPORTED, "the fp32 throughput mode covers fsmc_run and the windowed DRMH runs");
  if (k->family != FSMC_ESS || t->prior_kind != FSMC_PRIOR_DENSE)
    return fail(FSMC_ERR_UNSUPPORTED, "the batched prior transform is for the elliptical kernel with a dense prior");
  if (!nu || !req_chain || !req_count)
    return fail(FSMC_ERR_ARG, "advance_prior needs nu, req_chain, req_count");
  return advance_common(7, k, t, st, n, variant, order, tick_limit, mode, out, nullptr, nullptr, nu,
                        req_chain, req_count, lanes, stream_);
}

fsmc_status fsmc_advance_prior_part(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st, int64_t n,
                                    int32_t variant, const int32_t* order, int64_t tick_limit, int32_t mode,
                                    const fsmc_outputs* out, double* nu, int32_t* req_chain,
                                    int32_t* req_count, int32_t lanes, int64_t j_lo, int64_t j_hi,
                                    int32_t part, void* stream_) {
  FSMC_NVTX("fsmc_advance_prior_part");
  fsmc_status s = check_args(k, t, st);
  if (s != FSMC_OK) return s;
  if (k->precision != 0) return fail(FSMC_ERR_UNSUPPORTED, "the fp32 throughput mode covers fsmc_run and the windowed DRMH runs");
  if (k->family != FSMC_ESS || t->prior_kind != FSMC_PRIOR_DENSE)
    return fail(FSMC_ERR_UNSUPPORTED, "the batched prior transform is for the elliptical kernel with a dense prior");
  if (!nu || !req_chain || !req_count || part < 0)
    return fail(FSMC_ERR_ARG, "advance_prior_part needs nu, req_chain, req_count and a part index");
  return advance_common(7, k, t, st, n, variant, order, tick_limit, mode, out, nullptr, nullptr, nu,
                        req_chain, req_count, lanes, stream_, nullptr, j_lo, j_hi, part);
}

// nu[r] = L nu[r] in place, every row summed in the sampling kernel's order
// (k ascending, one fma per term): the bit-exact batched prior transform
__global__ void __launch_bounds__(256) prior_apply_kernel(const double* __restrict__ Lt, double* nu, int d) {
  extern __shared__ double eps[];
  double* row = nu + (size_t)blockIdx.x * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) eps[i] = row[i];
  __syncthreads();
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    double acc = 0.0;
    for (int k = 0; k <= i; k++) acc = fma(__ldg(&Lt[(size_t)k * d + i]), eps[k], acc);
    row[i] = acc;
  }
}

// device math for tests: the restated functions against the library ones
__global__ void dmath_eval_kernel(int fn, const double* __restrict__ x, long long n, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double v = x[i];
    double r;
    switch (fn) {
      case 0: r = exp(v); break;
      case 1: r = exp_c(v); break;
      case 2: r = gl_exp(v); break;
      case 3: r = gl_log(v); break;
      case 4: r = log(v); break;
      case 5: r = sin(v); break;
      case 6: r = cos(v); break;
      case 7: { double sv, cv; sincos(v, &sv, &cv); r = sv; break; }
      default: { double sv, cv; sincos(v, &sv, &cv); r = cv; break; }
    }
    out[i] = r;
  }
}

fsmc_status fsmc_dmath_eval(int32_t fn, const double* x, int64_t n, double* out, void* stream_) {
  if (!x || !out || n < 0 || fn < 0 || fn > 8) return fail(FSMC_ERR_ARG, "dmath_eval: fn in 0..8, x, out");
  if (n == 0) return FSMC_OK;
  fsmc::count_launch();
  dmath_eval_kernel<<<(unsigned)std::min<long long>((n + 255) / 256, 148 * 16), 256, 0, (cudaStream_t)stream_>>>(
      fn, x, (long long)n, out);
  CUDA_TRY(cudaGetLastError());
  return FSMC_OK;
}

fsmc_status fsmc_prior_apply(const fsmc_target* t, double* nu, int64_t k, void* stream_) {
  FSMC_NVTX("fsmc_prior_apply");
  if (!t || !nu || k < 0) return fail(FSMC_ERR_ARG, "prior_apply needs a target and nu");
  if (t->prior_kind != FSMC_PRIOR_DENSE || !t->prior_t)
    return fail(FSMC_ERR_ARG, "prior_apply needs a dense prior factor");
  if (k == 0) return FSMC_OK;
  const size_t sb = (size_t)t->dim * sizeof(double);
  if (sb > 48 * 1024)
    CUDA_TRY(cudaFuncSetAttribute((const void*)prior_apply_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb));
  fsmc::count_launch();
  prior_apply_kernel<<<(unsigned)k, 256, sb, (cudaStream_t)stream_>>>(t->prior_t, nu, (int)t->dim);
  CUDA_TRY(cudaGetLastError());
  return FSMC_OK;
}

fsmc_status fsmc_run_windowed(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st, int64_t n,
                              int32_t variant, const int32_t* order, int64_t tick_limit, int32_t mode,
                              const fsmc_outputs* out, int64_t window, double* draws, int32_t lanes,
                              void* stream_) {
  return fsmc_run_windowed_overlap(k, t, st, n, variant, order, tick_limit, mode, out, window, draws, lanes,
                                   1, stream_);
}

fsmc_status fsmc_run_windowed_overlap(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st, int64_t n,
                                      int32_t variant, const int32_t* order, int64_t tick_limit,
                                      int32_t mode, const fsmc_outputs* out, int64_t window, double* draws,
                                      int32_t lanes, int32_t parts, void* stream_) {
  return fsmc_run_windowed_egress(k, t, st, n, variant, order, tick_limit, mode, out, window, draws, lanes,
                                  parts, nullptr, stream_);
}

fsmc_status fsmc_run_windowed_egress(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st, int64_t n,
                                     int32_t variant, const int32_t* order, int64_t tick_limit,
                                     int32_t mode, const fsmc_outputs* out, int64_t window, double* draws,
                                     int32_t lanes, int32_t parts, const fsmc_egress* eg, void* stream_) {
  FSMC_NVTX("fsmc_run_windowed_egress");
  fsmc_status s = check_args(k, t, st);
  if (s != FSMC_OK) return s;
  if (k->family != FSMC_DRMH) return fail(FSMC_ERR_UNSUPPORTED, "pre-drawn windows are for the DRMH kernels");
  if (!draws || window < t->dim + 1 || window > 65536)
    return fail(FSMC_ERR_ARG, "windowed run needs draws [m][window], dim + 1 <= window <= 65536");
  if (n < 0) return fail(FSMC_ERR_ARG, "n must be >= 0");
  if (variant < FSMC_PLAIN || variant > FSMC_AMORTIZED) return fail(FSMC_ERR_ARG, "bad step variant");
  GE ge;
  if (!pick_config(k->family, t->dim, lanes, ge, t->kind))
    return fail(FSMC_ERR_UNSUPPORTED, "no compiled (lanes, elements) configuration for this dimension");
  if ((s = check_f32(k, t, ge)) != FSMC_OK) return s;
  Params p;
  memset(&p, 0, sizeof(p));
  p.k = *k; p.t = *t; p.st = *st;
  p.t.full = 1;
  if (out) p.out = *out;
  p.n = n;
  p.tick_limit = tick_limit;
  p.variant = variant;
  p.mode = mode;
  int K = n_states(k);
  p.default_order = 1;
  for (int i = 0; i < K; i++) {
    p.order[i] = order ? order[i] : (i == 0 ? K : i);
    if (p.order[i] != (i == 0 ? K : i)) p.default_order = 0;
  }
  p.draws = draws;
  p.window = window;
  if (parts < 0 || parts > kMaxParts) return fail(FSMC_ERR_ARG, "windowed run: parts must be in 0..16");
  const bool pipelined = parts == 0;
  if (pipelined && k->split_body)   // a split proposal can end a window between its draws
    return fail(FSMC_ERR_UNSUPPORTED, "pipelined windows need the one-block DRMH proposal (split_body = 0)");
  if (pipelined) parts = 1;
  if (st->m < parts) parts = 1;
  cudaStream_t cs = (cudaStream_t)stream_;
  unsigned* w = st->work;
  // parts > 1: the chains in contiguous parts, each alternating its draw
  // generation and window kernels on its own stream, so one part's kernels
  // fill the SMs another part's kernel tail and launch gaps leave idle
  // host_samples (pinned): rows every chain has finished are copied to the
  // host on the egress stream while later rows are still being sampled
  const bool egress = eg && out && n > 0 &&
                      ((eg->samples && out->samples) || (out->loop_counts64 && (eg->loop_counts || eg->iter_counts)));
  cudaStream_t side[kMaxParts] = {};
  cudaEvent_t ev_fork = nullptr, ev_join[kMaxParts] = {}, ev_egress = nullptr;
  if (parts > 1 || egress) CUDA_TRY(side_streams(side));
  if (parts > 1) {
    CUDA_TRY(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    for (int h = 1; h < parts; h++) CUDA_TRY(cudaEventCreateWithFlags(&ev_join[h], cudaEventDisableTiming));
  }
  const size_t row_bytes = (size_t)st->m * t->dim * sizeof(double);
  const size_t crow = (size_t)st->m * sizeof(int64_t);
  long long rows_sent = 0;
  auto send_rows = [&](long long upto) -> cudaError_t {
    if (!egress || upto <= rows_sent) return cudaSuccess;
    const long long a = rows_sent, nr = upto - rows_sent;
    rows_sent = upto;
    cudaError_t e = cudaSuccess;
    if (eg->samples && out->samples)
      e = cudaMemcpyAsync((char*)eg->samples + a * row_bytes, (const char*)out->samples + a * row_bytes,
                          (size_t)nr * row_bytes, cudaMemcpyDeviceToHost, side[0]);
    if (out->loop_counts64) {
      for (int l = 0; e == cudaSuccess && eg->loop_counts && l < eg->n_loops; l++)
        e = cudaMemcpyAsync(eg->loop_counts + ((size_t)l * n + a) * st->m,
                            out->loop_counts64 + ((size_t)l * n + a) * st->m, (size_t)nr * crow,
                            cudaMemcpyDeviceToHost, side[0]);
      if (e == cudaSuccess && eg->iter_counts)
        e = cudaMemcpyAsync(eg->iter_counts + (size_t)a * st->m,
                            out->loop_counts64 + ((size_t)eg->iter_loop * n + a) * st->m, (size_t)nr * crow,
                            cudaMemcpyDeviceToHost, side[0]);
    }
    return e;
  };
  // per chain part: rows [part_sent[h], upto) of the part's chain columns
  // (pitched copies), so a part's finished rows leave without waiting for the
  // slowest chain of every other part
  long long part_sent[kMaxParts] = {};
  static int trace = -1;   // FSMC_EGRESS_TRACE=1: host time of every egress copy issued (stderr)
  if (trace < 0) trace = getenv("FSMC_EGRESS_TRACE") ? 1 : 0;
  static int nocopy = -1;  // FSMC_EGRESS_NOCOPY=1 (experiments): the egress bookkeeping without the copies
  if (nocopy < 0) nocopy = getenv("FSMC_EGRESS_NOCOPY") ? 1 : 0;
  const auto t_start = std::chrono::steady_clock::now();
  double t_wait = 0.0, t_send = 0.0;   // host ms in progress-check waits / egress copy calls (trace)
  auto send_part = [&](int h, long long lo, long long hi, long long upto) -> cudaError_t {
    if (!egress || upto <= part_sent[h] || hi <= lo) return cudaSuccess;
    if (trace)
      fprintf(stderr, "egress %.3f ms part %d rows %lld..%lld\n",
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count(), h,
              part_sent[h], upto);
    const long long a = part_sent[h], nr = upto - part_sent[h];
    part_sent[h] = upto;
    const size_t d8 = (size_t)t->dim * sizeof(double);
    cudaError_t e = cudaSuccess;
    if (nocopy) return e;
    if (eg->samples && out->samples)
      e = cudaMemcpy2DAsync((char*)eg->samples + a * row_bytes + lo * d8, row_bytes,
                            (const char*)out->samples + a * row_bytes + lo * d8, row_bytes,
                            (size_t)(hi - lo) * d8, (size_t)nr, cudaMemcpyDeviceToHost, side[0]);
    if (out->loop_counts64) {
      const size_t w8 = (size_t)(hi - lo) * sizeof(int64_t);
      for (int l = 0; e == cudaSuccess && eg->loop_counts && l < eg->n_loops; l++)
        e = cudaMemcpy2DAsync(eg->loop_counts + ((size_t)l * n + a) * st->m + lo, crow,
                              out->loop_counts64 + ((size_t)l * n + a) * st->m + lo, crow, w8, (size_t)nr,
                              cudaMemcpyDeviceToHost, side[0]);
      if (e == cudaSuccess && eg->iter_counts)
        e = cudaMemcpy2DAsync(eg->iter_counts + (size_t)a * st->m + lo, crow,
                              out->loop_counts64 + ((size_t)eg->iter_loop * n + a) * st->m + lo, crow, w8,
                              (size_t)nr, cudaMemcpyDeviceToHost, side[0]);
    }
    return e;
  };
  static int draw_bps = -1;   // draws-kernel blocks per SM (FSMC_DRAW_BLOCKS_PER_SM; 0 = fill)
  if (draw_bps < 0) {
    const char* e = getenv("FSMC_DRAW_BLOCKS_PER_SM");
    draw_bps = e ? atoi(e) : 0;
    if (draw_bps < 0) draw_bps = 0;
  }
  static int win_bps = -1;   // window-kernel blocks per SM (FSMC_WIN_BLOCKS_PER_SM; 0 = occupancy)
  if (win_bps < 0) {
    const char* e = getenv("FSMC_WIN_BLOCKS_PER_SM");
    win_bps = e ? atoi(e) : 0;
    if (win_bps < 0) win_bps = 0;
  }
#ifndef FSMC_KCHECK   // rounds between progress checks (1: C2 e2e 3.80e8 vs 3.77e8 at 2)
#define FSMC_KCHECK 1
#endif
  if (pipelined) {
    // Pipelined windows: one chain range, draws double-buffered ([2][m][window]).
    // Every window runs each unfinished chain exactly window / (dim + 1)
    // proposals (a DRMH proposal takes dim normals and one uniform; the run
    // stops a window right after the proposal that no longer leaves room for
    // another), so window r + 1 of chain j starts at a counter known before
    // window r runs: base_j + (r + 1) * stride.  The generator fills window
    // r + 1 on its own stream while window r runs; a chain that finishes
    // early simply never reads its later windows.
    const long long per = t->dim + 1;
    const long long stride = (window / per) * per;
    long long* base = nullptr;
    CUDA_TRY(cudaMallocAsync((void**)&base, (size_t)st->m * sizeof(long long), cs));
    CUDA_TRY(cudaMemcpy2DAsync(base, sizeof(long long), st->ints + FSMC_I_COUNTER, FSMC_NINT * sizeof(int64_t),
                               sizeof(long long), (size_t)st->m, cudaMemcpyDeviceToDevice, cs));
    if (!egress) CUDA_TRY(side_streams(side));
    cudaStream_t gs = side[1];
    Params pw = p;
    pw.j_lo = 0;
    pw.j_hi = st->m;
    pw.next_chain = w;
    pw.unfinished = w + 8;
    pw.min_count = egress ? w + 9 : nullptr;
    pw.draw_blocks_per_sm = draw_bps;
    pw.win_blocks_per_sm = win_bps;
    pw.draw_base = base;
    pw.draw_stride = stride;
    Params pg = pw;
    double* buf[2] = {draws, draws + (size_t)st->m * window};
    cudaEvent_t eg[2], ew[2], ev_start, ev_gen_done;
    for (int b = 0; b < 2; b++) {
      CUDA_TRY(cudaEventCreateWithFlags(&eg[b], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&ew[b], cudaEventDisableTiming));
    }
    CUDA_TRY(cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&ev_gen_done, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(ev_start, cs));
    CUDA_TRY(cudaStreamWaitEvent(gs, ev_start, 0));
    pg.draws = buf[0];
    pg.draw_round = 0;
    CUDA_TRY(dispatch_family(6, ge, pg, gs));
    CUDA_TRY(cudaEventRecord(eg[0], gs));
    const int kCheck = FSMC_KCHECK;
    unsigned* hc = nullptr;   // [2 checks][unfinished, lowest count]
    CUDA_TRY(cudaHostAlloc(&hc, 4 * sizeof(unsigned), cudaHostAllocDefault));
    cudaEvent_t evc[2];
    for (int b = 0; b < 2; b++) CUDA_TRY(cudaEventCreateWithFlags(&evc[b], cudaEventDisableTiming));
    bool pending[2] = {false, false};
    int cur = 0;
    for (long long r = 0;; r++) {
    FSMC_NVTX("windowed round");
      FSMC_NVTX("windowed round");
      const int b = (int)(r & 1);
      pg.draws = buf[b ^ 1];   // the next window, into the half window r - 1 used
      pg.draw_round = r + 1;
      if (r >= 1) CUDA_TRY(cudaStreamWaitEvent(gs, ew[b ^ 1], 0));
      CUDA_TRY(dispatch_family(6, ge, pg, gs));
      CUDA_TRY(cudaEventRecord(eg[b ^ 1], gs));
      CUDA_TRY(cudaStreamWaitEvent(cs, eg[b], 0));
      CUDA_TRY(cudaMemsetAsync(pw.next_chain, 0, sizeof(unsigned), cs));
      CUDA_TRY(cudaMemsetAsync(pw.unfinished, 0, sizeof(unsigned), cs));
      if (egress) CUDA_TRY(cudaMemsetAsync(pw.min_count, 0xff, sizeof(unsigned), cs));
      pw.draws = buf[b];
      pw.draw_round = r;
      CUDA_TRY(dispatch_family(5, ge, pw, cs));
      CUDA_TRY(cudaEventRecord(ew[b], cs));
      if (r % kCheck != kCheck - 1) continue;
      // progress, read one check late (as the parts loop below)
      CUDA_TRY(cudaMemcpyAsync(hc + cur * 2, pw.unfinished, (egress ? 2 : 1) * sizeof(unsigned),
                               cudaMemcpyDeviceToHost, cs));
      CUDA_TRY(cudaEventRecord(evc[cur], cs));
      pending[cur] = true;
      const int prev = cur ^ 1;
      cur = prev;
      if (!pending[prev]) continue;
      pending[prev] = false;
      CUDA_TRY(cudaEventSynchronize(evc[prev]));
      const unsigned* v = hc + prev * 2;
      if (!v[0]) break;
      if (egress && v[1] != 0xffffffffu) CUDA_TRY(send_rows(std::min<long long>(n, v[1])));
    }
    for (int b = 0; b < 2; b++) {
      if (pending[b]) CUDA_TRY(cudaEventSynchronize(evc[b]));
      CUDA_TRY(cudaEventDestroy(evc[b]));
    }
    CUDA_TRY(cudaFreeHost(hc));
    // the generator stream's last (unused) window joins the run's stream
    CUDA_TRY(cudaEventRecord(ev_gen_done, gs));
    CUDA_TRY(cudaStreamWaitEvent(cs, ev_gen_done, 0));
    CUDA_TRY(cudaFreeAsync(base, cs));
    if (egress) {
      CUDA_TRY(send_rows(n));
      CUDA_TRY(cudaEventCreateWithFlags(&ev_egress, cudaEventDisableTiming));
      CUDA_TRY(cudaEventRecord(ev_egress, side[0]));
      CUDA_TRY(cudaStreamWaitEvent(cs, ev_egress, 0));
      CUDA_TRY(cudaEventDestroy(ev_egress));
    }
    for (int b = 0; b < 2; b++) {
      CUDA_TRY(cudaEventDestroy(eg[b]));
      CUDA_TRY(cudaEventDestroy(ew[b]));
    }
    CUDA_TRY(cudaEventDestroy(ev_start));
    CUDA_TRY(cudaEventDestroy(ev_gen_done));
    return FSMC_OK;
  }
  static int part_streams = -1;   // FSMC_PART_STREAMS: streams the chain parts share (1..15)
  if (part_streams < 0) {
    const char* e = getenv("FSMC_PART_STREAMS");
    part_streams = e ? atoi(e) : kMaxParts - 1;
    part_streams = std::max(1, std::min(part_streams, kMaxParts - 1));
  }
  Params ph[kMaxParts];
  cudaStream_t sh[kMaxParts];
  for (int h = 0; h < parts; h++) {
    ph[h] = p;
    ph[h].j_lo = st->m * h / parts;
    ph[h].j_hi = st->m * (h + 1) / parts;
    ph[h].next_chain = w + 16 * h;
    ph[h].unfinished = w + 16 * h + 8;   // [8] unfinished chains, [9] lowest sample count seen
    ph[h].min_count = egress ? w + 16 * h + 9 : nullptr;
    ph[h].draw_blocks_per_sm = draw_bps;
    // parts share FSMC_PART_STREAMS streams round robin (default: one per
    // part up to 15; parts on one stream run back to back -- measured slower)
    const int hs = h % part_streams;
    sh[h] = hs == 0 ? cs : side[hs];
  }
  if (parts > 1) {
    CUDA_TRY(cudaEventRecord(ev_fork, cs));
    for (int h = 1; h < parts; h++) CUDA_TRY(cudaStreamWaitEvent(sh[h], ev_fork, 0));
  }
  // progress checks every kCheck rounds, read one check late: each check's
  // counters go to pinned host memory asynchronously and are consumed at the
  // next check, so the streams always hold queued rounds and never drain (a
  // part seen finished stops receiving rounds; the <= kCheck rounds queued
  // past its end find no unfinished chain and exit at once)
  const int kCheck = FSMC_KCHECK;   // rounds between progress checks
  unsigned* hc = nullptr;   // [2 checks][kMaxParts][unfinished, lowest count]
  CUDA_TRY(cudaHostAlloc(&hc, 2 * kMaxParts * 2 * sizeof(unsigned), cudaHostAllocDefault));
  cudaEvent_t evc[2][kMaxParts] = {};
  for (int b = 0; b < 2; b++)
    for (int h = 0; h < parts; h++) CUDA_TRY(cudaEventCreateWithFlags(&evc[b][h], cudaEventDisableTiming));
  bool live[kMaxParts], asked[2][kMaxParts] = {};
  for (int h = 0; h < kMaxParts; h++) live[h] = h < parts;
  bool pending[2] = {false, false};
  int cur = 0;
  // at most gen_slots draw-generation kernels in flight: generator k (in
  // launch order over parts and rounds) starts after generator k - gen_slots
  // has finished, so the full-occupancy generators do not crowd out the
  // latency-bound window kernels of the other parts
  // (measured on B200, C2 at 8 parts: 3.62e8 samples/s unbounded, 4.08e8
  // with 2 slots; default parts / 4, FSMC_GEN_SLOTS overrides, 0 = unbounded)
  static int gen_slots_env = -2;
  if (gen_slots_env == -2) {
    const char* e = getenv("FSMC_GEN_SLOTS");
    gen_slots_env = e ? std::max(0, atoi(e)) : -1;
  }
  const int gen_slots = std::min(kMaxParts, gen_slots_env >= 0 ? gen_slots_env : (parts >= 4 ? parts / 4 : 0));
  cudaEvent_t gen_ring[kMaxParts] = {};
  for (int i = 0; i < gen_slots; i++) CUDA_TRY(cudaEventCreateWithFlags(&gen_ring[i], cudaEventDisableTiming));
  long long gen_k = 0;
  for (long long r = 0;; r++) {
    FSMC_NVTX("windowed round");
    for (int h = 0; h < parts; h++) {
      if (!live[h]) continue;
      if (gen_slots > 0 && gen_k >= gen_slots) CUDA_TRY(cudaStreamWaitEvent(sh[h], gen_ring[gen_k % gen_slots], 0));
      CUDA_TRY(dispatch_family(6, ge, ph[h], sh[h]));
      if (gen_slots > 0) CUDA_TRY(cudaEventRecord(gen_ring[gen_k % gen_slots], sh[h]));
      gen_k++;
      CUDA_TRY(cudaMemsetAsync(ph[h].next_chain, 0, sizeof(unsigned), sh[h]));
      CUDA_TRY(cudaMemsetAsync(ph[h].unfinished, 0, sizeof(unsigned), sh[h]));
      if (egress) CUDA_TRY(cudaMemsetAsync(ph[h].min_count, 0xff, sizeof(unsigned), sh[h]));
      CUDA_TRY(dispatch_family(5, ge, ph[h], sh[h]));
    }
    if (r % kCheck != kCheck - 1) continue;
    for (int h = 0; h < parts; h++) {
      asked[cur][h] = live[h];
      if (!live[h]) continue;
      CUDA_TRY(cudaMemcpyAsync(hc + (cur * kMaxParts + h) * 2, ph[h].unfinished,
                               (egress ? 2 : 1) * sizeof(unsigned), cudaMemcpyDeviceToHost, sh[h]));
      CUDA_TRY(cudaEventRecord(evc[cur][h], sh[h]));
    }
    pending[cur] = true;
    const int prev = cur ^ 1;
    cur = prev;
    if (!pending[prev]) continue;
    pending[prev] = false;
    bool any = false;
    for (int h = 0; h < parts; h++) {
      if (!asked[prev][h]) continue;
      auto tw0 = std::chrono::steady_clock::now();
      CUDA_TRY(cudaEventSynchronize(evc[prev][h]));
      t_wait += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tw0).count();
      const unsigned* v = hc + (prev * kMaxParts + h) * 2;
      if (!v[0]) live[h] = false;
      any = any || v[0];
      // rows below every chain's sample count in the part are final (a part
      // that finished, or whose last round skipped every chain, has all n)
      if (egress) {
        const long long rows = !v[0] ? n : (v[1] != 0xffffffffu ? std::min<long long>(n, v[1]) : 0);
        auto ts0 = std::chrono::steady_clock::now();
        CUDA_TRY(send_part(h, ph[h].j_lo, ph[h].j_hi, rows));
        t_send += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ts0).count();
      }
    }
    if (!any) break;
  }
  // the unconsumed check still copies into hc: let it land before freeing
  for (int b = 0; b < 2; b++)
    for (int h = 0; h < parts; h++) {
      if (pending[b] && asked[b][h]) CUDA_TRY(cudaEventSynchronize(evc[b][h]));
      CUDA_TRY(cudaEventDestroy(evc[b][h]));
    }
  CUDA_TRY(cudaFreeHost(hc));
  for (int i = 0; i < gen_slots; i++) CUDA_TRY(cudaEventDestroy(gen_ring[i]));
  if (trace)
    fprintf(stderr, "windowed run: host %.3f ms, %.3f ms in check waits, %.3f ms in egress copy calls\n",
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count(),
            t_wait, t_send);
  if (egress) {
    for (int h = 0; h < parts; h++) CUDA_TRY(send_part(h, ph[h].j_lo, ph[h].j_hi, n));
    CUDA_TRY(cudaEventCreateWithFlags(&ev_egress, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(ev_egress, side[0]));
    CUDA_TRY(cudaStreamWaitEvent(cs, ev_egress, 0));
    CUDA_TRY(cudaEventDestroy(ev_egress));
  }
  if (parts > 1) {
    for (int h = 1; h < parts; h++) {
      CUDA_TRY(cudaEventRecord(ev_join[h], sh[h]));
      CUDA_TRY(cudaStreamWaitEvent(cs, ev_join[h], 0));
      CUDA_TRY(cudaEventDestroy(ev_join[h]));   // released once the wait completes
    }
    CUDA_TRY(cudaEventDestroy(ev_fork));
  }
  return FSMC_OK;
}

fsmc_status fsmc_profile_blocks(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st,
                                int64_t tick_limit, unsigned long long* cycles, void* stream_) {
  FSMC_NVTX("fsmc_profile_blocks");
  fsmc_status s = check_args(k, t, st);
  if (s != FSMC_OK) return s;
  if (k->precision != 0) return fail(FSMC_ERR_UNSUPPORTED, "the fp32 throughput mode covers fsmc_run and the windowed DRMH runs");
  if (!cycles || tick_limit < 0) return fail(FSMC_ERR_ARG, "profile needs cycles[16] and tick_limit >= 0");
  // one chain per warp where compiled: a lane group then never waits on
  // other chains' divergent blocks, so its clock deltas are its own blocks
  GE ge;
  if (!pick_config(k->family, t->dim, 32, ge, t->kind) && !pick_config(k->family, t->dim, 0, ge, t->kind))
    return fail(FSMC_ERR_UNSUPPORTED, "no compiled (lanes, elements) configuration for this dimension");
  Params p;
  memset(&p, 0, sizeof(p));
  p.k = *k; p.t = *t; p.st = *st;
  p.t.full = k->family != FSMC_ESS;
  p.n = 0;
  p.tick_limit = tick_limit;
  p.variant = FSMC_PLAIN;
  p.mode = 1;
  p.prof = cycles;
  cudaStream_t cs = (cudaStream_t)stream_;
  p.next_chain = st->work;
  CUDA_TRY(cudaMemsetAsync(p.next_chain, 0, sizeof(unsigned), cs));
  CUDA_TRY(dispatch_family(4, ge, p, cs));
  return FSMC_OK;
}

fsmc_status fsmc_lockstep_run(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st, int64_t n,
                              const fsmc_outputs* out, int32_t lanes, void* stream_) {
  FSMC_NVTX("fsmc_lockstep_run");
  fsmc_status s = check_args(k, t, st);
  if (s != FSMC_OK) return s;
  if (k->precision != 0) return fail(FSMC_ERR_UNSUPPORTED, "the fp32 throughput mode covers fsmc_run and the windowed DRMH runs");
  GE ge;
  if (!pick_config(k->family, t->dim, lanes, ge, t->kind))
    return fail(FSMC_ERR_UNSUPPORTED, "no compiled (lanes, elements) configuration for this dimension");
  Params p;
  memset(&p, 0, sizeof(p));
  p.k = *k; p.t = *t; p.st = *st;
  p.t.full = k->family != FSMC_ESS;
  if (out) p.out = *out;
  p.n = n;
  cudaStream_t cs = (cudaStream_t)stream_;
  unsigned* w = st->work;
  p.bar_count = w + 1;
  p.bar_gen = w + 2;
  p.active_flags = w + 3;
  CUDA_TRY(cudaMemsetAsync(w + 1, 0, 4 * sizeof(unsigned), cs));
  CUDA_TRY(dispatch_family(2, ge, p, cs));
  return FSMC_OK;
}

fsmc_status fsmc_lockstep_barrier_probe(const fsmc_kernel* k, const fsmc_target* t, fsmc_state* st,
                                        int64_t iters, int32_t lanes, void* stream_) {
  FSMC_NVTX("fsmc_lockstep_barrier_probe");
  fsmc_status s = check_args(k, t, st);
  if (s != FSMC_OK) return s;
  if (k->precision != 0) return fail(FSMC_ERR_UNSUPPORTED, "the fp32 throughput mode covers fsmc_run and the windowed DRMH runs");
  if (iters < 1) return fail(FSMC_ERR_ARG, "iters must be >= 1");
  GE ge;
  if (!pick_config(k->family, t->dim, lanes, ge, t->kind))
    return fail(FSMC_ERR_UNSUPPORTED, "no compiled (lanes, elements) configuration for this dimension");
  Params p;
  memset(&p, 0, sizeof(p));
  p.k = *k; p.t = *t; p.st = *st;
  p.t.full = k->family != FSMC_ESS;
  p.n = iters;
  cudaStream_t cs = (cudaStream_t)stream_;
  unsigned* w = st->work;
  p.bar_count = w + 1;
  p.bar_gen = w + 2;
  p.active_flags = w + 3;
  CUDA_TRY(cudaMemsetAsync(w + 1, 0, 5 * sizeof(unsigned), cs));
  CUDA_TRY(dispatch_family(9, ge, p, cs));
  return FSMC_OK;
}

fsmc_status fsmc_copy_to_host_2d(void* dst, const void* src, int64_t pitch, int64_t width, int64_t rows,
                                 void* stream_) {
  if (!dst || !src || pitch < width || width < 0 || rows < 0) return fail(FSMC_ERR_ARG, "bad 2-D copy");
  if (!rows || !width) return FSMC_OK;
  CUDA_TRY(cudaMemcpy2DAsync(dst, (size_t)pitch, src, (size_t)pitch, (size_t)width, (size_t)rows,
                             cudaMemcpyDeviceToHost, (cudaStream_t)stream_));
  return FSMC_OK;
}

fsmc_status fsmc_target_eval(const fsmc_target* t, const double* X, int64_t m, double* lp, double* grad,
                             int32_t family, int32_t lanes, void* stream_) {
  FSMC_NVTX("fsmc_target_eval");
  if (!t || !X || !lp || m < 0) return fail(FSMC_ERR_ARG, "bad target_eval args");
  if (!m) return FSMC_OK;
  GE ge;
  if (!pick_config(family ? family : FSMC_ESS, t->dim, lanes, ge, t->kind))
    return fail(FSMC_ERR_UNSUPPORTED, "dimension not supported");
  fsmc_target tt = *t;
  tt.full = family != FSMC_ESS;   // 0 = the default layout, full log density
  cudaStream_t cs = (cudaStream_t)stream_;
  long long groups = (m + kThreads / ge.g - 1) / (kThreads / ge.g);
  int blocks = (int)std::min<long long>(groups, 148LL * 8);
#define X(GG, EE)                                                                           \
  if (ge.g == GG && ge.e == EE) {                                                           \
    CUDA_TRY(allow_smem(target_eval_kernel<GG, EE>, smem_bytes<GG, EE>(group_doubles(tt))));     \
    fsmc::count_launch();                                                         \
    target_eval_kernel<GG, EE><<<blocks, kThreads, smem_bytes<GG, EE>(group_doubles(tt)), cs>>>(tt, X, m, lp, grad); \
    CUDA_TRY(cudaGetLastError());                                                         \
    return FSMC_OK;                                                                       \
  }
  FSMC_EVAL_CONFIGS(X)
#undef X
  return fail(FSMC_ERR_UNSUPPORTED, "dimension not supported");
}

fsmc_status fsmc_logreg_epilogue(const float* Z, const float* y, int64_t rows, int64_t N, float* R,
                                 double* lp, void* stream_) {
  FSMC_NVTX("fsmc_logreg_epilogue");
  if (!Z || !y || !R || !lp || rows < 0 || N < 1) return fail(FSMC_ERR_ARG, "bad epilogue args");
  if (!rows) return FSMC_OK;
  if (rows > 65535) return fail(FSMC_ERR_ARG, "at most 65535 rows per epilogue call");
  dim3 grid((unsigned)((N + kEpiCols - 1) / kEpiCols), (unsigned)rows);
  fsmc::count_launch();
  logreg_epilogue_kernel<<<grid, 256, 0, (cudaStream_t)stream_>>>(Z, y, N, R, lp);
  CUDA_TRY(cudaGetLastError());
  return FSMC_OK;
}

fsmc_status fsmc_diag_partials(const double* samples, int64_t n, int64_t m, int64_t dim, int64_t burn,
                               int64_t lag0, int64_t n_lags, double* chain_mean, double* acov,
                               double* chain_var, void* stream_) {
  FSMC_NVTX("fsmc_diag_partials");
  if (!samples || n - burn < 2 || m < 1 || dim < 1 || !chain_mean) return fail(FSMC_ERR_ARG, "bad diag args");
  cudaStream_t cs = (cudaStream_t)stream_;
  if (lag0 == 0) {
    long long tot = m * dim;
    fsmc::count_launch();
    diag_mean_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, cs>>>(samples, n, m, dim, burn, chain_mean);
    CUDA_TRY(cudaGetLastError());
  }
  if (n_lags > 0 && acov) {
    if (n_lags != kLagTile) return fail(FSMC_ERR_ARG, "n_lags must be 32 (one lag tile per call)");
    CUDA_TRY(cudaMemsetAsync(acov, 0, sizeof(double) * kLagTile * dim, cs));
    long long tot = m * dim;
    size_t sm = dim <= 128 ? sizeof(double) * kLagTile * dim : 0;
    // wide targets reduce in global atomics: past the first tile (no per-chain
    // variance), each thread folds 8 chains first
    const long long cpt = (dim > 128 && lag0 > 0) ? 8 : 1;
    tot = ((m + cpt - 1) / cpt) * dim;
    fsmc::count_launch();
    diag_acov_kernel<<<(unsigned)((tot + 127) / 128), 128, sm, cs>>>(samples, n, m, dim, burn, lag0,
                                                                     chain_mean, acov, chain_var, cpt);
    CUDA_TRY(cudaGetLastError());
  }
  return FSMC_OK;
}

}  // extern "C"
