// kernels.cuh -- the three per-family kernels and their launchers.
//
//   fsm_init_kernel   init_batch                     lockstep.py:175-206
//   fsm_run_kernel    run_fsm_batched tick loop      lockstep.py:308-406
//   lockstep_kernel   run_standard_batched           lockstep.py:238-305
//
// Included by one translation unit per family (fam_*.cu) so the families
// compile in parallel.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <utility>

#include "configs.h"
#include "fsm_device.cuh"
#include "launch_count.h"

namespace fsmc {

constexpr int kThreads = 128;


// dynamic shared memory: one cooperative-normal scratch per warp, then the
// per-group plugin scratch (dim doubles for dense operators plus whatever
// the plugin asks for in fsmc_target.scratch, e.g. a GP kernel matrix)
__host__ __device__ inline int group_doubles(const fsmc_target& t) { return t.dim + t.scratch; }
template <int G, int E>
__device__ __forceinline__ double* warp_scratch(double* smem, int gd) {
  return smem + (threadIdx.x >> 5) * normal_scratch_doubles<E>();
}
template <int G, int E>
__device__ __forceinline__ double* group_scratch(double* smem, int gd) {
  return smem + (kThreads / 32) * normal_scratch_doubles<E>() + (threadIdx.x / G) * gd;
}
// a family's vectors kept in the group's shared memory (FF::SVECS, the NUTS
// trajectory ends) follow the plugin scratch in each group's region
template <class FF, int G, int E>
__host__ __device__ inline int group_doubles_f(const fsmc_target& t) {
  return group_doubles(t) + FF::SVECS * G * E;
}
template <class FF, int G>
__device__ __forceinline__ void bind_state(FF& f, double* sm, const fsmc_target& t, const Grp<G>& grp) {
  if constexpr (FF::SVECS > 0) f.bind(sm + group_doubles(t), grp.lane);
}
template <int G, int E>
inline size_t smem_bytes(int gd) {
  return ((size_t)(kThreads / G) * gd + (size_t)(kThreads / 32) * normal_scratch_doubles<E>()) *
         sizeof(double);
}
// opt a kernel into more than 48 KB of dynamic shared memory when needed
template <class K>
inline cudaError_t allow_smem(K* kern, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// registers: 4 resident blocks per SM for thread-per-chain configurations so
// that a full batch of chains is co-resident (no second wave)
#ifndef FSMC_WARP_MIN_BLOCKS
#define FSMC_WARP_MIN_BLOCKS 3
#endif
template <int G>
__host__ __device__ constexpr int min_blocks() { return G == 1 ? 4 : (G == 32 ? FSMC_WARP_MIN_BLOCKS : (G == 128 ? 4 : 1)); }
// block-per-chain NUTS (G = 128, C5's advance kernel) keeps its registers: 4
// resident blocks would spill its twelve-vector state
// fp32 throughput-mode families (half the register footprint per vector):
// more resident blocks
// warp-per-chain families with vectors in shared memory (NUTS ends): fewer
// registers, more resident blocks
#ifndef FSMC_SMEM_WARP_MIN_BLOCKS
#define FSMC_SMEM_WARP_MIN_BLOCKS 4
#endif
#ifndef FSMC_F32_MIN_BLOCKS
#define FSMC_F32_MIN_BLOCKS 5          // thread-per-chain groups
#endif
#ifndef FSMC_F32_WARP_MIN_BLOCKS
#define FSMC_F32_WARP_MIN_BLOCKS 4     // warp-per-chain groups (NUTS: 12 vectors + checkpoints)
#endif
template <class FF>
constexpr bool is_f32_family() {
  return std::is_same<typename std::remove_reference<decltype(std::declval<FF&>().x[0])>::type, float>::value;
}
template <template <int, int> class F, int G, int E>
__host__ __device__ constexpr int min_blocks_for() {
  return is_f32_family<F<G, E>>() ? (G == 1 ? FSMC_F32_MIN_BLOCKS : FSMC_F32_WARP_MIN_BLOCKS)
                                  : ((G == 128 && F<G, E>::GRAD) ? 1
                                     : ((G == 32 && F<G, E>::SVECS > 0) ? FSMC_SMEM_WARP_MIN_BLOCKS : min_blocks<G>()));
}

struct LaunchCtx {
  int num_sms;
};

// ---------------------------------------------------------------- init
template <template <int, int> class F, int G, int E>
__global__ void __launch_bounds__(kThreads) fsm_init_kernel(Params p, uint64_t parent_stream,
                                                            long long chain_offset, const double* x0,
                                                            double jitter) {
  extern __shared__ double smem[];
  Grp<G> grp;
  const int gib = threadIdx.x / G;
  double* sm = group_scratch<G, E>(smem, group_doubles_f<F<G, E>, G, E>(p.t));
  const long long groups = (long long)gridDim.x * (kThreads / G);
  const int d = p.t.dim;
  double* ws = warp_scratch<G, E>(smem, group_doubles_f<F<G, E>, G, E>(p.t));
  for (long long j = (long long)blockIdx.x * (kThreads / G) + gib; j < p.st.m; j += groups) {
    Core c;
    memset(&c, 0, sizeof(c));
    c.ws = ws;
    uint64_t stream = split_stream(parent_stream, (uint64_t)(chain_offset + j));  // prng.py:84-94
    c.hsc = hash_seed_stream(p.st.seed, stream);
    c.state = 1;
    F<G, E> f;
    bind_state<F<G, E>, G>(f, sm, p.t, grp);
#pragma unroll
    for (int e = 0; e < E; e++) {
      int i = grp.idx(e);
      f.x[e] = (i < d && x0) ? x0[i] : 0.0;
    }
    if (jitter > 0.0) {  // lockstep.py:195-198: N(0, jitter^2 I) offset drawn first
      double eps[E];
      normal_vec<G, E>(c, d, eps, grp);
#pragma unroll
      for (int e = 0; e < E; e++) f.x[e] = f.x[e] + jitter * eps[e];
    }
    bool ok = true;
    if constexpr (F<G, E>::SHAPE == SHAPE_NESTED) {
      f.init_state();
      f.ck = nullptr;
    } else if (p.b_defer) {
      f.init_pre();   // the evaluation point is x (vec row 0); fsm_init_finish_kernel completes
    } else {
      f.init_pre();
      double lp = target_eval<G, E, false>(p.t, f.ev(), f.evg(), sm, grp);
      if (is_target_failure(lp)) {
        set_error(c, FSMC_E_TARGET, 1);
        ok = false;
      } else {
        ok = f.init_post(c, lp);
      }
    }
    f.store(p, j, grp);
    if (grp.lane == 0) {
      core_store(c, p, j);
      p.st.ints[(size_t)j * FSMC_NINT + FSMC_I_STREAM] = (int64_t)stream;
      p.st.ints[(size_t)j * FSMC_NINT + FSMC_I_DRAW0] = (int64_t)c.ctr;
      if (!ok) report_error(c, p, j);
    }
  }
}

// deferred init, second half: init_post with the batched evaluation of the
// starting point (lp[j], j = chain), exactly as fsm_init_kernel would
template <template <int, int> class F, int G, int E>
__global__ void __launch_bounds__(kThreads) fsm_init_finish_kernel(Params p) {
  extern __shared__ double smem[];
  Grp<G> grp;
  double* sm = group_scratch<G, E>(smem, group_doubles_f<F<G, E>, G, E>(p.t));
  const int gib = threadIdx.x / G;
  const long long groups = (long long)gridDim.x * (kThreads / G);
  for (long long j = (long long)blockIdx.x * (kThreads / G) + gib; j < p.st.m; j += groups) {
    Core c;
    core_load(c, p, j);
    if (c.err_kind != FSMC_E_NONE) continue;
    F<G, E> f;
    bind_state<F<G, E>, G>(f, sm, p.t, grp);
    f.load(p, j, grp);
    bool ok = true;
    if constexpr (F<G, E>::SHAPE != SHAPE_NESTED) {
      f.init_pre();
      const double lp = p.b_init_lp[j];
      if (is_target_failure(lp)) {
        set_error(c, FSMC_E_TARGET, 1);
        ok = false;
      } else {
        ok = f.init_post(c, lp);
      }
    }
    f.store(p, j, grp);
    if (grp.lane == 0) {
      core_store(c, p, j);
      if (!ok) report_error(c, p, j);
    }
  }
}

// ----------------------------------------------------------------- run
// Every lane group pulls chains from a queue and runs each to completion
// with its state in registers.  No barrier anywhere: chains in different
// states simply execute different blocks.
template <template <int, int> class F, int G, int E, int TK, int VAR = 0>
__global__ void __launch_bounds__(kThreads, (min_blocks_for<F, G, E>())) fsm_run_kernel(Params p) {
  extern __shared__ double smem[];
  Grp<G> grp;
  double* sm = group_scratch<G, E>(smem, group_doubles_f<F<G, E>, G, E>(p.t));
  double* ws = warp_scratch<G, E>(smem, group_doubles_f<F<G, E>, G, E>(p.t));
  while (true) {   // chains [j_lo, j_hi) of the state block (fsmc_run_egress runs it in parts)
    long long j = 0;
    if (grp.lane == 0) j = atomicAdd(p.next_chain, 1u);
    j = p.j_lo + grp.bcast_ll(j, 0);
    if (j >= p.j_hi) break;
    Core c;
    core_load(c, p, j);
    c.ws = ws;
    if (c.err_kind != FSMC_E_NONE) continue;
    F<G, E> f;
    bind_state<F<G, E>, G>(f, sm, p.t, grp);
    f.load(p, j, grp);
    bool ok = true;
    const long long n_stop = p.mode == 0 ? p.n : (1LL << 62);
#pragma unroll 1
    while (c.count < n_stop && c.tick < p.tick_limit)
      if (!tick<F<G, E>, G, E, TK, false, VAR>(p, c, f, sm, j, grp)) { ok = false; break; }
    f.store(p, j, grp);
    if (grp.lane == 0) {
      core_store(c, p, j);
      if (!ok) report_error(c, p, j);
    }
  }
}

// ------------------------------------------------------------ windowed
#ifndef FSMC_WIN_NT
#define FSMC_WIN_NT 0
#endif
// fsm_run_kernel over pre-drawn windows (fsmc_run_windowed): the chain's
// draws at counters dbase .. dbase + window - 1 are in p.draws[j]; it ticks
// while a tick's worst case (dim + 1 draws for DRMH) still fits.
#ifndef FSMC_WIN_MINB
#define FSMC_WIN_MINB 0      // > 0: resident blocks the window kernels are compiled for
#endif
template <template <int, int> class F, int G, int E>
__host__ __device__ constexpr int window_min_blocks() {
  return FSMC_WIN_MINB > 0 ? FSMC_WIN_MINB : min_blocks_for<F, G, E>();
}
template <template <int, int> class F, int G, int E, int TK, int VAR = 0>
__global__ void __launch_bounds__(kThreads, (window_min_blocks<F, G, E>())) fsm_window_kernel(Params p) {
  extern __shared__ double smem[];
  Grp<G> grp;
  // no cooperative-normal scratch: the draws are pre-generated, and the
  // shared memory left unallocated becomes L1 for the draw windows
  double* sm = smem + (threadIdx.x / G) * group_doubles(p.t);
  double* ws = nullptr;
  const long long lim = p.window - (p.t.dim + 1);
  while (true) {
    long long j = 0;
    if (grp.lane == 0) j = atomicAdd(p.next_chain, 1u);
    j = p.j_lo + grp.bcast_ll(j, 0);
    if (j >= p.j_hi) break;
    Core c;
    core_load(c, p, j);
    c.ws = ws;
    if (c.err_kind != FSMC_E_NONE) continue;
    const long long n_stop = p.mode == 0 ? p.n : (1LL << 62);
    if (c.count >= n_stop || c.tick >= p.tick_limit) continue;
    c.dw = p.draws + (size_t)j * p.window;
    c.dbase = c.ctr;
    FSMC_CHECK(!p.draw_base || c.ctr == (uint64_t)p.draw_base[j] + (uint64_t)(p.draw_round * p.draw_stride));
    c.dlim = p.window;
    F<G, E> f;
    bind_state<F<G, E>, G>(f, sm, p.t, grp);
    f.load(p, j, grp);
    bool ok = true;
    if constexpr (VAR == 1 && F<G, E>::FULLD && FSMC_WIN_NT) {
      // DRMH, default bundled order: every tick is exactly one proposal of
      // dim + 1 draws, so the window and the tick limit fix the tick count
      const long long per = G * E + 1;
      long long nt = (lim - (long long)(c.ctr - c.dbase)) / per + 1;
      nt = nt < p.tick_limit - c.tick ? nt : p.tick_limit - c.tick;
      const int left = (int)(n_stop - c.count < (1LL << 30) ? n_stop - c.count : (1LL << 30));
      const int count0 = (int)c.count;
#pragma unroll 1
      for (int t = 0; t < (int)nt && (int)c.count - count0 < left; t++)
        if (!tick<F<G, E>, G, E, TK, false, VAR>(p, c, f, sm, j, grp)) { ok = false; break; }
    } else {
#pragma unroll 1
      while (c.count < n_stop && c.tick < p.tick_limit && (long long)(c.ctr - c.dbase) <= lim)
        if (!tick<F<G, E>, G, E, TK, false, VAR>(p, c, f, sm, j, grp)) { ok = false; break; }
    }
    f.store(p, j, grp);
    if (grp.lane == 0) {
      core_store(c, p, j);
      if (!ok) report_error(c, p, j);
      else if (c.count < n_stop && c.tick < p.tick_limit) atomicAdd(p.unfinished, 1u);
      if (p.min_count) atomicMin(p.min_count, (unsigned)min(c.count, 0xfffffffeLL));
    }
  }
}

// ------------------------------------------------------------- profile
// fsm_run_kernel with clock64() timing around every block and evaluation
// (measure_block_costs, lockstep.py:454-498): the same ticks, the same
// draws; only the per-state cycle totals in p.prof are extra.
template <template <int, int> class F, int G, int E>
__global__ void __launch_bounds__(kThreads, min_blocks<G>()) fsm_profile_kernel(Params p) {
  extern __shared__ double smem[];
  Grp<G> grp;
  double* sm = group_scratch<G, E>(smem, group_doubles_f<F<G, E>, G, E>(p.t));
  double* ws = warp_scratch<G, E>(smem, group_doubles_f<F<G, E>, G, E>(p.t));
  while (true) {
    long long j = 0;
    if (grp.lane == 0) j = atomicAdd(p.next_chain, 1u);
    j = grp.bcast_ll(j, 0);
    if (j >= p.st.m) break;
    Core c;
    core_load(c, p, j);
    c.ws = ws;
    if (c.err_kind != FSMC_E_NONE) continue;
    F<G, E> f;
    bind_state<F<G, E>, G>(f, sm, p.t, grp);
    f.load(p, j, grp);
    bool ok = true;
#pragma unroll 1
    while (c.tick < p.tick_limit)
      if (!tick<F<G, E>, G, E, 0, true>(p, c, f, sm, j, grp, p.prof)) { ok = false; break; }
    f.store(p, j, grp);
    if (grp.lane == 0) {
      core_store(c, p, j);
      if (!ok) report_error(c, p, j);
    }
  }
}

// ------------------------------------------------------------- advance
// Batched-evaluation mode: every chain runs to its next log-density request
// and parks the point in the compact request list (see fsmc_advance).
template <template <int, int> class F, int G, int E, int TK = 0, bool INLINE = false>
__global__ void __launch_bounds__(kThreads, (min_blocks_for<F, G, E>())) fsm_advance_kernel(Params p) {
  extern __shared__ double smem[];
  Grp<G> grp;
  double* sm = group_scratch<G, E>(smem, group_doubles_f<F<G, E>, G, E>(p.t));
  double* ws = warp_scratch<G, E>(smem, group_doubles_f<F<G, E>, G, E>(p.t));
  while (true) {
    long long j = 0;
    if (grp.lane == 0) j = atomicAdd(p.next_chain, 1u);
    j = p.j_lo + grp.bcast_ll(j, 0);
    if (j >= p.j_hi) break;
    Core c;
    core_load(c, p, j);
    c.ws = ws;
    if (c.err_kind != FSMC_E_NONE) continue;
    F<G, E> f;
    bind_state<F<G, E>, G>(f, sm, p.t, grp);
    f.load(p, j, grp);
    long long resume = p.st.ints[(size_t)j * FSMC_NINT + FSMC_I_RESUME];
    bool ok = true;
    advance_chain<F<G, E>, G, E, TK, INLINE>(p, c, f, sm, j, grp, resume, ok);
    f.store(p, j, grp);
    if (grp.lane == 0) {
      core_store(c, p, j);
      if (p.b_level && ok) atomicMin((unsigned long long*)&p.b_level[1], (unsigned long long)c.count);
      p.st.ints[(size_t)j * FSMC_NINT + FSMC_I_RESUME] = resume;
      if (!ok) report_error(c, p, j);
    }
  }
}

// ------------------------------------------------------------ lock-step
// Grid-wide "any" + barrier.  Every thread of the (cooperatively launched,
// hence co-resident) grid calls it the same number of times.
__device__ __forceinline__ bool grid_any(const Params& p, bool pred, unsigned& phase) {
  int blk = __syncthreads_or(pred ? 1 : 0);
  if (threadIdx.x == 0) {
    if (blk) atomicOr(&p.active_flags[phase & 1], 1u);
    __threadfence();
    unsigned gen = *p.bar_gen;
    if (atomicAdd(p.bar_count, 1u) == gridDim.x - 1) {
      *p.bar_count = 0;
      p.active_flags[(phase + 1) & 1] = 0;
      __threadfence();
      atomicAdd((unsigned*)p.bar_gen, 1u);
    } else {
      while (*p.bar_gen == gen) {
      }
    }
    __threadfence();
  }
  __syncthreads();
  bool any = ((volatile unsigned*)p.active_flags)[phase & 1] != 0;
  phase++;
  return any;
}

// The lock-step baseline's synchronisation cost alone: the same cooperative
// grid as lockstep_kernel for this configuration, doing nothing but `iters`
// grid_any rounds (fsmc_lockstep_barrier_probe), so the bench can state how
// much of a lock-step step is barrier rather than sampling work.
static __global__ void __launch_bounds__(kThreads) barrier_probe_kernel(Params p, long long iters) {
  unsigned phase = 0;
  bool any = false;
#pragma unroll 1
  for (long long i = 0; i < iters; i++)
    any = grid_any(p, threadIdx.x == 0 && (long long)blockIdx.x == i % gridDim.x, phase) || any;
  if (!any && threadIdx.x == 0) p.active_flags[2] = 1u;   // never taken; keeps the loop live
}

// vmap semantics of each kernel's monolithic sampler (drmh.py:163-169,
// elliptical.py:122-132, nuts.py:237-248, slice_sampling.py:135-143): every while-loop test is a
// barrier across all chains of the wave, so a sample costs max over chains of
// its loop count.  Written as a uniform program counter so the state body
// (and its log-density evaluation) is instantiated once.
template <template <int, int> class F, int G, int E, int TK>
__global__ void __launch_bounds__(kThreads) lockstep_kernel(Params p) {
  using FF = F<G, E>;
  extern __shared__ double smem[];
  Grp<G> grp;
  double* sm = group_scratch<G, E>(smem, group_doubles_f<FF, G, E>(p.t));
  const long long j = p.wave_lo + (long long)blockIdx.x * (kThreads / G) + threadIdx.x / G;
  bool live = j < p.wave_hi;
  Core c;
  c.ws = warp_scratch<G, E>(smem, group_doubles_f<FF, G, E>(p.t));
  FF f;
  bind_state<FF, G>(f, sm, p.t, grp);
  if (live) {
    core_load(c, p, j);
    c.ws = warp_scratch<G, E>(smem, group_doubles_f<FF, G, E>(p.t));
    f.load(p, j, grp);
    live = c.err_kind == FSMC_E_NONE;
  }
  enum { PC_INIT, PC_OUTER, PC_INNER, PC_END };
  unsigned phase = 0;
#pragma unroll 1
  for (long long i = 0; i < p.n; i++) {
    if (live) { c.count = i; c.tick = i; c.pend[0] = c.pend[1] = c.pend[2] = 0; }
    int pc = PC_INIT;
    bool outer = false;
#pragma unroll 1
    while (true) {
      int s = 0;
      if (pc == PC_INIT) {
        s = 1;
        pc = PC_OUTER;
      } else if constexpr (FF::SHAPE == SHAPE_SEQ) {
        if (pc == PC_OUTER) {  // while _expand_continue(z)
          bool co = live && f.loop_continue(p);
          if (grid_any(p, co, phase)) s = co ? 2 : 0;
          else { s = 3; pc = PC_INNER; }
        } else {  // while _shrink_continue(z)
          bool ci = live && f.loop2_continue();
          if (grid_any(p, ci, phase)) s = ci ? 4 : 0;
          else { s = 5; pc = PC_END; }
        }
      } else if constexpr (FF::SHAPE == SHAPE_NESTED) {
        if (pc == PC_OUTER) {  // while _outer_continue(z)
          bool co = live && f.outer_continue(p);
          if (!grid_any(p, co, phase)) { s = 5; pc = PC_END; }
          else { outer = co; s = co ? 2 : 0; pc = PC_INNER; }
        } else {  // while _inner_continue(z)
          bool ci = outer && live && f.inner_continue();
          if (grid_any(p, ci, phase)) s = ci ? 3 : 0;
          else { s = (outer && live) ? 4 : 0; pc = PC_OUTER; }
        }
      } else {  // while _continue(z) / _below_threshold(z)
        bool co = live && f.loop_continue(p);
        if (grid_any(p, co, phase)) s = co ? 2 : 0;
        else { s = FF::K; pc = PC_END; }
      }
      // one while-loop body: PROPOSE, or the split body's states 2..K-1
      const int s_last = (s == 2 && FF::SHAPE == SHAPE_SPLIT) ? 5 : s;
#pragma unroll 1
      for (int ss = s; live && s && ss <= s_last; ss++) {
        bool did = false;
        if (!run_state<FF, G, E, TK>(p, c, f, ss, did, sm, grp)) live = false;
        count_block<FF>(c, ss);
        if (did) c.shared++;
      }
      if (pc == PC_END) break;
    }
    // per-sample loop counts were accumulated in pend by count_block
    if (live) flush_sample<FF, G, E>(p, c, f, j, grp);
  }
  if (j < p.wave_hi) {
    f.store(p, j, grp);
    if (grp.lane == 0) {
      core_store(c, p, j);
      if (c.err_kind != FSMC_E_NONE) report_error(c, p, j);
    }
  }
}

// ------------------------------------------------------------- launchers
template <template <int, int> class F, int G, int E, int TK>
struct Launch {
  static size_t smem(const Params& p) { return smem_bytes<G, E>(group_doubles_f<F<G, E>, G, E>(p.t)); }
  static cudaError_t init(const Params& p, uint64_t ps, long long off, const double* x0, double jit,
                          cudaStream_t s) {
    long long groups = (p.st.m + (kThreads / G) - 1) / (kThreads / G);
    int blocks = (int)std::min<long long>(groups, 1 << 20);
    cudaError_t e = allow_smem(fsm_init_kernel<F, G, E>, smem(p));
    if (e != cudaSuccess) return e;
    count_launch();
    fsm_init_kernel<F, G, E><<<blocks, kThreads, smem(p), s>>>(p, ps, off, x0, jit);
    return cudaGetLastError();
  }
  static cudaError_t init_finish(const Params& p, cudaStream_t s) {
    long long groups = (p.st.m + (kThreads / G) - 1) / (kThreads / G);
    int blocks = (int)std::min<long long>(groups, 1 << 20);
    count_launch();
    cudaError_t ea = allow_smem(fsm_init_finish_kernel<F, G, E>, smem(p));
    if (ea != cudaSuccess) return ea;
    fsm_init_finish_kernel<F, G, E><<<blocks, kThreads, smem(p), s>>>(p);
    return cudaGetLastError();
  }
  // a persistent chain-queue kernel with as many blocks as are co-resident
  template <class KF>
  static cudaError_t persistent(KF* kern, const Params& p, const LaunchCtx& lc, cudaStream_t s,
                                size_t sm_bytes = 0, long long chains = -1, int max_per_sm = 0) {
    const size_t sb = sm_bytes ? sm_bytes : smem(p);
    int occ = 0;
    cudaError_t e = allow_smem(kern, sb);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, sb);
    if (e != cudaSuccess) return e;
    if (max_per_sm > 0 && occ > max_per_sm) occ = max_per_sm;
    if (occ < 1) occ = 1;
    if (chains < 0) chains = p.st.m;
    long long need = (chains + (kThreads / G) - 1) / (kThreads / G);
    int blocks = (int)std::max<long long>(1, std::min<long long>(need, (long long)occ * lc.num_sms));
    count_launch();
    kern<<<blocks, kThreads, sb, s>>>(p);
    return cudaGetLastError();
  }
  static bool unrolled(const Params& p) {
    return TK != 0 && p.variant == FSMC_BUNDLED && p.default_order;
  }
  static cudaError_t run(const Params& p, const LaunchCtx& lc, cudaStream_t s) {
    if constexpr (TK != 0) {
      if (unrolled(p)) return persistent(fsm_run_kernel<F, G, E, TK, 1>, p, lc, s, 0, p.j_hi - p.j_lo);
#if FSMC_VAR2
      if (p.variant != FSMC_BUNDLED)
        return persistent(fsm_run_kernel<F, G, E, TK, 2>, p, lc, s, 0, p.j_hi - p.j_lo);
#endif
    }
    return persistent(fsm_run_kernel<F, G, E, TK, 0>, p, lc, s, 0, p.j_hi - p.j_lo);
  }
  static cudaError_t profile(const Params& p, const LaunchCtx& lc, cudaStream_t s) {
    return persistent(fsm_profile_kernel<F, G, E>, p, lc, s);
  }
  static cudaError_t window(const Params& p, const LaunchCtx& lc, cudaStream_t s) {
    const size_t sb = std::max<size_t>(8, (size_t)(kThreads / G) * group_doubles(p.t) * sizeof(double));
    if constexpr (TK != 0)
      if (unrolled(p))
        return persistent(fsm_window_kernel<F, G, E, TK, 1>, p, lc, s, sb, p.j_hi - p.j_lo, p.win_blocks_per_sm);
    return persistent(fsm_window_kernel<F, G, E, TK, 0>, p, lc, s, sb, p.j_hi - p.j_lo, p.win_blocks_per_sm);
  }
  static cudaError_t advance(const Params& p, const LaunchCtx& lc, cudaStream_t s) {
    return persistent(fsm_advance_kernel<F, G, E>, p, lc, s, 0, p.j_hi - p.j_lo);
  }
  // fsmc_advance_prior: evaluations inline, parked only at the prior transform
  static cudaError_t advance_prior(const Params& p, const LaunchCtx& lc, cudaStream_t s) {
    return persistent(fsm_advance_kernel<F, G, E, TK, true>, p, lc, s, 0, p.j_hi - p.j_lo);
  }
  // the first wave of lockstep(): same blocks, same co-residency
  static cudaError_t barrier_probe(Params p, const LaunchCtx& lc, cudaStream_t s) {
    int occ = 0;
    cudaError_t e = allow_smem(lockstep_kernel<F, G, E, TK>, smem(p));
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lockstep_kernel<F, G, E, TK>, kThreads, smem(p));
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorLaunchOutOfResources;
    const long long per_block = kThreads / G;
    const long long cap = (long long)occ * lc.num_sms * per_block;
    const long long chains = std::min<long long>(p.st.m, cap);
    int blocks = (int)((chains + per_block - 1) / per_block);
    long long iters = p.n;
    void* args[] = {&p, &iters};
    count_launch();
    return cudaLaunchCooperativeKernel((const void*)barrier_probe_kernel, dim3(blocks), dim3(kThreads), args, 0, s);
  }
  static cudaError_t lockstep(Params p, const LaunchCtx& lc, cudaStream_t s) {
    int occ = 0;
    cudaError_t e = allow_smem(lockstep_kernel<F, G, E, TK>, smem(p));
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lockstep_kernel<F, G, E, TK>,
                                                                  kThreads, smem(p));
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorLaunchOutOfResources;
    const long long per_block = kThreads / G;
    const long long cap = (long long)occ * lc.num_sms * per_block;
    for (long long lo = 0; lo < p.st.m; lo += cap) {
      p.wave_lo = lo;
      p.wave_hi = std::min<long long>(p.st.m, lo + cap);
      int blocks = (int)((p.wave_hi - lo + per_block - 1) / per_block);
      void* args[] = {&p};
      count_launch();
      e = cudaLaunchCooperativeKernel((const void*)lockstep_kernel<F, G, E, TK>, dim3(blocks),
                                      dim3(kThreads), args, smem(p), s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
};

// op: 0 init, 1 run, 2 lock-step, 3 advance, 4 profile, 7 advance with batched prior, 8 deferred-init finish, 9 lock-step barrier probe (5 windowed run and 6 draws: fam_drmh.cu).  TK: compile-time plugin (0 = run-time switch)
template <template <int, int> class F, int G, int E, int TK = 0>
cudaError_t launch_op(int op, Params& p, const LaunchCtx& lc, cudaStream_t s, uint64_t ps,
                      long long off, const double* x0, double jit) {
  if (op == 0) return Launch<F, G, E, 0>::init(p, ps, off, x0, jit, s);
  if (op == 8) return Launch<F, G, E, 0>::init_finish(p, s);
  if (op == 1) return Launch<F, G, E, TK>::run(p, lc, s);
  if (op == 3) return Launch<F, G, E, 0>::advance(p, lc, s);
  if (op == 4) return Launch<F, G, E, 0>::profile(p, lc, s);
  if (op == 7) {
    if constexpr (F<G, E>::PRIOR) return Launch<F, G, E, TK>::advance_prior(p, lc, s);
    return cudaErrorInvalidConfiguration;
  }
  if (op == 9) return Launch<F, G, E, TK>::barrier_probe(p, lc, s);
  return Launch<F, G, E, TK>::lockstep(p, lc, s);
}

}  // namespace fsmc
