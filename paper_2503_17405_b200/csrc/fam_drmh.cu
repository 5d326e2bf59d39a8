// fam_drmh.cu -- Drmh kernels for the compiled (lanes, elements) pairs.
#include "kernels.cuh"

namespace fsmc {

// The DRMH draw pattern (drmh.py:85-88): from the chain's draw origin on,
// every group of dim + 1 counters is dim normals then one uniform.  One warp
// fills one chain's window at a time (coalesced 256 B stores): uniforms and
// central-branch normals directly, tail-branch normals through a per-warp
// queue evaluated with every lane busy (the compaction of normal_vec).
constexpr int kDrawChunk = 256;   // window slots per warp pass (tail-queue capacity)
__global__ void __launch_bounds__(256) drmh_draws_kernel(Params p) {
  __shared__ double qy_all[8][kDrawChunk];
  __shared__ unsigned qk_all[8][kDrawChunk];
  const int nw = blockDim.x >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int W = (int)p.window, d = p.t.dim, per = d + 1;
  double* qy = qy_all[wid];
  unsigned* qk = qk_all[wid];
  const unsigned lt = (1u << lane) - 1u;
  const int step = 32 % per;             // phase advance between a lane's slots
  const long long n_stop = p.mode == 0 ? p.n : (1LL << 62);
  for (long long j = p.j_lo + (long long)blockIdx.x * nw + wid; j < p.j_hi; j += (long long)gridDim.x * nw) {
    const int64_t* q = p.st.ints + (size_t)j * FSMC_NINT;
    if (q[FSMC_I_ERR_KIND] != FSMC_E_NONE || q[FSMC_I_COUNT] >= n_stop || q[FSMC_I_TICK] >= p.tick_limit)
      continue;
    // pipelined windows: the counter this window starts at is known up front
    const uint64_t ctr0 = p.draw_base ? (uint64_t)p.draw_base[j] + (uint64_t)(p.draw_round * p.draw_stride)
                                      : (uint64_t)q[FSMC_I_COUNTER];
    const uint64_t hsc = hash_seed_stream(p.st.seed, (uint64_t)q[FSMC_I_STREAM]);
    int phase = (int)((ctr0 - (uint64_t)q[FSMC_I_DRAW0]) % (uint64_t)per) + lane % per;
    if (phase >= per) phase -= per;
    double* out = p.draws + (size_t)j * W;
    for (int c0 = 0; c0 < W; c0 += kDrawChunk) {
      const int c1 = min(W, c0 + kDrawChunk);
      int nt = 0;
#pragma unroll 4
      for (int k0 = c0; k0 < c1; k0 += 32) {
        // branch-free: every lane evaluates the central branch (uniform and
        // tail lanes discard it), so the warp never splits three ways
        const int k = k0 + lane;
        const bool live = k < c1;
        const double bd = (double)(bits(hsc, ctr0 + (uint64_t)k) >> 11);
        const bool uni = phase == d;
        bool neg;
        double yr;
        const bool central = ndtri_classify((bd + 0.5) * INV_2_53, &yr, &neg);  // prng.py:103-111
        const double vc = ndtri_central(yr);
        const double v = uni ? bd * INV_2_53 : vc;                               // prng.py:97-100
        const bool tail = live && !uni && !central;
        if (live && !tail) out[k] = v;
        phase += step;
        phase = phase >= per ? phase - per : phase;
        const unsigned bt = __ballot_sync(0xffffffffu, tail);
        if (tail) {
          const int pos = nt + __popc(bt & lt);
          qy[pos] = yr;
          qk[pos] = (unsigned)k | (neg ? 0x80000000u : 0u);
        }
        nt += __popc(bt);
      }
      __syncwarp();
      for (int t = lane; t < nt; t += 32) {
        const unsigned kk = qk[t];
        out[kk & 0x7fffffffu] = ndtri_tail(qy[t], (kk >> 31) != 0);
      }
      __syncwarp();
    }
  }
}

// The same window fill with U slots per lane per pass: the U raw draws, their
// classification and their central-branch polynomials are straight-line code
// (the branch-free division), so U independent dependency chains interleave;
// the tail queue is then fed once per pass.  Bit-identical to the kernel above.
#ifndef FSMC_GEN_U
#define FSMC_GEN_U 4
#endif
#ifndef FSMC_GEN_PIPE
#define FSMC_GEN_PIPE 0
#endif
// register budget: ptxas's default for (256) threads (64 registers) measured
// fastest; FSMC_GEN_MINB > 0 forces a minimum number of resident blocks
#ifndef FSMC_GEN_MINB
#define FSMC_GEN_MINB 0
#endif
#if FSMC_GEN_MINB > 0
#define FSMC_GEN_BOUNDS __launch_bounds__(256, FSMC_GEN_MINB)
#else
#define FSMC_GEN_BOUNDS __launch_bounds__(256)
#endif
template <int U>
__global__ void FSMC_GEN_BOUNDS drmh_draws_ilp_kernel(Params p) {
  __shared__ double qy_all[8][kDrawChunk];
  __shared__ unsigned qk_all[8][kDrawChunk];
  const int nw = blockDim.x >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int W = (int)p.window, d = p.t.dim, per = d + 1;
  double* qy = qy_all[wid];
  unsigned* qk = qk_all[wid];
  const unsigned lt = (1u << lane) - 1u;
  const int step = 32 % per;             // phase advance between a lane's slots
  const long long n_stop = p.mode == 0 ? p.n : (1LL << 62);
  for (long long j = p.j_lo + (long long)blockIdx.x * nw + wid; j < p.j_hi; j += (long long)gridDim.x * nw) {
    const int64_t* q = p.st.ints + (size_t)j * FSMC_NINT;
    if (q[FSMC_I_ERR_KIND] != FSMC_E_NONE || q[FSMC_I_COUNT] >= n_stop || q[FSMC_I_TICK] >= p.tick_limit)
      continue;
    // pipelined windows: the counter this window starts at is known up front
    const uint64_t ctr0 = p.draw_base ? (uint64_t)p.draw_base[j] + (uint64_t)(p.draw_round * p.draw_stride)
                                      : (uint64_t)q[FSMC_I_COUNTER];
    const uint64_t hsc = hash_seed_stream(p.st.seed, (uint64_t)q[FSMC_I_STREAM]);
    int phase = (int)((ctr0 - (uint64_t)q[FSMC_I_DRAW0]) % (uint64_t)per) + lane % per;
    if (phase >= per) phase -= per;
    double* out = p.draws + (size_t)j * W;
#if FSMC_GEN_PIPE
    // software-pipelined: the next pass's integer hashes are computed in the
    // same basic block as this pass's fp64 polynomials, so one warp's
    // instruction stream mixes the integer and fp64 pipes
    uint64_t hb[U];
#pragma unroll
    for (int u = 0; u < U; u++) hb[u] = bits(hsc, ctr0 + (uint64_t)(32 * u + lane)) >> 11;
#endif
    for (int c0 = 0; c0 < W; c0 += kDrawChunk) {
      const int c1 = min(W, c0 + kDrawChunk);
      int nt = 0;
      for (int k0 = c0; k0 < c1; k0 += 32 * U) {
        double bd[U], yr[U], vc[U];
        bool neg[U], cen[U], uni[U];
#if FSMC_GEN_PIPE
#pragma unroll
        for (int u = 0; u < U; u++) {
          bd[u] = (double)hb[u];
          uni[u] = phase == d;
          phase += step;
          phase = phase >= per ? phase - per : phase;
        }
        // next pass (k0 + 32U; past the window end the values are unused)
#pragma unroll
        for (int u = 0; u < U; u++)
          hb[u] = bits(hsc, ctr0 + (uint64_t)(k0 + 32 * (U + u) + lane)) >> 11;
#else
#pragma unroll
        for (int u = 0; u < U; u++) {   // prng.py:58-81, 103-111
          bd[u] = (double)(bits(hsc, ctr0 + (uint64_t)(k0 + 32 * u + lane)) >> 11);
          uni[u] = phase == d;
          phase += step;
          phase = phase >= per ? phase - per : phase;
        }
#endif
#pragma unroll
        for (int u = 0; u < U; u++) cen[u] = ndtri_classify((bd[u] + 0.5) * INV_2_53, &yr[u], &neg[u]);
#pragma unroll
        for (int u = 0; u < U; u++) vc[u] = ndtri_central_sl(yr[u]);
#pragma unroll
        for (int u = 0; u < U; u++) {
          const int k = k0 + 32 * u + lane;
          const bool live = k < c1;
          const double v = uni[u] ? bd[u] * INV_2_53 : vc[u];     // prng.py:97-100
          const bool tail = live && !uni[u] && !cen[u];
          FSMC_CHECK(!live || k < W);
          if (live && !tail) out[k] = v;
          const unsigned bt = __ballot_sync(0xffffffffu, tail);
          if (tail) {
            const int pos = nt + __popc(bt & lt);
            qy[pos] = yr[u];
            qk[pos] = (unsigned)k | (neg[u] ? 0x80000000u : 0u);
          }
          nt += __popc(bt);
        }
      }
      __syncwarp();
      // the queue two items per lane at a time (straight-line tail: the two
      // dependency chains interleave); a chunk holds ~63 tails, so one pass
#ifndef FSMC_TAIL_SL
#define FSMC_TAIL_SL 2
#endif
      if (FSMC_TAIL_SL != 1) {
        for (int t = lane; t < nt; t += 32) {
          const unsigned kk = qk[t];
          FSMC_CHECK((int)(kk & 0x7fffffffu) < W && nt <= kDrawChunk);
          out[kk & 0x7fffffffu] = FSMC_TAIL_SL == 2 ? ndtri_tail_sl(qy[t], (kk >> 31) != 0)
                                                    : ndtri_tail(qy[t], (kk >> 31) != 0);
        }
      } else
      for (int t = lane; t < nt; t += 64) {
        const int t2 = t + 32 < nt ? t + 32 : t;
        const unsigned k1 = qk[t], k2 = qk[t2];
        const double v1 = ndtri_tail_sl(qy[t], (k1 >> 31) != 0);
        const double v2 = ndtri_tail_sl(qy[t2], (k2 >> 31) != 0);
        out[k1 & 0x7fffffffu] = v1;
        out[k2 & 0x7fffffffu] = v2;
      }
      __syncwarp();
    }
  }
}

// The window fill with the central branch compacted as well: U slots per lane
// per pass are hashed and classified; uniforms are stored at once, central
// and tail items go to two per-warp queues.  The central queue is a 256-entry
// ring carried across chunks and drained 32U items at a time (U polynomials
// per lane, straight-line), so no lane evaluates a polynomial whose result it
// discards (a uniform or a tail slot: a third of the slots); the remainder is
// drained once at the window's end.  Bit-identical to the kernels above.
#ifndef FSMC_GEN_CQ
#define FSMC_GEN_CQ 0
#endif
template <int U>
__global__ void FSMC_GEN_BOUNDS drmh_draws_cq_kernel(Params p) {
  static_assert(32 * U <= 128, "ring holds at most 127 carried + 32U new items");
  __shared__ double qy_all[8][kDrawChunk];
  __shared__ unsigned qk_all[8][kDrawChunk];
  __shared__ double cy_all[8][256];
  __shared__ unsigned ck_all[8][256];
  const int nw = blockDim.x >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int W = (int)p.window, d = p.t.dim, per = d + 1;
  double* qy = qy_all[wid];
  unsigned* qk = qk_all[wid];
  double* cy = cy_all[wid];
  unsigned* ck = ck_all[wid];
  const unsigned lt = (1u << lane) - 1u;
  const int step = 32 % per;
  const long long n_stop = p.mode == 0 ? p.n : (1LL << 62);
  for (long long j = p.j_lo + (long long)blockIdx.x * nw + wid; j < p.j_hi; j += (long long)gridDim.x * nw) {
    const int64_t* q = p.st.ints + (size_t)j * FSMC_NINT;
    if (q[FSMC_I_ERR_KIND] != FSMC_E_NONE || q[FSMC_I_COUNT] >= n_stop || q[FSMC_I_TICK] >= p.tick_limit)
      continue;
    const uint64_t ctr0 = p.draw_base ? (uint64_t)p.draw_base[j] + (uint64_t)(p.draw_round * p.draw_stride)
                                      : (uint64_t)q[FSMC_I_COUNTER];
    const uint64_t hsc = hash_seed_stream(p.st.seed, (uint64_t)q[FSMC_I_STREAM]);
    int phase = (int)((ctr0 - (uint64_t)q[FSMC_I_DRAW0]) % (uint64_t)per) + lane % per;
    if (phase >= per) phase -= per;
    double* out = p.draws + (size_t)j * W;
    unsigned chead = 0, ctail = 0;   // central ring [chead, ctail) (mod 256)
    // U central polynomials per lane from the ring head; `all`: a partial
    // batch (lanes past the tail compute on a dummy and store nothing)
    auto drain = [&](bool all) {
      double yv[U], rv[U];
      unsigned kv[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const unsigned t = chead + (unsigned)(32 * u + lane);
        const bool has = !all || t < ctail;
        yv[u] = has ? cy[t & 255u] : 0.75;
        kv[u] = has ? ck[t & 255u] : 0xffffffffu;
      }
#pragma unroll
      for (int u = 0; u < U; u++) rv[u] = ndtri_central_sl(yv[u]);
#pragma unroll
      for (int u = 0; u < U; u++)
        if (kv[u] != 0xffffffffu) {
          FSMC_CHECK((int)kv[u] < W);
          out[kv[u]] = rv[u];
        }
      chead = all ? ctail : chead + 32u * U;
    };
    for (int c0 = 0; c0 < W; c0 += kDrawChunk) {
      const int c1 = min(W, c0 + kDrawChunk);
      int nt = 0;
      for (int k0 = c0; k0 < c1; k0 += 32 * U) {
        double bd[U], yr[U];
        bool neg[U], cen[U], uni[U];
#pragma unroll
        for (int u = 0; u < U; u++) {   // prng.py:58-81, 103-111
          bd[u] = (double)(bits(hsc, ctr0 + (uint64_t)(k0 + 32 * u + lane)) >> 11);
          uni[u] = phase == d;
          phase += step;
          phase = phase >= per ? phase - per : phase;
        }
#pragma unroll
        for (int u = 0; u < U; u++) cen[u] = ndtri_classify((bd[u] + 0.5) * INV_2_53, &yr[u], &neg[u]);
#pragma unroll
        for (int u = 0; u < U; u++) {
          const int k = k0 + 32 * u + lane;
          const bool live = k < c1;
          if (live && uni[u]) out[k] = bd[u] * INV_2_53;       // prng.py:97-100
          const bool cn = live && !uni[u] && cen[u];
          const bool tl = live && !uni[u] && !cen[u];
          const unsigned bc = __ballot_sync(0xffffffffu, cn);
          const unsigned bt = __ballot_sync(0xffffffffu, tl);
          if (cn) {
            const unsigned pos = (ctail + __popc(bc & lt)) & 255u;
            cy[pos] = yr[u];
            ck[pos] = (unsigned)k;
          }
          if (tl) {
            const int pos = nt + __popc(bt & lt);
            qy[pos] = yr[u];
            qk[pos] = (unsigned)k | (neg[u] ? 0x80000000u : 0u);
          }
          ctail += __popc(bc);
          nt += __popc(bt);
        }
        __syncwarp();
        if (ctail - chead >= 32u * U) {
          drain(false);
          __syncwarp();
        }
      }
      for (int t = lane; t < nt; t += 32) {
        const unsigned kk = qk[t];
        FSMC_CHECK((int)(kk & 0x7fffffffu) < W && nt <= kDrawChunk);
        out[kk & 0x7fffffffu] = ndtri_tail_sl(qy[t], (kk >> 31) != 0);
      }
      __syncwarp();
    }
    while (ctail != chead) {   // the window's remainder
      drain(true);
      __syncwarp();
    }
  }
}

static cudaError_t launch_drmh_draws(const Params& p, int num_sms, cudaStream_t s) {
  const int threads = 256, nw = threads / 32;
  long long need = (p.j_hi - p.j_lo + nw - 1) / nw;
  const int per_sm = p.draw_blocks_per_sm > 0 ? p.draw_blocks_per_sm : 8;
  int blocks = (int)std::max<long long>(1, std::min<long long>(need, (long long)num_sms * per_sm));
  count_launch();
  if (FSMC_GEN_CQ) drmh_draws_cq_kernel<FSMC_GEN_U><<<blocks, threads, 0, s>>>(p);
  else if (FSMC_GEN_U > 1) drmh_draws_ilp_kernel<FSMC_GEN_U><<<blocks, threads, 0, s>>>(p);
  else drmh_draws_kernel<<<blocks, threads, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t dispatch_drmh(int op, int g, int e, Params& p, const LaunchCtx& lc, cudaStream_t s,
                           uint64_t ps, long long off, const double* x0, double jit) {
  // the compile-time MoG kernels unroll FSMC_MOG_SPECIAL_MODES modes: more
  // modes run on the run-time plugin switch
  const int kind = (p.t.kind == FSMC_T_MOG && p.t.n_modes > FSMC_MOG_SPECIAL_MODES) ? -1 : p.t.kind;
  if (op == 6) return launch_drmh_draws(p, lc.num_sms, s);
  if (p.k.precision == 1 && !p.k.split_body) {   // fp32 throughput mode: the sampling runs only
#define F(GG, EE, TK)                                                                \
  if (g == GG && e == EE && kind == TK) {                                            \
    if (op == 5) return Launch<DrmhWF, GG, EE, TK>::window(p, lc, s);                \
    if (op == 1) return Launch<DrmhF, GG, EE, TK>::run(p, lc, s);                    \
  }
    FSMC_DRMH_F32(F)
#undef F
    if (op == 1 || op == 5) return cudaErrorNotSupported;
  }
  if (op == 5) {  // windowed run: the DR = true families
    if (p.k.split_body) {
#define X(GG, EE) \
  if (g == GG && e == EE) return Launch<DrmhSplitW, GG, EE, 0>::window(p, lc, s);
      FSMC_DRMH_SPLIT_CONFIGS(X)
#undef X
      return cudaErrorInvalidConfiguration;
    }
    // the benchmark plugins at their exact dimension (G * E): guard-free kernels
#define S(GG, EE, TK)                                                                 \
  if (g == GG && e == EE && kind == TK) {                                             \
    if (p.t.dim == GG * EE) return Launch<DrmhWX, GG, EE, TK>::window(p, lc, s);      \
    return Launch<DrmhW, GG, EE, TK>::window(p, lc, s);                               \
  }
    FSMC_DRMH_SPECIAL(S)
#undef S
#define X(GG, EE) \
  if (g == GG && e == EE) return Launch<DrmhW, GG, EE, 0>::window(p, lc, s);
    FSMC_DRMH_CONFIGS(X)
#undef X
    return cudaErrorInvalidConfiguration;
  }
  if (p.k.split_body) {
#define X(GG, EE) \
  if (g == GG && e == EE) return launch_op<DrmhSplit, GG, EE>(op, p, lc, s, ps, off, x0, jit);
    FSMC_DRMH_SPLIT_CONFIGS(X)
#undef X
    return cudaErrorInvalidConfiguration;
  }
#define S(GG, EE, TK)                                                                            \
  if (g == GG && e == EE && kind == TK) {                                                        \
    if (op == 1 && p.t.dim == GG * EE) return Launch<DrmhX, GG, EE, TK>::run(p, lc, s);          \
    return launch_op<Drmh, GG, EE, TK>(op, p, lc, s, ps, off, x0, jit);                          \
  }
  if (op != 0) {
    FSMC_DRMH_SPECIAL(S)
  }
#undef S
#define X(GG, EE) \
  if (g == GG && e == EE) return launch_op<Drmh, GG, EE>(op, p, lc, s, ps, off, x0, jit);
  FSMC_DRMH_CONFIGS(X)
#undef X
  return cudaErrorInvalidConfiguration;
}
}  // namespace fsmc
