// logreg_tc.cu -- fused tcgen05 evaluation of the Bayesian logistic-regression
// target across chains (BASELINE config 5).
//
// For a tile of 128 chains (rows of Theta, bf16) the CTA streams the design
// matrix in 64-row tiles and, per tile,
//   S   = Theta X_tile^T          tcgen05.mma M=128 N=64  K=256  -> TMEM (fp32)
//   R   = sigmoid(S),  sp += softplus(S)        (epilogue warps, registers)
//   G  += R X_tile                tcgen05.mma M=128 N=256 K=64   -> TMEM (fp32)
// so the [chains x N] logits never leave the SM (the flash-attention shape).
// The label terms are linear in theta and precomputed once: with c = X^T y,
//   lp = theta.c - sum softplus(z) - theta.theta/2,   grad = c - G - theta.
// Operands arrive by TMA in the canonical K-major SWIZZLE_128B layout: X
// [N][256] for the first product, X^T [256][N] for the second.  Warp roles:
//   warp 0  TMA producer of Theta and the X tiles (one elected lane)
//   warp W_XT  TMA producer of the X^T tiles (one elected lane)
//   warp 1  TMEM allocator + MMA issuer (one elected lane)
// X and X^T stages have separate full/empty barriers: an X stage is released
// as soon as the first product has read it, so X loads run ahead of the
// epilogue while X^T (needed two tiles later) streams in behind it.
//   warps 2 .. 2+4*EPI_SPLIT-1  epilogue (16 warps): TMEM lane quadrant (warp % 4) x a
//              column slice, one chain row per thread; sigmoid / softplus on
//              MUFU ex2, rcp and lg2
// S is double-buffered in TMEM so the epilogue of tile i overlaps MMA1 of i+1.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <string>

#include "../../include/fsmc.h"
#include "launch_count.h"
#include "nvtx_range.h"

namespace {

constexpr int BM = 128;       // chains per CTA (MMA M, TMEM lanes)
constexpr int BN = 64;        // design rows per tile (MMA1 N, MMA2 K)
constexpr int DF = 256;       // features (MMA1 K, MMA2 N)
constexpr int EPI_SPLIT = 4;                 // epilogue warps per TMEM lane quadrant
constexpr int N_EPI = 128 * EPI_SPLIT;        // epilogue threads
constexpr int COLS = BN / EPI_SPLIT;          // S columns per epilogue thread
constexpr int W_XT = 2 + N_EPI / 32;          // warp index of the X^T producer
constexpr int NTHREADS = 32 * (W_XT + 1);

// shared memory map (bytes from a 1024-aligned base)
constexpr uint32_t OFF_THETA = 0;                       // 4 atoms x [128 x 64] bf16 = 64 KB
constexpr uint32_t OFF_X = 64 * 1024;                   // 2 stages x 4 atoms x [64 x 64] = 2 x 32 KB
constexpr uint32_t OFF_XT = 128 * 1024;                 // 2 stages x [256 x 64] = 2 x 32 KB
constexpr uint32_t OFF_R = 192 * 1024;                  // 2 x [128 x 64] = 2 x 16 KB
constexpr uint32_t OFF_BAR = 224 * 1024;                // mbarriers + TMEM address
constexpr uint32_t SMEM_BYTES = OFF_BAR + 256 + 1024;   // + alignment slack

enum { B_FULLX0 = 0, B_EMPTYX0 = 2, B_SFULL0 = 4, B_SEMPTY0 = 6, B_RFULL0 = 8, B_REMPTY0 = 10,
       B_THETA = 12, B_GFULL = 13, B_FULLT0 = 14, B_EMPTYT0 = 16, N_BARS = 18 };

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// try_wait with a suspend-time hint: a waiting warp sleeps in the barrier
// unit instead of re-issuing its poll loop (which would steal issue slots
// from the epilogue warps sharing its scheduler)
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity), "r"(0x989680)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
// K-major, SWIZZLE_128B UMMA shared-memory descriptor (8-row atoms of 1024 B)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;             // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;   // stride byte offset: next 8-row group
  d |= (uint64_t)1 << 46;             // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;             // SWIZZLE_128B
  return d;
}
// kind::f16 instruction descriptor: 16-bit operands (format 1 = bf16, 0 =
// fp16) -> fp32 accumulator, both K-major
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N, uint32_t fmt) {
  return (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// operand element type: bf16 (8-bit mantissa) or fp16 (11-bit mantissa, the
// same issue rate; the design entries N(0,1)/sqrt(d) and sigmoid values in
// [0,1] sit well inside its range)
template <bool F16>
struct Op;
template <>
struct Op<false> {
  using T = __nv_bfloat16;
  static constexpr uint32_t fmt = 1;
  __device__ static uint32_t pack(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
  }
  __device__ static T from(float a) { return __float2bfloat16_rn(a); }
};
template <>
struct Op<true> {
  using T = __half;
  static constexpr uint32_t fmt = 0;
  __device__ static uint32_t pack(float a, float b) {
    __half2 v = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
  }
  __device__ static T from(float a) { return __float2half_rn(a); }
};
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

// 16 columns of fp32 from TMEM (this thread's lane)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; i++) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

template <bool F16>
__global__ void __launch_bounds__(NTHREADS, 1)
    logreg_tc_kernel(const __grid_constant__ CUtensorMap map_theta, const __grid_constant__ CUtensorMap map_x,
                     const __grid_constant__ CUtensorMap map_xt, const double* __restrict__ xty,
                     const double* __restrict__ theta64, long long M, long long N, double* __restrict__ lp,
                     double* __restrict__ grad) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_BAR + 8 * N_BARS);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const long long m0 = (long long)blockIdx.x * BM;
  const int T = (int)((N + BN - 1) / BN);
  auto bar = [&](int i) { return smem_u32(&bars[i]); };

  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; s++) {
      mbar_init(bar(B_FULLX0 + s), 1);
      mbar_init(bar(B_EMPTYX0 + s), 1);
      mbar_init(bar(B_FULLT0 + s), 1);
      mbar_init(bar(B_EMPTYT0 + s), 1);
      mbar_init(bar(B_SFULL0 + s), 1);
      mbar_init(bar(B_SEMPTY0 + s), N_EPI);
      mbar_init(bar(B_RFULL0 + s), N_EPI);
      mbar_init(bar(B_REMPTY0 + s), 1);
    }
    mbar_init(bar(B_THETA), 1);
    mbar_init(bar(B_GFULL), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // TMEM: 512 columns = S[0] | S[1] | G (256)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS[2] = {tmem, tmem + 64};
  const uint32_t tG = tmem + 128;

  if (warp == 0) {
    if (lane == 0) {  // ---------------------------------- TMA producer: Theta, X
      mbar_expect_tx(bar(B_THETA), BM * DF * 2);
      for (int a = 0; a < 4; a++) tma_load_2d(sbase + OFF_THETA + a * 16384, &map_theta, bar(B_THETA), a * 64, (int)m0);
      for (int i = 0; i < T; i++) {
        const int s = i & 1;
        mbar_wait(bar(B_EMPTYX0 + s), ((i >> 1) & 1) ^ 1);
        mbar_expect_tx(bar(B_FULLX0 + s), BN * DF * 2);
        for (int a = 0; a < 4; a++)
          tma_load_2d(sbase + OFF_X + s * 32768 + a * 8192, &map_x, bar(B_FULLX0 + s), a * 64, i * BN);
      }
    }
  } else if (warp == W_XT) {
    if (lane == 0) {  // ------------------------------------- TMA producer: X^T
      for (int i = 0; i < T; i++) {
        const int s = i & 1;
        mbar_wait(bar(B_EMPTYT0 + s), ((i >> 1) & 1) ^ 1);
        mbar_expect_tx(bar(B_FULLT0 + s), BN * DF * 2);
        tma_load_2d(sbase + OFF_XT + s * 32768, &map_xt, bar(B_FULLT0 + s), i * BN, 0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // --------------------------------------------- MMA issuer
      constexpr uint32_t ID1 = idesc_f16(BM, BN, Op<F16>::fmt);
      constexpr uint32_t ID2 = idesc_f16(BM, DF, Op<F16>::fmt);
      mbar_wait(bar(B_THETA), 0);
      tc_fence_after();
      auto mma2 = [&](int i) {  // G += R_i X_i  (K = 64 rows of tile i)
        const int s = i & 1;
        mbar_wait(bar(B_RFULL0 + s), (i >> 1) & 1);
        mbar_wait(bar(B_FULLT0 + s), (i >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < 4; k++)
          mma_bf16(tG, sdesc(sbase + OFF_R + s * 16384 + k * 32), sdesc(sbase + OFF_XT + s * 32768 + k * 32), ID2,
                   (i > 0 || k > 0) ? 1u : 0u);
        mma_commit(bar(B_REMPTY0 + s));
        mma_commit(bar(B_EMPTYT0 + s));
      };
      for (int i = 0; i < T; i++) {
        const int s = i & 1;
        mbar_wait(bar(B_FULLX0 + s), (i >> 1) & 1);
        mbar_wait(bar(B_SEMPTY0 + s), ((i >> 1) & 1) ^ 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < 16; k++) {  // S_i = Theta X_i^T, K = 256 in 4 atoms of 64
          const int a = k >> 2, kk = k & 3;
          mma_bf16(tS[s], sdesc(sbase + OFF_THETA + a * 16384 + kk * 32),
                   sdesc(sbase + OFF_X + s * 32768 + a * 8192 + kk * 32), ID1, k > 0 ? 1u : 0u);
        }
        mma_commit(bar(B_SFULL0 + s));
        mma_commit(bar(B_EMPTYX0 + s));
        if (i > 0) mma2(i - 1);
      }
      mma2(T - 1);
      mma_commit(bar(B_GFULL));
    }
  } else if (warp >= 2 && warp < W_XT) {  // ---------------------------- epilogue
    const int quad = warp & 3;            // TMEM lanes 32*quad .. 32*quad+31
    const int half = (warp - 2) >> 2;     // columns COLS*half .. COLS*half+COLS-1 of each S tile
    const int row = quad * 32 + lane;     // chain within the tile
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    double lp_acc = 0.0;
    for (int i = 0; i < T; i++) {
      const int s = i & 1;
      mbar_wait(bar(B_SFULL0 + s), (i >> 1) & 1);
      tc_fence_after();
      float z[COLS];
#pragma unroll
      for (int q = 0; q < COLS; q += 16) tmem_ld16(tS[s] + lane_off + half * COLS + q, z + q);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(bar(B_SEMPTY0 + s));
      // R = sigmoid(z) = 1 / (1 + e^-z);  sp += log(1 + e^z) = z + ln(1 + e^-z).
      // One exponential shared by both (z clamped at -87 keeps e^-z finite in
      // fp32; below that softplus < 1e-37), no sign select: 7 instructions
      // per element, the epilogue being issue-bound.  The validity test
      // (design rows past N) only runs on the last tile.
      uint32_t packed[COLS / 2];
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      const long long r0 = (long long)i * BN + half * COLS;
      const int valid = r0 + COLS <= N ? COLS : (int)(N > r0 ? N - r0 : 0);
#ifndef FSMC_SP_POLY
#define FSMC_SP_POLY 0
#endif
#if FSMC_SP_POLY
      // two MUFU operations per element (ex2, rcp) instead of three: with
      // e = 2^(-|z| log2 e) in (0, 1], softplus(z) = max(z, 0) + log1p(e) with
      // log1p on the FMA pipe (degree-8 minimax-like fit of log1p(e)/e on [0, 1],
      // |error| < 2e-7, mean bias 1e-8), sigmoid(z) = r or 1 - r, r = 1/(1 + e).
      // The epilogue was MUFU-bound (3 ops x 8192 elements per tile against
      // the tile's ~1100 tensor cycles); now MUFU and tensor balance.
      auto element = [&](float zz, float& sig) -> float {
        float en, r;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(en) : "f"(-1.4426950408889634f * fabsf(zz)));
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + en));
        sig = zz >= 0.0f ? r : 1.0f - r;
        float q = 5.186003710e-03f;
        q = fmaf(q, en, -2.921026794e-02f);
        q = fmaf(q, en, 7.754038125e-02f);
        q = fmaf(q, en, -1.358394190e-01f);
        q = fmaf(q, en, 1.905595565e-01f);
        q = fmaf(q, en, -2.482564859e-01f);
        q = fmaf(q, en, 3.331601067e-01f);
        q = fmaf(q, en, -4.999925590e-01f);
        q = fmaf(q, en, 9.999999209e-01f);
        return fmaf(q, en, fmaxf(zz, 0.0f));
      };
#else
      auto element = [&](float zz, float& sig) -> float {
        const float zc = fmaxf(zz, -87.0f);
        float en, l2;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(en) : "f"(-1.4426950408889634f * zc));
        const float ope = 1.0f + en;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(sig) : "f"(ope));
        asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l2) : "f"(ope));
        return fmaf(0.6931471805599453f, l2, zc);
      };
#endif
      if (valid == COLS) {
#pragma unroll
        for (int c = 0; c < COLS; c += 2) {
          float rv[2];
#pragma unroll
          for (int h = 0; h < 2; h++) acc[(c + h) & 3] += element(z[c + h], rv[h]);
          packed[c >> 1] = Op<F16>::pack(rv[0], rv[1]);
        }
      } else {
#pragma unroll
        for (int c = 0; c < COLS; c += 2) {
          float rv[2];
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const float sp = element(z[c + h], rv[h]);
            acc[(c + h) & 3] += (c + h) < valid ? sp : 0.0f;   // rows past N have x = 0: no G term
          }
          packed[c >> 1] = Op<F16>::pack(rv[0], rv[1]);
        }
      }
      lp_acc += (double)((acc[0] + acc[1]) + (acc[2] + acc[3]));
      mbar_wait(bar(B_REMPTY0 + s), ((i >> 1) & 1) ^ 1);
      uint8_t* rbase = smem + OFF_R + s * 16384 + (row >> 3) * 1024 + (row & 7) * 128;
#pragma unroll
      for (int q = 0; q < COLS / 8; q++) {  // this warp's 16-B chunks of the 128-B row, SWIZZLE_128B
        const int ch = half * (COLS / 8) + q;
        uint4 v = make_uint4(packed[q * 4], packed[q * 4 + 1], packed[q * 4 + 2], packed[q * 4 + 3]);
        *reinterpret_cast<uint4*>(rbase + ((ch ^ (row & 7)) << 4)) = v;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(bar(B_RFULL0 + s));
    }
    // G = sigmoid(S) X summed over every tile:
    //   grad = c - G - theta,  lp = theta.c - sum softplus - theta.theta / 2
    double* lp_x = reinterpret_cast<double*>(smem + OFF_R);   // R buffers are free now
    mbar_wait(bar(B_GFULL), 0);
    tc_fence_after();
    const long long chain = m0 + row;
    double part = -lp_acc;
#pragma unroll 1
    for (int c = half * (DF / EPI_SPLIT); c < (half + 1) * (DF / EPI_SPLIT); c += 16) {
      float g[16];
      tmem_ld16(tG + lane_off + c, g);
      tmem_wait_ld();
      if (chain < M) {
#pragma unroll
        for (int q = 0; q < 16; q++) {
          const double th = theta64[chain * DF + c + q];
          const double cy = __ldg(&xty[c + q]);
          part += th * cy - 0.5 * (th * th);
          grad[chain * DF + c + q] = (cy - (double)g[q]) - th;
        }
      }
    }
    if (half > 0) lp_x[(half - 1) * BM + row] = part;
    asm volatile("bar.sync 1, %0;" ::"n"(N_EPI));
    if (half == 0 && chain < M) {
#pragma unroll
      for (int h = 1; h < EPI_SPLIT; h++) part += lp_x[(h - 1) * BM + row];
      lp[chain] = part;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// fp64 chain positions -> 16-bit rows (padded to a multiple of 128 with zeros)
template <bool F16>
__global__ void to_half_kernel(const double* __restrict__ src, long long rows, long long rows_pad,
                               typename Op<F16>::T* __restrict__ dst) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= rows_pad * DF) return;
  dst[i] = Op<F16>::from(i < rows * DF ? (float)src[i] : 0.0f);
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encoder() {
  static EncodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
  }
  return fn;
}

// 2-D 16-bit tensor [rows][cols] (row-major), box [box_rows][64 cols], SWIZZLE_128B
bool make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows, bool f16) {
  EncodeTiled enc = encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

thread_local std::string g_err;

}  // namespace

extern "C" {

const char* fsmc_logreg_tc_last_error(void) { return g_err.c_str(); }

/* Fused tcgen05 logistic-regression evaluation (see fsmc.h).  operand: 0 =
 * bf16, 1 = fp16 (theta_h16 / x_h16 / xt_h16 then hold that type). */
fsmc_status fsmc_logreg_tc_eval2(const double* theta, int64_t k, void* theta_h16, const void* x_h16,
                                 const void* xt_h16, const double* xty, int64_t n_obs, int64_t dim, double* lp,
                                 double* grad, int32_t operand, void* stream_) {
  FSMC_NVTX("fsmc_logreg_tc_eval2");
  if (dim != DF) { g_err = "fused logistic-regression kernel is compiled for d = 256"; return FSMC_ERR_UNSUPPORTED; }
  if (!theta || !theta_h16 || !x_h16 || !xt_h16 || !xty || !lp || !grad || k < 0 || n_obs < 1 ||
      (operand != 0 && operand != 1)) {
    g_err = "bad arguments";
    return FSMC_ERR_ARG;
  }
  if (!k) return FSMC_OK;
  const bool f16 = operand == 1;
  cudaStream_t s = (cudaStream_t)stream_;
  const long long kpad = (k + BM - 1) / BM * BM;
  fsmc::count_launch(2);   // the conversion and logreg_tc_kernel
  const unsigned cb = (unsigned)((kpad * DF + 255) / 256);
  if (f16) to_half_kernel<true><<<cb, 256, 0, s>>>(theta, k, kpad, (__half*)theta_h16);
  else to_half_kernel<false><<<cb, 256, 0, s>>>(theta, k, kpad, (__nv_bfloat16*)theta_h16);
  CUtensorMap mt, mx, mxt;
  if (!make_map(&mt, theta_h16, kpad, DF, BM, f16) || !make_map(&mx, x_h16, n_obs, DF, BN, f16) ||
      !make_map(&mxt, xt_h16, DF, n_obs, DF, f16)) {
    g_err = "cuTensorMapEncodeTiled failed (alignment: n_obs must be a multiple of 8)";
    return FSMC_ERR_ARG;
  }
  // the shared-memory opt-in is a per-device function attribute
  static bool attr[2][64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  auto kern = f16 ? logreg_tc_kernel<true> : logreg_tc_kernel<false>;
  if (dev < 0 || dev >= 64 || !attr[f16][dev]) {
    cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (ea != cudaSuccess) { g_err = cudaGetErrorString(ea); return FSMC_ERR_CUDA; }
    if (dev >= 0 && dev < 64) attr[f16][dev] = true;
  }
  kern<<<(unsigned)(kpad / BM), NTHREADS, SMEM_BYTES, s>>>(mt, mx, mxt, xty, theta, k, n_obs, lp, grad);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { g_err = cudaGetErrorString(e); return FSMC_ERR_CUDA; }
  return FSMC_OK;
}

fsmc_status fsmc_logreg_tc_eval(const double* theta, int64_t k, void* theta_bf16, const void* x_bf16,
                                const void* xt_bf16, const double* xty, int64_t n_obs, int64_t dim, double* lp,
                                double* grad, void* stream_) {
  return fsmc_logreg_tc_eval2(theta, k, theta_bf16, x_bf16, xt_bf16, xty, n_obs, dim, lp, grad, 0, stream_);
}

}  // extern "C"
