// gp_chol.cu -- batched marginal likelihood of the GP-hyperparameter target
// (targets.py:191-265) for designs too large for the per-chain shared-memory
// plugin: the paper's section 7.2 workload (n = 414 observations).
//
// One CTA per requesting chain (grid-stride over the request list).  For
// theta = (sigma, tau, lam):
//   K = tau^2 exp(-lam^2 D2) + (sigma^2 + jitter) I,   K = L L^T,
//   lml = -|L^-1 y|^2 / 2 - sum log L_ii - n log(2 pi) / 2
// K is never stored: a left-looking blocked Cholesky (block columns of 32)
// forms each block column's entries of K from D2 on the fly and subtracts
// the already-factored columns,
//   C[i][t] = K(i, kb+t) - sum_{s<kb} L[i][s] L[kb+t][s]      (a GEMM, DFMA)
// then factors the 32 x 32 diagonal block (one warp), solves the panel
// below it, and writes the block column of L once, column-major, to the
// CTA's workspace slot (coalesced; read back by later block columns, L2
// resident).  The forward solve L v = y rides along block by block.
//
// Values agree with LAPACK's dpotrf/dpotrs (the reference's cho_factor /
// cho_solve) to rounding: a different summation order, no bit parity.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <string>

#include "../../include/fsmc.h"
#include "launch_count.h"
#include "nvtx_range.h"

namespace {

constexpr int NB = 32;                 // block-column width
constexpr int THREADS = 256;
constexpr int RS = THREADS / 4;        // row slots: thread (r, q) owns rows r + RS p, columns 8q .. 8q+7
constexpr int MAXP = 7;                // rows per thread per pass (RS * MAXP = 448 rows)
constexpr int LDC = NB + 1;
constexpr double LOG_2PI = 1.8378770664093454836;
constexpr unsigned long long FAILURE_BITS = 0x7ff80000dead0001ULL;   // fsm_device.cuh

std::string g_err;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double block_sum(double v, double* red8) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red8[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < THREADS / 32; w++) s += red8[w];
  return s;
}

// The gradient (targets.py:238-254): with A = alpha alpha^T - K^-1,
//   d_sigma = sigma tr(A),  d_tau = tau sum(A o E),  d_lam = -lam tau^2 sum(A o E o D2)
// from the factor L the value pass left in the CTA's workspace slot
// (column-major, lower) and v = L^-1 y (shared memory):
//   alpha = L^-T v                      back substitution, one row of L per step
//   W = L^-1                            right-looking: row k final, then a rank-1
//                                       update of the rows below; W stored
//                                       transposed in the slot's free upper half
//   E = exp(-lam^2 D2)                  over the lower half (L is no longer needed)
//   tr(K^-1 M) = sum_k w_k^T M w_k      w_k the rows of W, M = E and E o D2
// n^3/6 + 2 n^3/3 operations on top of the factorization; no library call.
__device__ void gp_gradient(double* __restrict__ Lc, const double* __restrict__ d2, int n,
                            double sg, double tau, double lam, double jitter, double* __restrict__ v,
                            double* __restrict__ sm, double* __restrict__ g) {
  const int tid = threadIdx.x;
  double* alpha = v;                 // in place
  double* wd = sm;                   // [n] diagonal of W = 1 / L_kk
  double* wr = sm + n;               // [n] the current row of W
  double* red8 = sm + 2 * n;         // [8] block-reduction scratch
  // alpha = L^-T v: i from n-1 down; v_k -= L_ik alpha_i for k < i (row i of L)
  for (int i = n - 1; i >= 0; i--) {
    __syncthreads();
    const double ai = alpha[i] / Lc[(size_t)i * n + i];
    __syncthreads();
    if (tid == 0) alpha[i] = ai;
    for (int kk = tid; kk < i; kk += THREADS) alpha[kk] -= Lc[(size_t)kk * n + i] * ai;
  }
  __syncthreads();
  for (int i = tid; i < n; i += THREADS) wd[i] = 1.0 / Lc[(size_t)i * n + i];
  // W = L^-1, W_ij (i > j) at Lc[i * n + j]; start from -L_ij / L_jj... right-looking:
  // row k of W is final once rows < k are applied: W_kj = (-sum_{m<k} L_km W_mj) / L_kk
  // with the update W_ij -= L_ik W_kj (i > k) done as soon as row k is final.
  for (int e = tid; e < n * n; e += THREADS) {      // clear the upper half (the W^T area)
    const int col = e / n, row = e - col * n;
    if (row < col) Lc[(size_t)col * n + row] = 0.0;
  }
  __syncthreads();
  for (int kr = 0; kr < n; kr++) {
    // row kr: entries j < kr hold -sum_{m<kr} L_km W_mj so far; divide by L_kk
    for (int j = tid; j < kr; j += THREADS) Lc[(size_t)kr * n + j] *= wd[kr];
    __syncthreads();
    // rank-1 update of rows i > kr with column kr of L and row kr of W (j <= kr)
    const int rows = n - kr - 1, cols = kr + 1;
    for (int e = tid; e < rows * cols; e += THREADS) {
      const int ii = e / cols, j = e - ii * cols, i = kr + 1 + ii;
      const double wkj = j == kr ? wd[kr] : Lc[(size_t)kr * n + j];
      Lc[(size_t)i * n + j] -= Lc[(size_t)kr * n + i] * wkj;   // L_i,kr at column kr, row i
    }
    __syncthreads();
  }
  // E over the lower half (diagonal included); alpha^T E alpha, alpha^T (E o D2) alpha
  const double nl2 = -(lam * lam);
  double qe = 0.0, qg = 0.0, aa = 0.0;
  for (int e = tid; e < n * n; e += THREADS) {
    const int col = e / n, row = e - col * n;
    if (row >= col) {
      const double dd = __ldg(&d2[(size_t)col * n + row]);   // symmetric: coalesced over rows
      const double ex = exp(nl2 * dd);
      Lc[(size_t)col * n + row] = ex;
      const double f = (row == col ? 1.0 : 2.0) * alpha[row] * alpha[col];
      qe += f * ex;
      qg += f * (ex * dd);
    }
  }
  for (int i = tid; i < n; i += THREADS) aa += alpha[i] * alpha[i];
  qe = block_sum(qe, red8);
  qg = block_sum(qg, red8);
  aa = block_sum(aa, red8);
  // tr(K^-1) and the two trace terms, one row of W at a time
  double tr = 0.0, te = 0.0, tg = 0.0;
  for (int kr = 0; kr < n; kr++) {
    __syncthreads();
    for (int j = tid; j <= kr; j += THREADS) wr[j] = j == kr ? wd[kr] : Lc[(size_t)kr * n + j];
    __syncthreads();
    for (int i = tid; i <= kr; i += THREADS) {
      const double wi = wr[i];
      tr += wi * wi;
      double ue = 0.0, ug = 0.0;
      for (int j = 0; j <= kr; j++) {           // E_ij from the lower half (symmetric)
        const double ex = i >= j ? Lc[(size_t)j * n + i] : Lc[(size_t)i * n + j];
        const double dd = __ldg(&d2[(size_t)j * n + i]);     // symmetric: coalesced over i
        ue = fma(ex, wr[j], ue);
        ug = fma(ex * dd, wr[j], ug);
      }
      te += wi * ue;
      tg += wi * ug;
    }
  }
  tr = block_sum(tr, red8);
  te = block_sum(te, red8);
  tg = block_sum(tg, red8);
  if (tid == 0) {
    g[0] = sg * (aa - tr);
    g[1] = tau * (qe - te);
    g[2] = -lam * tau * tau * (qg - tg);
  }
  __syncthreads();
}

template <bool GRAD>
__global__ void __launch_bounds__(THREADS, 1)
    gp_lml_kernel(const double* __restrict__ theta, int k, const double* __restrict__ d2,
                  const double* __restrict__ y, int n, double jitter, int residual,
                  double* __restrict__ work, double* __restrict__ lp, double* __restrict__ grad) {
  extern __shared__ double sm[];
  double* Cs = sm;                         // [n][LDC] the current block column, rows kb..n-1
  double* Bs = Cs + (size_t)n * LDC;       // [NB][LDC] staged L[kb+t][s0 .. s0+31]
  double* yr = Bs + NB * LDC;              // [n] right-hand side; v = L^-1 y in place
  double* red = yr + n;                    // [0] sum log L_ii, [1] |v|^2, [2] not positive definite
  double* Lc = work + (size_t)blockIdx.x * n * n;   // column-major L: Lc[s * n + i] = L[i][s]
  const int tid = threadIdx.x, q = tid & 3, r = tid >> 2, lane = tid & 31, warp = tid >> 5;

  for (int req = blockIdx.x; req < k; req += gridDim.x) {
    const double sg = theta[3 * req], tau = theta[3 * req + 1], lam = theta[3 * req + 2];
    const double nl2 = -(lam * lam), t2 = tau * tau, dg = sg * sg + jitter;
    for (int i = tid; i < n; i += THREADS) yr[i] = y[i];
    if (tid == 0) red[0] = red[1] = red[2] = 0.0;
    __syncthreads();

    for (int kb = 0; kb < n; kb += NB) {
      const int b = min(NB, n - kb);
      const int rows = n - kb;
      // ---- C = K(:, kb:kb+b) - L(:, 0:kb) L(kb:kb+b, 0:kb)^T, rows kb..n-1
      for (int i0 = 0; i0 < rows; i0 += RS * MAXP) {
        double acc[MAXP][8];
#pragma unroll
        for (int p = 0; p < MAXP; p++) {
          const int i = kb + i0 + r + RS * p;
#pragma unroll
          for (int c = 0; c < 8; c++) {
            const int t = 8 * q + c, j = kb + t;
            double v = 0.0;
            if (i < n && t < b && j <= i) {   // targets.py:211-212
              v = t2 * exp(nl2 * __ldg(&d2[(size_t)i * n + j]));
              if (i == j) v = v + dg;
            }
            acc[p][c] = v;
          }
        }
        for (int s0 = 0; s0 < kb; s0 += NB) {
          __syncthreads();
          for (int e = tid; e < NB * NB; e += THREADS) {
            const int sp = e / NB, t = e - sp * NB;
            Bs[t * LDC + sp] = t < b ? Lc[(size_t)(s0 + sp) * n + kb + t] : 0.0;
          }
          __syncthreads();
#pragma unroll 4
          for (int sp = 0; sp < NB; sp++) {
            double bv[8];
#pragma unroll
            for (int c = 0; c < 8; c++) bv[c] = Bs[(8 * q + c) * LDC + sp];
            const double* col = Lc + (size_t)(s0 + sp) * n;
#pragma unroll
            for (int p = 0; p < MAXP; p++) {
              const int i = kb + i0 + r + RS * p;
              const double a = i < n ? col[i] : 0.0;
#pragma unroll
              for (int c = 0; c < 8; c++) acc[p][c] = fma(-a, bv[c], acc[p][c]);
            }
          }
        }
#pragma unroll
        for (int p = 0; p < MAXP; p++) {
          const int il = i0 + r + RS * p;
          if (il < rows) {
#pragma unroll
            for (int c = 0; c < 8; c++) Cs[il * LDC + 8 * q + c] = acc[p][c];
          }
        }
      }
      __syncthreads();
      // ---- diagonal block: Cholesky (lane = row), log det, forward solve
      if (warp == 0) {
        bool bad = false;
        for (int j = 0; j < b; j++) {
          const double djj = Cs[j * LDC + j];
          bad |= !(djj > 0.0);
          const double ljj = sqrt(djj);
          __syncwarp();
          if (lane == j) Cs[j * LDC + j] = ljj;
          if (lane > j && lane < b) Cs[lane * LDC + j] = Cs[lane * LDC + j] / ljj;
          __syncwarp();
          if (lane > j && lane < b) {
            const double lij = Cs[lane * LDC + j];
            for (int t = j + 1; t <= lane; t++) Cs[lane * LDC + t] -= lij * Cs[t * LDC + j];
          }
        }
        __syncwarp();
        double lg = lane < b ? log(Cs[lane * LDC + lane]) : 0.0;
        lg = warp_sum(lg);
        double vv = 0.0;
        for (int j = 0; j < b; j++) {
          __syncwarp();
          const double v = yr[kb + j] / Cs[j * LDC + j];
          __syncwarp();
          if (lane == j) yr[kb + j] = v;
          if (lane > j && lane < b) yr[kb + lane] -= Cs[lane * LDC + j] * v;
          vv += v * v;
        }
        if (lane == 0) {
          red[0] += lg;
          red[1] += vv;
          if (bad) red[2] = 1.0;
        }
      }
      __syncthreads();
      // ---- panel: L[i][kb+t] = (C[i][t] - sum_{u<t} L[i][kb+u] L[kb+t][kb+u]) / L_tt;
      //      and the forward solve's update of the rows below
      for (int il = b + tid; il < rows; il += THREADS) {
        double* ci = Cs + il * LDC;
        double s = yr[kb + il];
        for (int t = 0; t < b; t++) {
          double v = ci[t];
          for (int u = 0; u < t; u++) v -= ci[u] * Cs[t * LDC + u];
          v = v / Cs[t * LDC + t];
          ci[t] = v;
          s -= v * yr[kb + t];
        }
        yr[kb + il] = s;
      }
      __syncthreads();
      // ---- the block column of L, column-major (coalesced over rows)
      for (int e = tid; e < b * rows; e += THREADS) {
        const int t = e / rows, il = e - t * rows;
        Lc[(size_t)(kb + t) * n + kb + il] = Cs[il * LDC + t];
      }
      __syncthreads();
    }
    const bool failed = red[2] != 0.0;
    if (tid == 0) {
      double v = -0.5 * red[1] - red[0] - 0.5 * n * LOG_2PI;   // targets.py:221-225
      if (!residual) v = v - 0.5 * (sg * sg + tau * tau + lam * lam) - 1.5 * LOG_2PI;
      lp[req] = failed || v != v ? __longlong_as_double((long long)FAILURE_BITS) : v;
    }
    __syncthreads();
    if constexpr (GRAD) {
      if (!failed) {   // Cs is free now: the gradient's scratch
        gp_gradient(Lc, d2, n, sg, tau, lam, jitter, yr, Cs, grad + 3 * (size_t)req);
        if (tid == 0 && !residual) {
          grad[3 * req] -= sg;
          grad[3 * req + 1] -= tau;
          grad[3 * req + 2] -= lam;
        }
      } else if (tid < 3) {
        grad[3 * (size_t)req + tid] = 0.0;
      }
      __syncthreads();
    }
  }
}

}  // namespace

extern "C" {

const char* fsmc_gp_last_error(void) { return g_err.c_str(); }

size_t fsmc_gp_lml_smem_bytes(int64_t n) { return (size_t)((n * LDC) + NB * LDC + n + 4) * sizeof(double); }

int64_t fsmc_gp_lml_max_rows(void) {   // the block column and the staged rows fit in 227 KB
  int64_t n = 2;
  while (fsmc_gp_lml_smem_bytes(n + 1) <= 227 * 1024) n++;
  return n;
}

fsmc_status fsmc_gp_lml(const double* theta, int64_t k, const double* d2, const double* y, int64_t n,
                        double jitter, int32_t residual, double* work, int64_t work_slots, double* lp,
                        void* stream_) {
  FSMC_NVTX("fsmc_gp_lml");
  return fsmc_gp_lml_grad(theta, k, d2, y, n, jitter, residual, work, work_slots, lp, nullptr, stream_);
}

fsmc_status fsmc_gp_lml_grad(const double* theta, int64_t k, const double* d2, const double* y, int64_t n,
                             double jitter, int32_t residual, double* work, int64_t work_slots, double* lp,
                             double* grad, void* stream_) {
  FSMC_NVTX("fsmc_gp_lml_grad");
  if (!theta || !d2 || !y || !work || !lp || k < 0 || n < 2 || work_slots < 1) {
    g_err = "gp_lml: bad arguments";
    return FSMC_ERR_ARG;
  }
  if (k == 0) return FSMC_OK;
  const size_t sb = fsmc_gp_lml_smem_bytes(n);
  if (n > fsmc_gp_lml_max_rows()) {
    g_err = "gp_lml: n too large for the shared-memory block column";
    return FSMC_ERR_UNSUPPORTED;
  }
  const void* kern = grad ? (const void*)gp_lml_kernel<true> : (const void*)gp_lml_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
  if (e == cudaSuccess) {
    const int grid = (int)(k < work_slots ? k : work_slots);
    fsmc::count_launch();
    if (grad)
      gp_lml_kernel<true><<<grid, THREADS, sb, (cudaStream_t)stream_>>>(theta, (int)k, d2, y, (int)n, jitter,
                                                                         residual, work, lp, grad);
    else
      gp_lml_kernel<false><<<grid, THREADS, sb, (cudaStream_t)stream_>>>(theta, (int)k, d2, y, (int)n, jitter,
                                                                          residual, work, lp, nullptr);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) {
    g_err = std::string("gp_lml: ") + cudaGetErrorString(e);
    return FSMC_ERR_CUDA;
  }
  return FSMC_OK;
}

}  // extern "C"
