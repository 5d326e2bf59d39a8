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

__global__ void __launch_bounds__(THREADS, 1)
    gp_lml_kernel(const double* __restrict__ theta, int k, const double* __restrict__ d2,
                  const double* __restrict__ y, int n, double jitter, int residual,
                  double* __restrict__ work, double* __restrict__ lp) {
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
    if (tid == 0) {
      double v = -0.5 * red[1] - red[0] - 0.5 * n * LOG_2PI;   // targets.py:221-225
      if (!residual) v = v - 0.5 * (sg * sg + tau * tau + lam * lam) - 1.5 * LOG_2PI;
      lp[req] = red[2] != 0.0 || v != v ? __longlong_as_double((long long)FAILURE_BITS) : v;
    }
    __syncthreads();
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
  cudaError_t e = cudaFuncSetAttribute((const void*)gp_lml_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
  if (e == cudaSuccess) {
    const int grid = (int)(k < work_slots ? k : work_slots);
    fsmc::count_launch();
    gp_lml_kernel<<<grid, THREADS, sb, (cudaStream_t)stream_>>>(theta, (int)k, d2, y, (int)n, jitter,
                                                                 residual, work, lp);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) {
    g_err = std::string("gp_lml: ") + cudaGetErrorString(e);
    return FSMC_ERR_CUDA;
  }
  return FSMC_OK;
}

}  // extern "C"
