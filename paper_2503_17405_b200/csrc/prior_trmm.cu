// prior_trmm.cu -- the elliptical slice sampler's batched prior transform on
// the fp64 tensor cores (BASELINE config 4).
//
// ESS INIT draws eps and forms nu = L eps (elliptical.py:68-82, line 73) with
// L the lower-triangular Cholesky factor of the Gaussian prior.  In
// fsmc_advance_prior mode every chain parks at INIT with eps in a row of
// nu [k][d]; this kernel transforms all parked rows at once:
//
//     out[r][i] = sum_{c <= i} L[i][c] eps[r][c]        (out = eps L^T)
//
// a triangular matrix product with B = L^T (upper triangular), which the
// target stores row-major as prior_t[c * d + i] = L[i][c] (zeros above the
// diagonal of L, so the diagonal tiles need no masking: they add exact 0s).
//
// DMMA (mma.sync m8n8k4 f64, the B200's fp64 tensor-core path; tcgen05 has
// no fp64 kind): a CTA owns a 64 x 64 tile of out, 4 warps as 2 (rows) x 2
// (columns), each warp a 32 x 32 register tile = 4 x 4 accumulator blocks.
// k runs in 16-wide slabs only up to the tile's last column (the triangle:
// half the work of a dense product), staged through shared memory by
// cp.async in a 3-deep pipeline.  Row strides are padded (20 and 72
// doubles) so each warp's fragment loads take the minimum two wavefronts.
// Column tiles are issued heaviest first (the last one reads all d/16 slabs).
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/fsmc.h"
#include "launch_count.h"
#include "nvtx_range.h"

namespace {

// tile: TM rows (chains) x TN columns, warps of WM x WN, k slabs of 16.
// 64 x 64 tiles: ~700 CTAs for a C4 round part (2731 rows x 1024), several
// resident per SM, so the heavy last column tiles (the whole k range) are
// spread over many CTAs instead of bounding the launch.
constexpr int TM = 64, TN = 64, WM = 32, WN = 32, TK = 16, STAGES = 3;
constexpr int WARPS = (TM / WM) * (TN / WN);
constexpr int THREADS = 32 * WARPS;
constexpr int MB = WM / 8, NB = WN / 8;     // accumulator blocks per warp
constexpr int SA = TK + 4;     // A slab row stride (doubles)
constexpr int SB = TN + 8;     // B slab row stride (doubles)
constexpr int A_DBL = TM * SA, B_DBL = TK * SB;
constexpr int STAGE_DBL = A_DBL + B_DBL;
constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE_DBL * sizeof(double);
static_assert((TM * TK / 2) % THREADS == 0 && (TK * TN / 2) % THREADS == 0, "copy split");

__device__ __forceinline__ void cp16(double* dst, const double* src, bool ok) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(src), "r"(ok ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(THREADS)
    prior_trmm_kernel(const double* __restrict__ eps, const double* __restrict__ Lt, double* __restrict__ out,
                      int rows, int d, int rtiles) {
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / (TN / WN), wn = warp % (TN / WN);
  // heaviest column tiles first (the last one reads all d/16 slabs): the
  // linear block order is column tile major, from the right
  const int ncol = (d + TN - 1) / TN;
  const int ct = ncol - 1 - (int)(blockIdx.x / rtiles);
  const int r0 = (int)(blockIdx.x % rtiles) * TM;
  const int i0 = ct * TN;
  const int kend = min(d, i0 + TN);                    // B[c][i] = 0 for c > i
  const int nslab = (kend + TK - 1) / TK;

  auto load = [&](int slab, int stage) {
    double* As = sm + stage * STAGE_DBL;
    double* Bs = As + A_DBL;
    const int k0 = slab * TK;
#pragma unroll
    for (int q = 0; q < TM * TK / 2 / THREADS; q++) {   // A: TM rows x 16 k, 8 chunks per row
      const int c = tid + q * THREADS;
      const int row = c >> 3, col = (c & 7) * 2;
      const int gr = r0 + row, gk = k0 + col;
      const bool ok = gr < rows && gk < d;
      cp16(As + row * SA + col, eps + (size_t)(ok ? gr : 0) * d + (ok ? gk : 0), ok);
    }
#pragma unroll
    for (int q = 0; q < TK * TN / 2 / THREADS; q++) {   // B: 16 k x TN i
      const int c = tid + q * THREADS;
      const int row = c / (TN / 2), col = (c % (TN / 2)) * 2;
      const int gk = k0 + row, gi = i0 + col;
      const bool ok = gk < d && gi < d;
      cp16(Bs + row * SB + col, Lt + (size_t)(ok ? gk : 0) * d + (ok ? gi : 0), ok);
    }
  };

  double acc[MB][NB][2];
#pragma unroll
  for (int a = 0; a < MB; a++)
#pragma unroll
    for (int b = 0; b < NB; b++) acc[a][b][0] = acc[a][b][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; s++) {
    if (s < nslab) load(s, s);
    cp_commit();
  }
  const int fr = lane >> 2, fc = lane & 3;             // fragment row / k index
#pragma unroll 1
  for (int slab = 0; slab < nslab; slab++) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    const int nxt = slab + STAGES - 1;
    if (nxt < nslab) load(nxt, nxt % STAGES);
    cp_commit();
    const double* As = sm + (slab % STAGES) * STAGE_DBL + (wm * WM + fr) * SA + fc;
    const double* Bs = sm + (slab % STAGES) * STAGE_DBL + A_DBL + fc * SB + wn * WN + fr;
#pragma unroll
    for (int kk = 0; kk < TK; kk += 4) {
      double a[MB], b[NB];
#pragma unroll
      for (int mb = 0; mb < MB; mb++) a[mb] = As[mb * 8 * SA + kk];
#pragma unroll
      for (int nb = 0; nb < NB; nb++) b[nb] = Bs[kk * SB + nb * 8];
#pragma unroll
      for (int mb = 0; mb < MB; mb++)
#pragma unroll
        for (int nb = 0; nb < NB; nb++) dmma(acc[mb][nb][0], acc[mb][nb][1], a[mb], b[nb]);
    }
  }
  cp_wait<0>();
  // accumulator block (mb, nb): row fr, columns 2 fc, 2 fc + 1
#pragma unroll
  for (int mb = 0; mb < MB; mb++) {
    const int gr = r0 + wm * WM + mb * 8 + fr;
    if (gr >= rows) continue;
#pragma unroll
    for (int nb = 0; nb < NB; nb++) {
      const int gi = i0 + wn * WN + nb * 8 + 2 * fc;
      if (gi < d) *reinterpret_cast<double2*>(out + (size_t)gr * d + gi) = make_double2(acc[mb][nb][0], acc[mb][nb][1]);
    }
  }
}

thread_local std::string g_err;

}  // namespace

extern "C" {

const char* fsmc_prior_trmm_last_error(void) { return g_err.c_str(); }

/* nu[r] = L nu[r] for k rows on the fp64 tensor cores (see the header). */
fsmc_status fsmc_prior_trmm(const fsmc_target* t, double* nu, double* tmp, int64_t k, void* stream_) {
  FSMC_NVTX("fsmc_prior_trmm");
  if (!t || !nu || !tmp || k < 0) { g_err = "prior_trmm needs a target, nu and tmp"; return FSMC_ERR_ARG; }
  if (t->prior_kind != FSMC_PRIOR_DENSE || !t->prior_t) {
    g_err = "prior_trmm needs a dense prior factor";
    return FSMC_ERR_ARG;
  }
  const int d = t->dim;
  if (d % 2 != 0) { g_err = "prior_trmm needs an even dimension (16-byte rows)"; return FSMC_ERR_UNSUPPORTED; }
  if (k == 0) return FSMC_OK;
  if (k > (1LL << 30)) { g_err = "too many rows"; return FSMC_ERR_ARG; }
  cudaStream_t s = (cudaStream_t)stream_;
  static bool attr[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr[dev]) {
    cudaError_t ea = cudaFuncSetAttribute(prior_trmm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)SMEM_BYTES);
    if (ea != cudaSuccess) { g_err = cudaGetErrorString(ea); return FSMC_ERR_CUDA; }
    if (dev >= 0 && dev < 64) attr[dev] = true;
  }
  // blocks: column tiles (heaviest first) x row tiles, one linear index
  const long long rt = (k + TM - 1) / TM, ct = (d + TN - 1) / TN;
  if (rt * ct >= (1LL << 31)) { g_err = "too many rows for one transform"; return FSMC_ERR_ARG; }
  fsmc::count_launch();
  prior_trmm_kernel<<<(unsigned)(rt * ct), THREADS, SMEM_BYTES, s>>>(nu, t->prior_t, tmp, (int)k, d, (int)rt);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { g_err = cudaGetErrorString(e); return FSMC_ERR_CUDA; }
  e = cudaMemcpyAsync(nu, tmp, (size_t)k * d * sizeof(double), cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) { g_err = cudaGetErrorString(e); return FSMC_ERR_CUDA; }
  return FSMC_OK;
}

}  // extern "C"
