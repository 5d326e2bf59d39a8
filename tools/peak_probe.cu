// peak_probe.cu -- measured issue-rate ceilings for the pipes the FSM step
// kernels use (the B200 guides list HBM and bf16 peaks only): fp64 DFMA,
// fp32 FFMA, 64-bit integer multiply (splitmix64's IMAD chains).
// Build: make tools/peak_probe ; run on the GPU box: tools/peak_probe > profiles/..json
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kIters = 1 << 14;
constexpr int kChains = 8;   // independent dependency chains per thread (ILP)

__global__ void dfma_kernel(double* out, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; c++) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < kIters; i++)
#pragma unroll
    for (int c = 0; c < kChains; c++) x[c] = fma(x[c], a, b);
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; c++) s += x[c];
  if (s == 12345.678) out[0] = s;
}
__global__ void ffma_kernel(float* out, float a, float b) {
  float x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; c++) x[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < kIters; i++)
#pragma unroll
    for (int c = 0; c < kChains; c++) x[c] = fmaf(x[c], a, b);
  float s = 0;
#pragma unroll
  for (int c = 0; c < kChains; c++) s += x[c];
  if (s == 12345.678f) out[0] = s;
}
__global__ void mul64_kernel(uint64_t* out, uint64_t a) {
  uint64_t x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; c++) x[c] = threadIdx.x + c * 0x9E3779B97F4A7C15ULL;
  for (int i = 0; i < kIters; i++)
#pragma unroll
    for (int c = 0; c < kChains; c++) x[c] = x[c] * a;
  uint64_t s = 0;
#pragma unroll
  for (int c = 0; c < kChains; c++) s ^= x[c];
  if (s == 42) out[0] = s;
}
__global__ void mix64_kernel(uint64_t* out) {
  uint64_t x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; c++) x[c] = threadIdx.x + c * 0x9E3779B97F4A7C15ULL;
  for (int i = 0; i < kIters / 4; i++)
#pragma unroll
    for (int c = 0; c < kChains; c++) {
      uint64_t z = x[c];
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
      x[c] = z ^ (z >> 31);
    }
  uint64_t s = 0;
#pragma unroll
  for (int c = 0; c < kChains; c++) s ^= x[c];
  if (s == 42) out[0] = s;
}

template <class K, class... A>
float time_ms(K kern, int blocks, int threads, A... args) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(args...);  // warm-up
  cudaEventRecord(e0);
  for (int r = 0; r < 5; r++) kern<<<blocks, threads>>>(args...);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / 5;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  void* buf;
  cudaMalloc(&buf, 64);
  const int blocks = sms * 8, threads = 256;
  const double thr = (double)blocks * threads;
  const double ops = thr * kIters * kChains;
  float t_d = time_ms(dfma_kernel, blocks, threads, (double*)buf, 1.0000001, 1e-9);
  float t_f = time_ms(ffma_kernel, blocks, threads, (float*)buf, 1.0000001f, 1e-9f);
  float t_m = time_ms(mul64_kernel, blocks, threads, (uint64_t*)buf, (uint64_t)0xBF58476D1CE4E5B9ULL);
  float t_x = time_ms(mix64_kernel, blocks, threads, (uint64_t*)buf);
  printf("{\"sms\": %d, \"clock_khz\": %d,\n", sms, clk);
  printf(" \"fp64_fma_tflops\": %.3f,\n", 2.0 * ops / (t_d * 1e-3) / 1e12);
  printf(" \"fp32_fma_tflops\": %.3f,\n", 2.0 * ops / (t_f * 1e-3) / 1e12);
  printf(" \"u64_mul_gops\": %.1f,\n", ops / (t_m * 1e-3) / 1e9);
  printf(" \"mix64_gops\": %.1f,\n", thr * (kIters / 4) * kChains / (t_x * 1e-3) / 1e9);
  printf(" \"how\": \"%d blocks x %d threads, %d independent chains per thread, %d dependent ops each; "
         "best-effort steady state, CUDA events over 5 launches\"}\n", blocks, threads, kChains, kIters);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
