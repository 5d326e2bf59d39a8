// fam_slice.cu -- Slice kernels (univariate: one lane, one element per chain).
#include "kernels.cuh"

namespace fsmc {
cudaError_t dispatch_slice(int op, int g, int e, Params& p, const LaunchCtx& lc, cudaStream_t s,
                           uint64_t ps, long long off, const double* x0, double jit) {
#define X(GG, EE) \
  if (g == GG && e == EE) return launch_op<Slice, GG, EE>(op, p, lc, s, ps, off, x0, jit);
  FSMC_SLICE_CONFIGS(X)
#undef X
  return cudaErrorInvalidConfiguration;
}
}  // namespace fsmc
