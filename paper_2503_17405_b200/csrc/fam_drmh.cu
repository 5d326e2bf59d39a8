// fam_drmh.cu -- Drmh kernels for the compiled (lanes, elements) pairs.
#include "kernels.cuh"

namespace fsmc {
cudaError_t dispatch_drmh(int op, int g, int e, Params& p, const LaunchCtx& lc, cudaStream_t s,
                           uint64_t ps, long long off, const double* x0, double jit) {
  const int kind = p.t.kind;
  if (p.k.split_body) {
#define X(GG, EE) \
  if (g == GG && e == EE) return launch_op<DrmhSplit, GG, EE>(op, p, lc, s, ps, off, x0, jit);
    FSMC_DRMH_SPLIT_CONFIGS(X)
#undef X
    return cudaErrorInvalidConfiguration;
  }
#define S(GG, EE, TK) \
  if (g == GG && e == EE && kind == TK) return launch_op<Drmh, GG, EE, TK>(op, p, lc, s, ps, off, x0, jit);
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
