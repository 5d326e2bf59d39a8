// fam_nuts.cu -- Nuts kernels for the compiled (lanes, elements) pairs.
#include "kernels.cuh"

namespace fsmc {
cudaError_t dispatch_nuts(int op, int g, int e, Params& p, const LaunchCtx& lc, cudaStream_t s,
                           uint64_t ps, long long off, const double* x0, double jit) {
  const int kind = p.t.kind;
#define S(GG, EE, TK) \
  if (g == GG && e == EE && kind == TK) return launch_op<Nuts, GG, EE, TK>(op, p, lc, s, ps, off, x0, jit);
  if (op != 0) {
    FSMC_NUTS_SPECIAL(S)
  }
#undef S
#define X(GG, EE) \
  if (g == GG && e == EE) return launch_op<Nuts, GG, EE>(op, p, lc, s, ps, off, x0, jit);
  FSMC_NUTS_CONFIGS(X)
#undef X
  return cudaErrorInvalidConfiguration;
}
}  // namespace fsmc
