// fam_nuts.cu -- Nuts kernels for the compiled (lanes, elements) pairs.
#include "kernels.cuh"

namespace fsmc {
cudaError_t dispatch_nuts(int op, int g, int e, Params& p, const LaunchCtx& lc, cudaStream_t s,
                           uint64_t ps, long long off, const double* x0, double jit) {
  const int kind = p.t.kind;
  if (p.k.precision == 1) {   // fp32 throughput mode: the sampling run only
#define F(GG, EE, TK) \
  if (op == 1 && g == GG && e == EE && kind == TK) return Launch<NutsF, GG, EE, TK>::run(p, lc, s);
    FSMC_NUTS_F32(F)
#undef F
    if (op == 1) return cudaErrorNotSupported;
  }
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
