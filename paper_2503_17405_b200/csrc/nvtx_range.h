// nvtx_range.h -- NVTX ranges around the engine's host entry points and the
// rounds of its multi-launch drivers (tracing per phase).
// Header-only NVTX v3: with no tool attached a push/pop is a call through a
// null-initialised function pointer, so the ranges stay in release builds;
// under nsys / ncu (--nvtx) they name the phases of a run.
#pragma once
#include <nvtx3/nvToolsExt.h>

namespace fsmc {
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace fsmc

#define FSMC_NVTX_CAT2(a, b) a##b
#define FSMC_NVTX_CAT(a, b) FSMC_NVTX_CAT2(a, b)
// a range from here to the end of the enclosing scope
#define FSMC_NVTX(name) ::fsmc::NvtxRange FSMC_NVTX_CAT(fsmc_nvtx_, __LINE__)(name)
