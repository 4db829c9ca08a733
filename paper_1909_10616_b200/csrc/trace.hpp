// NVTX ranges (SURVEY §5 tracing): header-only nvtx3; no-ops unless a profiler is attached.
#pragma once

#include <nvtx3/nvToolsExt.h>

namespace tt {
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace tt
