// nvtx.hpp — NVTX ranges around the host phases of the hot path (SURVEY §5 tracing): one
// range per measured batch and per Droplet round, visible in Nsight Systems / ncu --nvtx.
// NVTX v3 is header-only: with no tool attached every call is a no-op on a null pointer.
#pragma once
#include <nvtx3/nvToolsExt.h>

namespace db200 {
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace db200
