// spdm_panel.cuh — K1-fast: fp32 GCOOSpDM with shared-memory B panels.
// (placeholder until the panel kernel lands; the row-tile kernel serves all
// shapes meanwhile)
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace gcoo_b200 {

inline bool panel_applicable(int64_t, int64_t, int64_t, int64_t, int64_t, const float*, const float*) {
  return false;
}

inline void launch_panel(int64_t, int64_t, int64_t, int32_t, int64_t, const float*, const int32_t*,
                         const int32_t*, const int64_t*, const int64_t*, const float*, int64_t, float*,
                         int64_t, cudaStream_t) {}

}  // namespace gcoo_b200
