// Backward kernels (placeholder until the dK/dV and dQ passes land).
#pragma once
#include <cstddef>
#include <cstdio>
#include "../../include/hk_attn.h"

namespace hk {
inline hk_status launch_bwd(const void*, const void*, const void*, const void*, const float*, const void*, void*,
                            void*, void*, float*, int, int, int, int, int, bool, cudaStream_t, char* err,
                            size_t errlen) {
  snprintf(err, errlen, "hk_attn_bwd not built yet");
  return HK_ERR_UNSUPPORTED;
}
}  // namespace hk
