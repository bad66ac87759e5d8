// moa_tf32.cu — K4: fp32 GEMM as 3xTF32 on tcgen05 tensor cores (placeholder
// until the kernel lands; the dtype reports MOA_ERR_INVALID_DTYPE meanwhile).
#include "moa_internal.h"

namespace moa {
int tf32_tile_configs(int, const TileConfig** out) {
  *out = nullptr;
  return 0;
}
int launch_sgemm_3xtf32(const moa_plan_t&, int64_t, int64_t, int64_t, const float*, const float*, float*,
                        cudaStream_t) {
  set_error("3xTF32 kernel not built yet");
  return MOA_ERR_INVALID_DTYPE;
}
}  // namespace moa
