// moa_sgemm.cu — fp32 MoA-ONF GEMM kernels (K3 exact FFMA, K4 3xTF32). Filled in
// after the fp64 path; until then the fp32 dtypes report MOA_ERR_INVALID_DTYPE.
#include "moa_internal.h"

namespace moa {
int sgemm_tile_configs(int, const TileConfig** out) {
  *out = nullptr;
  return 0;
}
int launch_sgemm_ffma(const moa_plan_t&, int64_t, int64_t, int64_t, const float*, const float*, float*,
                      cudaStream_t) {
  set_error("fp32 kernels not built yet");
  return MOA_ERR_INVALID_DTYPE;
}
int launch_sgemm_3xtf32(const moa_plan_t&, int64_t, int64_t, int64_t, const float*, const float*, float*,
                        cudaStream_t) {
  set_error("3xTF32 kernel not built yet");
  return MOA_ERR_INVALID_DTYPE;
}
}  // namespace moa
