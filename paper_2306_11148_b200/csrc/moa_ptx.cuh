// moa_ptx.cuh — product-internal sm_100a device helpers shared by the kernel
// translation units (mbarrier, TMA, tile rasterisation) and the host-side TMA
// descriptor encoder. Not part of the ABI.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace moa {
#ifdef __CUDACC__
namespace ptx {

// ------------------------------- PTX helpers --------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n"
      " mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
// Grouped rasterisation of output tiles (L2 reuse of A row-panels / B col-panels).
__device__ __forceinline__ void tile_coords(int64_t t, int64_t tiles_m, int64_t tiles_n, int group, int64_t& tm,
                                            int64_t& tn) {
  const int64_t per_group = (int64_t)group * tiles_n;
  const int64_t g = t / per_group;
  const int64_t first = g * group;
  const int64_t rem = tiles_m - first;
  const int64_t gm = rem < group ? rem : group;
  const int64_t r = t - g * per_group;
  tm = first + r % gm;
  tn = r / gm;
}


}  // namespace ptx
#endif  // __CUDACC__

// Host: 2-D row-major tensor map {cols (inner), rows} with row stride ld, box
// {box_cols, box_rows}, the given swizzle, zero fill out of bounds. Returns false (and sets the error) on failure.
bool encode_2d(CUtensorMap* map, CUtensorMapDataType dt, int esize, const void* base, int64_t rows, int64_t cols,
               int box_cols, int box_rows, CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_128B,
               int64_t ld = -1 /* row stride in elements; -1 = cols */);

// Host: a zeroed device counter for one dynamically scheduled launch on `stream`
// (a slot of a per-device pool allocated once; zeroed with cudaMemsetAsync on the
// stream, so it is ordered before the kernel). Returns false (error set) on failure.
bool acquire_tile_counter(cudaStream_t stream, unsigned int** out);

}  // namespace moa
