// moa_tma.cpp — host-side TMA descriptor encoding (cuTensorMapEncodeTiled via the
// runtime's driver entry point, so libmoa.so needs no -lcuda).
#include <cstdio>
#include <map>
#include <mutex>
#include <string>

#include "moa_internal.h"
#include "moa_ptx.cuh"

namespace moa {

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool encode_2d(CUtensorMap* map, CUtensorMapDataType dt, int esize, const void* base, int64_t rows, int64_t cols,
               int box_cols, int box_rows, CUtensorMapSwizzle swizzle, int64_t ld) {
  auto enc = get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled entry point unavailable");
    return false;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld < 0 ? cols : ld) * (cuuint64_t)esize};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = enc(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[128];
    snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled failed (CUresult %d)", (int)r);
    set_error(buf);
    return false;
  }
  return true;
}

namespace {
constexpr int kCounterSlots = 4096;
struct CounterPool {
  unsigned int* dev = nullptr;
  unsigned int next = 0;
};
std::mutex g_ctr_mu;
std::map<int, CounterPool> g_ctr;
}  // namespace

bool acquire_tile_counter(cudaStream_t stream, unsigned int** out) {
  int device = 0;
  cudaError_t e = cudaGetDevice(&device);
  unsigned int* slot = nullptr;
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> lk(g_ctr_mu);
    CounterPool& pool = g_ctr[device];
    if (!pool.dev) e = cudaMalloc(&pool.dev, kCounterSlots * sizeof(unsigned int));  // library-owned, once
    if (e == cudaSuccess) slot = pool.dev + (pool.next++ % kCounterSlots);
  }
  if (e == cudaSuccess) e = cudaMemsetAsync(slot, 0, sizeof(unsigned int), stream);
  if (e != cudaSuccess) {
    set_error(std::string("tile counter: ") + cudaGetErrorString(e));
    return false;
  }
  *out = slot;
  return true;
}

}  // namespace moa
