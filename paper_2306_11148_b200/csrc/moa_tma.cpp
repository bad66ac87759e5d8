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
    RelaxedCapture relaxed_capture;
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

// A launch being captured into a CUDA graph keeps its slot addresses for every replay,
// while eager launches keep cycling through the ring: after a wrap-around an eager
// launch could share a counter (or split flags) with a replay running concurrently.
// So captured launches get dedicated slots, allocated here and owned by the process
// for its lifetime (graphs may outlive any scope the library could see).
static bool capturing(cudaStream_t stream) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  return stream && cudaStreamIsCapturing(stream, &st) == cudaSuccess && st == cudaStreamCaptureStatusActive;
}

static cudaError_t dedicated_zeroed(size_t bytes, unsigned int** out) {
  RelaxedCapture relaxed_capture;
  cudaStream_t ps = nullptr;
  cudaError_t e = cudaMalloc(out, bytes);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMemsetAsync(*out, 0, bytes, ps);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ps);
  if (ps) cudaStreamDestroy(ps);
  return e;
}

bool acquire_tile_counter(cudaStream_t stream, unsigned int** out) {
  int device = 0;
  cudaError_t e = cudaGetDevice(&device);
  unsigned int* slot = nullptr;
  if (e == cudaSuccess && capturing(stream)) {
    e = dedicated_zeroed(sizeof(unsigned int), &slot);  // (the memset node below resets it per replay)
  } else if (e == cudaSuccess) {
    std::lock_guard<std::mutex> lk(g_ctr_mu);
    CounterPool& pool = g_ctr[device];
    if (!pool.dev) {  // library-owned, once (capture-safe: not stream work)
      RelaxedCapture relaxed_capture;
      e = cudaMalloc(&pool.dev, kCounterSlots * sizeof(unsigned int));
    }
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

namespace {
// Split-tile flags: one uint32 per CTA boundary of a stream-K launch. The ring is
// zeroed once when created; every flag used by a launch is returned to 0 by its
// last reader inside that launch, so no per-launch memset is needed. Slots are
// handed out round-robin, so launches in flight on different streams (up to
// kFlagSlots / grid of them) never share a flag.
constexpr unsigned int kFlagSlots = 1u << 18;
struct FlagPool {
  unsigned int* dev = nullptr;
  unsigned int next = 0;
};
std::mutex g_flag_mu;
std::map<int, FlagPool> g_flag;
}  // namespace

bool acquire_split_flags(unsigned int count, cudaStream_t stream, unsigned int** out) {
  int device = 0;
  cudaError_t e = cudaGetDevice(&device);
  unsigned int* slot = nullptr;
  if (e == cudaSuccess && count > kFlagSlots) {
    set_error("split flags: grid larger than the flag pool");
    return false;
  }
  if (e == cudaSuccess && capturing(stream)) {
    e = dedicated_zeroed(count * sizeof(unsigned int), &slot);  // self-resetting, as the ring's
  } else if (e == cudaSuccess) {
    std::lock_guard<std::mutex> lk(g_flag_mu);
    FlagPool& pool = g_flag[device];
    if (!pool.dev) {  // library-owned, once; capture-safe: zeroed on a private stream
      RelaxedCapture relaxed_capture;
      cudaStream_t ps = nullptr;
      e = cudaMalloc(&pool.dev, kFlagSlots * sizeof(unsigned int));
      if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaMemsetAsync(pool.dev, 0, kFlagSlots * sizeof(unsigned int), ps);
      if (e == cudaSuccess) e = cudaStreamSynchronize(ps);
      if (ps) cudaStreamDestroy(ps);
    }
    if (e == cudaSuccess) {
      if (pool.next + count > kFlagSlots) pool.next = 0;
      slot = pool.dev + pool.next;
      pool.next += count;
    }
  }
  if (e != cudaSuccess) {
    set_error(std::string("split flags: ") + cudaGetErrorString(e));
    return false;
  }
  *out = slot;
  return true;
}

}  // namespace moa
