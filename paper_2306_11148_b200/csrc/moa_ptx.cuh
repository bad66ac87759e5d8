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
// Order this thread's generic-proxy shared-memory accesses with later async-proxy
// (TMA / tensor-core) accesses of the same bytes. Needed by every consumer that
// reads a stage with ld.shared before releasing it to a TMA producer (WAR), and
// after st.shared of operands the tensor core will read (RAW).
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
// ------------------------- stream-K schedule (K1) -----------------------------
// Balanced assignment of the (tile, k-slab) work of one launch to its G persistent
// CTAs. The first D = (T/G - 1)*G tiles (full waves but one) are data-parallel,
// CTA c taking tiles c, c+G, ... (K1's static schedule, kept in k-lockstep per wave
// by the wave gate). The last S = T - D tiles (S in [G, 2G)) are cut into G equal
// runs of k-slabs, run r on CTA r. A tile cut between runs r and r+1 has its low-k
// part ("head") at the end of run r and its high-k part ("tail") at the start of
// run r+1.
// Bitwise rule: the tail continues the fma chain from the stored low-k partial
// (DMMA/FFMA continue the chain from their C operand), so the result equals the
// unsplit tile. Within its run a CTA computes its head FIRST and its tail LAST.
// With runs R >= K slabs, run r reaches its tail after h_r + F_r = R - K + h_{r-1}
// >= h_{r-1} slabs of its own: never before run r-1's head is done (in the
// uniform-speed model; otherwise it waits on the flag, and there is no cycle: run 0
// has no tail).
__host__ __device__ __forceinline__ int64_t sk_first_tile(int64_t tiles, int64_t G) {
  return tiles >= 2 * G ? (tiles / G - 1) * G : 0;
}
struct SkRun {
  int64_t hb, ta, f0, f1;  // head tile, tail tile, whole tiles [f0, f1)
  int32_t hk, tk;          // head k-slabs [0, hk), tail k-slabs [tk, K)
};
__device__ __forceinline__ SkRun sk_run(int64_t tiles, int64_t ktiles, int64_t G, int64_t r) {
  const int64_t first = sk_first_tile(tiles, G);
  const int64_t U = (tiles - first) * ktiles;
  const int64_t u0 = U * r / G, u1 = U * (r + 1) / G;
  SkRun q;
  q.hb = first + u1 / ktiles;
  q.hk = (int32_t)(u1 % ktiles);
  q.ta = first + u0 / ktiles;
  q.tk = (int32_t)(u0 % ktiles);
  q.f0 = first + (u0 + ktiles - 1) / ktiles;
  q.f1 = first + u1 / ktiles;
  return q;
}

// Split-tile flag protocol (one flag per CTA boundary; W = consumer warps):
// each producing warp stores its partial, fences, and adds 1; each consuming warp
// waits for W, reads, and adds 1; the last of the 2W arrivals resets the flag to 0.
__device__ __forceinline__ void split_signal(unsigned int* flag, int lane) {
  __threadfence();
  __syncwarp();
  if (lane == 0) atomicAdd(flag, 1u);
}
__device__ __forceinline__ void split_wait(const unsigned int* flag, unsigned int need, int lane) {
  if (lane == 0) {
    unsigned int v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
      if (v >= need) break;
      __nanosleep(64);
    }
  }
  __syncwarp();
  __threadfence();
}
// K1's wave gate: spin (one producer thread) until `need` whole tiles have had all
// their loads issued.
__device__ __forceinline__ void wave_gate(const unsigned int* issued, unsigned int need) {
  unsigned int v;
  for (;;) {
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(issued) : "memory");
    if (v >= need) break;
    __nanosleep(128);
  }
}
__device__ __forceinline__ void split_release(unsigned int* flag, unsigned int total, int lane) {
  __syncwarp();
  if (lane == 0 && atomicAdd(flag, 1u) == total - 1) atomicExch(flag, 0u);
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

// The same map in 32-bit arithmetic, for K1's latency tiles, whose prologue sits on
// the critical path of a few-us launch (three 64-bit divisions: ~0.05-0.1 us of it,
// profiles/r02/small_n_oneshot.json). Their tile count stays below 2^32 for any C that
// fits in memory (2^32 tiles of 16x16 doubles would be 8 TiB). (The large tiles keep
// the 64-bit map; a 32-bit one was slower at 8192^3 through code generation.)
__device__ __forceinline__ void tile_coords32(int64_t t64, int64_t tiles_m64, int64_t tiles_n, int group,
                                              int64_t& tm, int64_t& tn) {
  const uint32_t t = (uint32_t)t64, tiles_m = (uint32_t)tiles_m64;
  const uint32_t per_group = (uint32_t)group * (uint32_t)tiles_n;
  const uint32_t g = t / per_group;
  const uint32_t first = g * (uint32_t)group;
  const uint32_t rem = tiles_m - first;
  const uint32_t gm = rem < (uint32_t)group ? rem : (uint32_t)group;
  const uint32_t r = t - g * per_group;
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

// Host: a zeroed device counter for one launch on `stream` (a slot of a per-device
// pool allocated once; zeroed with cudaMemsetAsync on the stream, so it is ordered
// before the kernel): K1's wave gate counts the whole tiles whose loads are all
// issued in it. Returns false (error set) on failure.
bool acquire_tile_counter(cudaStream_t stream, unsigned int** out);
// Host: `count` zeroed split-tile flags for one stream-K launch (a window of a
// per-device ring, zeroed once at creation; every launch leaves its flags at 0 —
// see split_signal / split_wait). Returns false (error set) on failure.
bool acquire_split_flags(unsigned int count, cudaStream_t stream, unsigned int** out);

}  // namespace moa
