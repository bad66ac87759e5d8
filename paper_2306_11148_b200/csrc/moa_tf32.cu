// moa_tf32.cu — K4: fp32 MoA-ONF GEMM as 3xTF32 on the 5th-generation tensor
// cores (tcgen05.mma kind::tf32, fp32 accumulators in TMEM).
//
//   C[(i*p)+j] := sum_k A[(i*n)+k] * B[(k*p)+j]      (Eq. 3)
//   computed as  Ab*Bb + Ab*Bs + As*Bb  with  x = xb + xs,  xb = x & 0xFFFFE000,
//   xs = x - xb (exact in fp32) — north_star's "documented TF32/3xTF32 tensor-core
//   variant"; NOT exact (tolerance 5e-3 vs ip.c, reported separately).
//
// Measured on B200 (tools/probe/umma_probe.cu): the TF32 datapath TRUNCATES an fp32
// operand to its top 19 bits, so the raw fp32 tile already IS the exact big part
// xb. Only the small parts are materialised.
//
// Structure (persistent, one CTA per SM, BM x BN output tiles, k-slabs of 32):
//   warp 0      TMA producer: A row segments (BM rows x 32 floats, K-major,
//               SWIZZLE_128B) and B row segments (32 k-rows x 32-float boxes,
//               MN-major, SWIZZLE_128B_ATOM_32B — the only MN-major layout the
//               tensor core accepts for 32-bit operands). B is used exactly as it
//               is stored, row-major, never transposed (Fig. 1).
//   warps 2..5  converters: small = x - trunc19(x) for the whole slab (the split is
//               elementwise, so the small slab has the raw slab's layout), then
//               fence.proxy.async so the tensor core sees the generic writes.
//   warp 1      TMEM allocator + MMA issuer (one thread): per k-step of 8,
//               3 x tcgen05.mma (M=128, N=BN, K=8) into a TMEM accumulator;
//               tcgen05.commit frees the stage / publishes the finished tile.
//   warps 6..9  epilogue: tcgen05.ld 32x32b -> registers -> global (row-major C), and
//               the same bits to up to 8 further destinations (the fused-gather
//               epilogue of moa_gemm_scatter / moa_gemm_lifted_gather, as K1/K3).
// Accumulators are double-buffered in TMEM (2 x BN columns).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <string>

#include "moa_internal.h"
#include "moa_ptx.cuh"

namespace moa {
namespace {
using namespace ptx;

constexpr int kBM = 128, kBK = 32;           // floats
constexpr int kRowBytes = kBK * 4;           // 128
constexpr int kABytes = kBM * kRowBytes;     // 16 KiB
constexpr int kBBox = 32 * kRowBytes;        // one B box: 32 k-rows x 32 floats = 4 KiB
constexpr int kThreads = 10 * 32;
constexpr int kConvThreads = 128;

// Instruction descriptor: D fp32 (c_format=1 @4), A,B tf32 (=2 @7, @10), A K-major
// (bit15=0), B MN-major (bit16=1), N>>3 @17, M>>4 @24.
constexpr uint32_t tf32_idesc(int bn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (1u << 16) | ((uint32_t)(bn >> 3) << 17) |
         ((uint32_t)(kBM >> 4) << 24);
}

template <int BN, int STAGES>
struct K4Traits {
  static constexpr int kBBytes = (BN / 32) * kBBox;
  static constexpr int kRawBytes = kABytes + kBBytes;
  static constexpr int kStageBytes = 2 * kRawBytes;  // raw + small
  static constexpr int kAccCols = BN;
  static constexpr int kTmemCols = 2 * BN;
  static constexpr int kSmem = 1024 + STAGES * kStageBytes + (3 * STAGES + 4) * 8 + 16;
  static_assert(kTmemCols <= 512, "TMEM has 512 columns");
  static constexpr uint32_t kIdesc = tf32_idesc(BN);
};

// ---------------------------- tcgen05 helpers ----------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_smem), "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Shared-memory matrix descriptor (sm_100 UMMA): start>>4 [0,14), LBO>>4 [16,30),
// SBO>>4 [32,46), version=1 [46,48), layout at [61,64): SWIZZLE_128B = 2,
// SWIZZLE_128B_BASE32B = 1.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint64_t layout) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (layout << 61);
}

__device__ __forceinline__ float tf32_small(float x) {
  return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    k_sgemm_3xtf32(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   float* __restrict__ C, int64_t m, int64_t n, int64_t p, int64_t ldc, int accumulate,
                   int64_t tiles_m, int64_t tiles_n, int group, const __grid_constant__ PeerDst peers) {
  using Tr = K4Traits<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw0 = smem_u32(smem_raw);
  const uint32_t base = (raw0 + 1023u) & ~1023u;
  uint8_t* sptr = smem_raw + (base - raw0);
  const uint32_t bars = base + STAGES * Tr::kStageBytes;
  const uint32_t raw_full = bars, sml_full = bars + 8 * STAGES, empty = bars + 16 * STAGES;
  const uint32_t acc_full = bars + 24 * STAGES, acc_empty = acc_full + 16;
  const uint32_t tmem_slot = acc_empty + 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tiles = tiles_m * tiles_n;
  const int ktiles = (int)((n + kBK - 1) / kBK);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(raw_full + 8 * s, 1);
      mbar_init(sml_full + 8 * s, kConvThreads / 32);
      mbar_init(empty + 8 * s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(acc_full + 8 * s, 1);
      mbar_init(acc_empty + 8 * s, 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, Tr::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(sptr + (tmem_slot - base));

  if (warp == 0) {
    // ------------------------------- TMA producer -------------------------------
    if (lane == 0) {
      prefetch_tmap(&tmA);
      prefetch_tmap(&tmB);
      int st = 0;
      uint32_t ph = 0;
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        int64_t tm, tn;
        tile_coords(t, tiles_m, tiles_n, group, tm, tn);
        for (int kt = 0; kt < ktiles; ++kt) {
          mbar_wait(empty + 8 * st, ph ^ 1u);
          const uint32_t fb = raw_full + 8 * st;
          mbar_arrive_expect_tx(fb, Tr::kRawBytes);
          const uint32_t dst = base + st * Tr::kStageBytes;
          tma_load_2d(dst, &tmA, fb, kt * kBK, (int)(tm * kBM));
#pragma unroll
          for (int b = 0; b < BN / 32; ++b)
            tma_load_2d(dst + kABytes + b * kBBox, &tmB, fb, (int)(tn * BN) + 32 * b, kt * kBK);
          if (++st == STAGES) {
            st = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    // -------------------------------- MMA issuer --------------------------------
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      int ab = 0;
      uint32_t aph = 0;
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        mbar_wait(acc_empty + 8 * ab, aph ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(ab * Tr::kAccCols);
        for (int kt = 0; kt < ktiles; ++kt) {
          mbar_wait(raw_full + 8 * st, ph);
          mbar_wait(sml_full + 8 * st, ph);
          tc_fence_after();
          const uint32_t a_big = base + st * Tr::kStageBytes, b_big = a_big + kABytes;
          const uint32_t a_sml = a_big + Tr::kRawBytes, b_sml = a_sml + kABytes;
#pragma unroll
          for (int kk = 0; kk < kBK / 8; ++kk) {
            // A: K-major, k-step of 8 floats = 32 B inside the 128 B swizzle row; SBO = 8 rows.
            const uint64_t dAb = smem_desc(a_big + kk * 32, 16, 1024, 2);
            const uint64_t dAs = smem_desc(a_sml + kk * 32, 16, 1024, 2);
            // B: MN-major BASE32B, k-step of 8 rows = 1024 B; LBO = next 32-column box,
            // SBO = next group of 4 k-rows.
            const uint64_t dBb = smem_desc(b_big + kk * 1024, kBBox, 512, 1);
            const uint64_t dBs = smem_desc(b_sml + kk * 1024, kBBox, 512, 1);
            const uint32_t acc0 = (kt > 0 || kk > 0) ? 1u : 0u;
            mma_tf32(d, dAs, dBb, Tr::kIdesc, acc0);   // small terms first
            mma_tf32(d, dAb, dBs, Tr::kIdesc, 1u);
            mma_tf32(d, dAb, dBb, Tr::kIdesc, 1u);
          }
          tc_commit(empty + 8 * st);  // raw + small slab free once these MMAs complete
          if (++st == STAGES) {
            st = 0;
            ph ^= 1u;
          }
        }
        tc_commit(acc_full + 8 * ab);  // tile's accumulator complete
        if (++ab == 2) {
          ab = 0;
          aph ^= 1u;
        }
      }
    }
  } else if (warp < 6) {
    // -------------------------------- converters --------------------------------
    const int ct = threadIdx.x - 64;  // 0..127
    int st = 0;
    uint32_t ph = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
      for (int kt = 0; kt < ktiles; ++kt) {
        mbar_wait(raw_full + 8 * st, ph);  // implies the stage's previous MMAs are done
        const float4* src = reinterpret_cast<const float4*>(sptr + st * Tr::kStageBytes);
        float4* sml = reinterpret_cast<float4*>(sptr + st * Tr::kStageBytes + Tr::kRawBytes);
#pragma unroll 4
        for (int i = ct; i < Tr::kRawBytes / 16; i += kConvThreads) {
          const float4 x = src[i];
          sml[i] = make_float4(tf32_small(x.x), tf32_small(x.y), tf32_small(x.z), tf32_small(x.w));
        }
        fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
        __syncwarp();
        if (lane == 0) mbar_arrive(sml_full + 8 * st);
        if (++st == STAGES) {
          st = 0;
          ph ^= 1u;
        }
      }
    }
  } else {
    // --------------------------------- epilogue ---------------------------------
    const int quad = warp & 3;  // TMEM lanes quad*32 .. +31 (tcgen05.ld lane restriction)
    const int row_in_tile = quad * 32 + lane;
    int ab = 0;
    uint32_t aph = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
      int64_t tm, tn;
      tile_coords(t, tiles_m, tiles_n, group, tm, tn);
      mbar_wait(acc_full + 8 * ab, aph);
      __syncwarp();  // reconverge before tcgen05.ld (.sync.aligned)
      tc_fence_after();
      const int64_t row = tm * kBM + row_in_tile;
      const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(ab * Tr::kAccCols);
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        uint32_t r[16];
        tmem_ld16(taddr + c, r);
        tmem_ld_wait();
        const int64_t col = tn * BN + c;
        if (row < m) {
          float* dst = C + row * ldc + col;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (col + 4 * q < p) {
              float4 v = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                     __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
              if (accumulate) {  // 3xTF32 is not exact anyway: add the prior C in the epilogue
                const float4 o = *reinterpret_cast<const float4*>(dst + 4 * q);
                v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
              }
              *reinterpret_cast<float4*>(dst + 4 * q) = v;
              // the fused-gather epilogue (as K1/K3 PEER): the same bits to every extra
              // destination, e.g. the other ranks' C_full over NVLink
              for (int d = 0; d < peers.nd; ++d)
                *reinterpret_cast<float4*>(reinterpret_cast<float*>(peers.dst[d]) + row * ldc + col + 4 * q) = v;
            }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty + 8 * ab);
      if (++ab == 2) {
        ab = 0;
        aph ^= 1u;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, Tr::kTmemCols);
  }
}

// ------------------------------- K4 "TS" variant -------------------------------
// Same pipeline, but both A parts live in TMEM: the converter warps read each raw A
// row from shared memory into registers (the thread owns the row = its TMEM lane),
// split it, and write big and small with tcgen05.st; the MMAs take A from TMEM
// ([a_tmem]) and only B from shared memory. This removes every A operand read and
// the A_small store from the shared-memory port, which the SS variant saturates.
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <int BN, int STAGES>
struct K4TSTraits {
  static constexpr int kBBytes = (BN / 32) * kBBox;
  static constexpr int kRawBytes = kABytes + kBBytes;
  static constexpr int kStageBytes = kRawBytes + kBBytes;  // raw A + raw B + small B
  static constexpr int kAccBufs = (2 * BN + 64 * STAGES <= 512) ? 2 : 1;
  static constexpr int kACol0 = kAccBufs * BN;              // A slots after the accumulators
  static constexpr int kTmemCols = 512;
  static constexpr int kSmem = 1024 + STAGES * kStageBytes + (3 * STAGES + 4) * 8 + 16;
  static_assert(kAccBufs * BN + 64 * STAGES <= 512, "TMEM columns");
  static constexpr uint32_t kIdesc = tf32_idesc(BN);
};

template <int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    k_sgemm_3xtf32_ts(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      float* __restrict__ C, int64_t m, int64_t n, int64_t p, int64_t ldc, int accumulate,
                      int64_t tiles_m, int64_t tiles_n, int group, const __grid_constant__ PeerDst peers) {
  using Tr = K4TSTraits<BN, STAGES>;
  constexpr int NB = Tr::kAccBufs;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw0 = smem_u32(smem_raw);
  const uint32_t base = (raw0 + 1023u) & ~1023u;
  uint8_t* sptr = smem_raw + (base - raw0);
  const uint32_t bars = base + STAGES * Tr::kStageBytes;
  const uint32_t raw_full = bars, sml_full = bars + 8 * STAGES, empty = bars + 16 * STAGES;
  const uint32_t acc_full = bars + 24 * STAGES, acc_empty = acc_full + 16;
  const uint32_t tmem_slot = acc_empty + 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tiles = tiles_m * tiles_n;
  const int ktiles = (int)((n + kBK - 1) / kBK);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(raw_full + 8 * s, 1);
      mbar_init(sml_full + 8 * s, kConvThreads / 32);
      mbar_init(empty + 8 * s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(acc_full + 8 * s, 1);
      mbar_init(acc_empty + 8 * s, 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, Tr::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(sptr + (tmem_slot - base));

  if (warp == 0) {
    if (lane == 0) {
      prefetch_tmap(&tmA);
      prefetch_tmap(&tmB);
      int st = 0;
      uint32_t ph = 0;
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        int64_t tm, tn;
        tile_coords(t, tiles_m, tiles_n, group, tm, tn);
        for (int kt = 0; kt < ktiles; ++kt) {
          mbar_wait(empty + 8 * st, ph ^ 1u);
          const uint32_t fb = raw_full + 8 * st;
          mbar_arrive_expect_tx(fb, Tr::kRawBytes);
          const uint32_t dst = base + st * Tr::kStageBytes;
          tma_load_2d(dst, &tmA, fb, kt * kBK, (int)(tm * kBM));
#pragma unroll
          for (int b = 0; b < BN / 32; ++b)
            tma_load_2d(dst + kABytes + b * kBBox, &tmB, fb, (int)(tn * BN) + 32 * b, kt * kBK);
          if (++st == STAGES) {
            st = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      int ab = 0;
      uint32_t aph = 0;
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        mbar_wait(acc_empty + 8 * ab, aph ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(ab * BN);
        for (int kt = 0; kt < ktiles; ++kt) {
          mbar_wait(raw_full + 8 * st, ph);
          mbar_wait(sml_full + 8 * st, ph);
          tc_fence_after();
          const uint32_t b_big = base + st * Tr::kStageBytes + kABytes, b_sml = b_big + Tr::kBBytes;
          const uint32_t a_big = tmem + (uint32_t)(Tr::kACol0 + 64 * st), a_sml = a_big + 32;
#pragma unroll
          for (int kk = 0; kk < kBK / 8; ++kk) {
            const uint64_t dBb = smem_desc(b_big + kk * 1024, kBBox, 512, 1);
            const uint64_t dBs = smem_desc(b_sml + kk * 1024, kBBox, 512, 1);
            const uint32_t acc0 = (kt > 0 || kk > 0) ? 1u : 0u;
            mma_tf32_ts(d, a_sml + kk * 8, dBb, Tr::kIdesc, acc0);  // small terms first
            mma_tf32_ts(d, a_big + kk * 8, dBs, Tr::kIdesc, 1u);
            mma_tf32_ts(d, a_big + kk * 8, dBb, Tr::kIdesc, 1u);
          }
          tc_commit(empty + 8 * st);
          if (++st == STAGES) {
            st = 0;
            ph ^= 1u;
          }
        }
        tc_commit(acc_full + 8 * ab);
        if (++ab == NB) {
          ab = 0;
          aph ^= 1u;
        }
      }
    }
  } else if (warp < 6) {
    // converters: thread = A row (its TMEM lane) for the A split; all 128 threads
    // cooperatively split B into the small-B slab.
    const int ct = threadIdx.x - 64;
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    int st = 0;
    uint32_t ph = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
      for (int kt = 0; kt < ktiles; ++kt) {
        mbar_wait(raw_full + 8 * st, ph);  // implies the stage's previous MMAs are done
        __syncwarp();  // reconverge before tcgen05.st (.sync.aligned)
        uint8_t* sa = sptr + st * Tr::kStageBytes;
        uint32_t big[32], sml[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {  // 16-B chunk c of the 128-B row (k = 4c..4c+3)
          const float4 x = *reinterpret_cast<const float4*>(sa + row * kRowBytes + ((c ^ (row & 7)) << 4));
          const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint32_t b = __float_as_uint(xs[e]) & 0xFFFFE000u;
            big[4 * c + e] = b;
            sml[4 * c + e] = __float_as_uint(xs[e] - __uint_as_float(b));
          }
        }
        const uint32_t ta = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(Tr::kACol0 + 64 * st);
        tmem_st32(ta, big);
        tmem_st32(ta + 32, sml);
        const float4* srcB = reinterpret_cast<const float4*>(sa + kABytes);
        float4* smlB = reinterpret_cast<float4*>(sa + kABytes + Tr::kBBytes);
#pragma unroll 4
        for (int i = ct; i < Tr::kBBytes / 16; i += kConvThreads) {
          const float4 x = srcB[i];
          smlB[i] = make_float4(tf32_small(x.x), tf32_small(x.y), tf32_small(x.z), tf32_small(x.w));
        }
        tmem_st_wait();
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(sml_full + 8 * st);
        if (++st == STAGES) {
          st = 0;
          ph ^= 1u;
        }
      }
    }
  } else {
    const int quad = warp & 3;
    const int row_in_tile = quad * 32 + lane;
    int ab = 0;
    uint32_t aph = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
      int64_t tm, tn;
      tile_coords(t, tiles_m, tiles_n, group, tm, tn);
      mbar_wait(acc_full + 8 * ab, aph);
      __syncwarp();  // reconverge before tcgen05.ld (.sync.aligned)
      tc_fence_after();
      const int64_t row = tm * kBM + row_in_tile;
      const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(ab * BN);
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        uint32_t r[16];
        tmem_ld16(taddr + c, r);
        tmem_ld_wait();
        const int64_t col = tn * BN + c;
        if (row < m) {
          float* dst = C + row * ldc + col;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (col + 4 * q < p) {
              float4 v = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                     __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
              if (accumulate) {
                const float4 o = *reinterpret_cast<const float4*>(dst + 4 * q);
                v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
              }
              *reinterpret_cast<float4*>(dst + 4 * q) = v;
              for (int d = 0; d < peers.nd; ++d)  // fused-gather epilogue (see above)
                *reinterpret_cast<float4*>(reinterpret_cast<float*>(peers.dst[d]) + row * ldc + col + 4 * q) = v;
            }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty + 8 * ab);
      if (++ab == NB) {
        ab = 0;
        aph ^= 1u;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, Tr::kTmemCols);
  }
}

template <int BN, int ST>
int launch_k4ts(const moa_plan_t& plan, const GemmArgs& g, cudaStream_t stream) {
  using Tr = K4TSTraits<BN, ST>;
  CUtensorMap ta, tb;
  const int64_t m = g.m, n = g.n, p = g.p;
  if (!encode_2d(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, g.A, m, n, kBK, kBM, CU_TENSOR_MAP_SWIZZLE_128B, g.lda) ||
      !encode_2d(&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, g.B, n, p, 32, kBK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                 g.ldb))
    return MOA_ERR_CUDA;
  auto kern = k_sgemm_3xtf32_ts<BN, ST>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [&] {
    RelaxedCapture relaxed_capture;
    attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Tr::kSmem);
  });
  if (attr_err != cudaSuccess) {
    set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(attr_err));
    return MOA_ERR_CUDA;
  }
  PeerDst peers{};
  if (g.peers) peers = *g.peers;
  kern<<<plan.grid, kThreads, Tr::kSmem, stream>>>(ta, tb, (float*)g.C, m, n, p, g.ldc, g.accumulate, plan.tiles_m,
                                                   plan.tiles_n, plan.raster_group, peers);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("k_sgemm_3xtf32_ts launch: ") + cudaGetErrorString(e));
    return MOA_ERR_CUDA;
  }
  return MOA_OK;
}

// (bn, stages): (192, 3) and (256, 2) are the TMEM-A ("TS") kernel, (128, 3) the
// all-shared-memory ("SS") kernel, kept as the block-size-sweep reference. eta =
// per-tile efficiency measured once at N=16384 (profiles/r01_configs_fp32_ts.json:
// 244.7 / 216.0 / 188.8 TF/s): 192 keeps double-buffered accumulators (2x192 + 2x64
// A columns = 512) and a 3-stage ring; 256 fits only one accumulator and 2 stages.
TileConfig kK4Configs[] = {
    {MOA_KERNEL_SGEMM_3XTF32, kBM, 192, kBK, 3, kThreads, 1, K4TSTraits<192, 3>::kSmem, 1.0},
    {MOA_KERNEL_SGEMM_3XTF32, kBM, 256, kBK, 2, kThreads, 1, K4TSTraits<256, 2>::kSmem, 0.88},
    {MOA_KERNEL_SGEMM_3XTF32, kBM, 128, kBK, 3, kThreads, 1, K4Traits<128, 3>::kSmem, 0.77},
};

template <int BN, int ST>
int launch_k4(const moa_plan_t& plan, const GemmArgs& g, cudaStream_t stream) {
  using Tr = K4Traits<BN, ST>;
  CUtensorMap ta, tb;
  const int64_t m = g.m, n = g.n, p = g.p;
  if (!encode_2d(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, g.A, m, n, kBK, kBM, CU_TENSOR_MAP_SWIZZLE_128B, g.lda) ||
      !encode_2d(&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, g.B, n, p, 32, kBK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                 g.ldb))
    return MOA_ERR_CUDA;
  float* C = (float*)g.C;
  auto kern = k_sgemm_3xtf32<BN, ST>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [&] {
    RelaxedCapture relaxed_capture;
    attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Tr::kSmem);
  });
  if (attr_err != cudaSuccess) {
    set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(attr_err));
    return MOA_ERR_CUDA;
  }
  PeerDst peers{};
  if (g.peers) peers = *g.peers;
  kern<<<plan.grid, kThreads, Tr::kSmem, stream>>>(ta, tb, C, m, n, p, g.ldc, g.accumulate, plan.tiles_m,
                                                   plan.tiles_n, plan.raster_group, peers);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("k_sgemm_3xtf32 launch: ") + cudaGetErrorString(e));
    return MOA_ERR_CUDA;
  }
  return MOA_OK;
}

}  // namespace

int tf32_tile_configs(int kernel, const TileConfig** out) {
  if (kernel == MOA_KERNEL_SGEMM_3XTF32) {
    *out = kK4Configs;
    return (int)(sizeof(kK4Configs) / sizeof(kK4Configs[0]));
  }
  *out = nullptr;
  return 0;
}

int launch_sgemm_3xtf32(const moa_plan_t& plan, const GemmArgs& g, cudaStream_t stream) {
  if (plan.bn == 256 && plan.stages == 2) return launch_k4ts<256, 2>(plan, g, stream);
  if (plan.bn == 192 && plan.stages == 3) return launch_k4ts<192, 3>(plan, g, stream);
  if (plan.bn == 128 && plan.stages == 3) return launch_k4<128, 3>(plan, g, stream);
  set_error("no compiled 3xTF32 instance for this plan");
  return MOA_ERR_INVALID_SHAPE;
}

}  // namespace moa
