// moa_sgemm.cu — fp32 MoA-ONF GEMM kernels for sm_100a.
//
//   C[(i*p)+j] := sum_k A[(i*n)+k] * B[(k*p)+j]      (Eq. 3)
//
// K3 k_sgemm_ffma   : exact fp32. Persistent, warp-specialised: one producer warp
//                     streams A row segments (BM x 32 floats) and B row segments
//                     (32 k-rows x 32-float boxes) by TMA into an S-stage ring;
//                     8 consumer warps each own 16 rows x ... of C as 8x8 thread
//                     tiles and run packed FFMA2 (fma.rn.f32x2) outer products:
//                     the scalar A[i][k] (broadcast operand, no MOV) times the
//                     contiguous pair B[k][j..j+1] — the scalar-vector axpy of
//                     Fig. 1, two columns per instruction. As K1,
//                     a PEER instantiation fuses the all-gather of C into the
//                     epilogue.
// K3g k_sgemm_generic: same arithmetic, predicated loads (n or p not multiples
//                     of 4, pointers not 16-B aligned).
//
// Every C element is the fma chain over k = 0..n-1 ascending from +0 — Fig. 3
// ip.c with its update fused (reading R3) — bit for bit, for any finite input.
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

constexpr int kBKf = 32;              // floats per k-slab: one 128-byte row segment
constexpr int kRowB = kBKf * 4;       // 128
constexpr int kBoxBf = 32 * kRowB;    // one B box: 32 k-rows x 32 floats = 4 KiB

// d = a*b + c on packed pairs; `a` is a scalar broadcast to both lanes
// (ptxas encodes it as an .F32 broadcast operand of FFMA2). Measured A/B: the
// same kernel with scalar FFMA runs at 52.9 TF/s vs 61.4 with FFMA2 (N=16384).
__device__ __forceinline__ void ffma2(float2& c, float a, float2 b) {
  uint64_t aa, bb, cc, r;
  asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a));
  asm("mov.b64 %0, {%1, %2};" : "=l"(bb) : "f"(b.x), "f"(b.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(cc) : "f"(c.x), "f"(c.y));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(aa), "l"(bb), "l"(cc));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(c.x), "=f"(c.y) : "l"(r));
}

// Thread tile: rows ty*8 + r (r < 8), columns tx*4 + {0..3} and 64 + tx*4 + {0..3}
// of a 128 x 128 CTA tile; warp w holds ty = 2w, 2w+1 and tx = 0..15.
struct SAcc {
  float2 v[8][4];
};

__device__ __forceinline__ void sacc_zero(SAcc& c) {
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int q = 0; q < 4; ++q) c.v[r][q] = make_float2(0.f, 0.f);
}

// One 32-wide k-slab from the swizzled stage (A: 128 rows x 128 B; B: 4 boxes).
//   A element (row, k) at row*128 + (((k>>2) ^ (row&7))<<4) + (k&3)*4
//   B element (k, c)   at (c>>5)*4096 + k*128 + ((((c&31)>>2) ^ (k&7))<<4) + (c&3)*4
// The A loads of a warp touch 2 distinct 16-B chunks (broadcast); the B loads of
// each 8-lane phase cover 8 distinct 16-B chunks of a 128-B row: no conflicts.
__device__ __forceinline__ void ffma_slab(SAcc& c, const uint8_t* sA, const uint8_t* sB, int ty, int tx) {
  const uint8_t* arow = sA + ty * 8 * kRowB;
  const int ch = tx & 7;
  const uint8_t* b0 = sB + (tx >> 3) * kBoxBf;
  const uint8_t* b1 = sB + (2 + (tx >> 3)) * kBoxBf;
  // 4 k at a time: one LDS.128 per row brings A[row][k..k+3] (one swizzled 16-B
  // chunk), then for each of the 4 k (ascending) two LDS.128 of B and 32 FFMA2.
#pragma unroll
  for (int k4 = 0; k4 < kBKf; k4 += 4) {
    float4 a[8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
      a[r] = *reinterpret_cast<const float4*>(arow + r * kRowB + (((k4 >> 2) ^ r) << 4));
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const int k = k4 + kk;
      const int boff = k * kRowB + ((ch ^ (k & 7)) << 4);
      const float4 x = *reinterpret_cast<const float4*>(b0 + boff);
      const float4 y = *reinterpret_cast<const float4*>(b1 + boff);
      // B pair outer, rows inner: each 64-bit B operand feeds 8 consecutive FFMA2
      // (operand-reuse cache), the 32-bit A scalar changes. Same-box A/B against
      // rows-outer (A reused 4x): 61.75 vs 61.32 TF/s at N=16384, identical bits
      // (profiles/r01_ab_k3.log). Each c.v[r][q] still sees k ascending.
      const float2 bq[4] = {make_float2(x.x, x.y), make_float2(x.z, x.w), make_float2(y.x, y.y),
                            make_float2(y.z, y.w)};
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const float ar = kk == 0 ? a[r].x : kk == 1 ? a[r].y : kk == 2 ? a[r].z : a[r].w;
          ffma2(c.v[r][q], ar, bq[q]);
        }
    }
  }
}

// Accumulate mode: continue each element's fma chain from the C in memory.
template <bool kVec>
__device__ __forceinline__ void sload(SAcc& c, const float* __restrict__ C, int64_t m, int64_t p, int64_t ldc,
                                      int64_t row0, int64_t col0, int ty, int tx) {
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int64_t row = row0 + ty * 8 + r;
    const float* crow = C + row * ldc;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t col = col0 + h * 64 + tx * 4;
      float v[4] = {0.f, 0.f, 0.f, 0.f};
      if (row < m) {
        if (kVec) {
          if (col < p) {
            const float4 x = *reinterpret_cast<const float4*>(crow + col);
            v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
          }
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (col + e < p) v[e] = crow[col + e];
        }
      }
      c.v[r][2 * h] = make_float2(v[0], v[1]);
      c.v[r][2 * h + 1] = make_float2(v[2], v[3]);
    }
  }
}

template <bool kVec>
__device__ __forceinline__ void sstore(const SAcc& c, float* __restrict__ C, int64_t m, int64_t p, int64_t ldc,
                                       int64_t row0, int64_t col0, int ty, int tx) {
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int64_t row = row0 + ty * 8 + r;
    if (row >= m) continue;
    float* crow = C + row * ldc;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t col = col0 + h * 64 + tx * 4;
      const float2 lo = c.v[r][2 * h], hi = c.v[r][2 * h + 1];
      if (kVec) {
        if (col < p) *reinterpret_cast<float4*>(crow + col) = make_float4(lo.x, lo.y, hi.x, hi.y);
      } else {
        const float v[4] = {lo.x, lo.y, hi.x, hi.y};
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (col + e < p) crow[col + e] = v[e];
      }
    }
  }
}

template <int STAGES>
struct K3Traits {
  static constexpr int BM = 128, BN = 128;
  static constexpr int kConsumerWarps = 8;
  static constexpr int kThreads = (kConsumerWarps + 1) * 32;
  static constexpr int kABytes = BM * kRowB;
  static constexpr int kBBytes = kBKf * BN * 4;
  static constexpr int kStageBytes = kABytes + kBBytes;
  // (Lagged consumer groups as in K1 were measured here too: -0.15% at 4096^3 to
  // 16384^3, profiles/r02/ab_k3_lag.jsonl; not taken.)
  static constexpr int kSmem = 1024 + STAGES * kStageBytes + 2 * STAGES * 8;
};

// ACC is compile-time so the plain path keeps its register allocation. PEER: the
// fused all-gather epilogue (as K1's): every final tile is also stored to each
// peers.dst[d] (same ldc), e.g. other ranks' C_full over NVLink.
template <int STAGES, bool ACC, bool PEER>
__global__ void __launch_bounds__(K3Traits<STAGES>::kThreads, 1)
    k_sgemm_ffma(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 float* __restrict__ C, int64_t m, int64_t n, int64_t p, int64_t ldc, int64_t tiles_m,
                 int64_t tiles_n, int group, const __grid_constant__ PeerDst peers) {
  using Tr = K3Traits<STAGES>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t sbase = (raw + 1023u) & ~1023u;
  const uint8_t* sptr = smem_raw + (sbase - raw);
  const uint32_t full0 = sbase + STAGES * Tr::kStageBytes;
  const uint32_t empty0 = full0 + STAGES * 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tiles = tiles_m * tiles_n;
  const int ktiles = (int)((n + kBKf - 1) / kBKf);

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, Tr::kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == Tr::kConsumerWarps) {
    if (lane == 0) {
      prefetch_tmap(&tmA);
      prefetch_tmap(&tmB);
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        int64_t tm, tn;
        tile_coords(t, tiles_m, tiles_n, group, tm, tn);
        const int row0 = (int)(tm * Tr::BM), col0 = (int)(tn * Tr::BN);
        for (int kt = 0; kt < ktiles; ++kt) {
          mbar_wait(empty0 + 8 * stage, phase ^ 1u);
          const uint32_t fb = full0 + 8 * stage;
          mbar_arrive_expect_tx(fb, Tr::kStageBytes);
          const uint32_t sa = sbase + stage * Tr::kStageBytes;
          tma_load_2d(sa, &tmA, fb, kt * kBKf, row0);
#pragma unroll
          for (int b = 0; b < Tr::BN / 32; ++b) tma_load_2d(sa + Tr::kABytes + b * kBoxBf, &tmB, fb, col0 + 32 * b, kt * kBKf);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
    return;
  }

  const int tx = lane & 15, ty = warp * 2 + (lane >> 4);
  SAcc acc;
  int stage = 0;
  uint32_t phase = 0;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    int64_t tm, tn;
    tile_coords(t, tiles_m, tiles_n, group, tm, tn);
    if constexpr (ACC)
      sload<true>(acc, C, m, p, ldc, tm * Tr::BM, tn * Tr::BN, ty, tx);
    else
      sacc_zero(acc);
    for (int kt = 0; kt < ktiles; ++kt) {
      mbar_wait(full0 + 8 * stage, phase);
      const uint8_t* sa = sptr + stage * Tr::kStageBytes;
      ffma_slab(acc, sa, sa + Tr::kABytes, ty, tx);
      fence_proxy_async_smem();  // LDS reads before the producer's next TMA write (WAR)
      __syncwarp();
      if (lane == 0) mbar_arrive(empty0 + 8 * stage);
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1u;
      }
    }
    sstore<true>(acc, C, m, p, ldc, tm * Tr::BM, tn * Tr::BN, ty, tx);
    if constexpr (PEER)
      for (int d = 0; d < peers.nd; ++d)
        sstore<true>(acc, reinterpret_cast<float*>(peers.dst[d]), m, p, ldc, tm * Tr::BM, tn * Tr::BN, ty, tx);
  }
}

// Generic: 256 threads, single stage, predicated scalar loads into the same layout.
__global__ void __launch_bounds__(256)
    k_sgemm_generic(const float* __restrict__ A, const float* __restrict__ B, float* __restrict__ C, int64_t m,
                    int64_t n, int64_t p, int64_t lda, int64_t ldb, int64_t ldc, int accumulate, int64_t tiles_m,
                    int64_t tiles_n, int group, const __grid_constant__ PeerDst peers) {
  constexpr int BM = 128, BN = 128;
  __shared__ __align__(1024) uint8_t sm[BM * kRowB + kBKf * BN * 4];
  float* sA = reinterpret_cast<float*>(sm);
  float* sB = reinterpret_cast<float*>(sm + BM * kRowB);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tx = lane & 15, ty = warp * 2 + (lane >> 4);
  const int64_t tiles = tiles_m * tiles_n;
  SAcc acc;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    int64_t tm, tn;
    tile_coords(t, tiles_m, tiles_n, group, tm, tn);
    const int64_t row0 = tm * BM, col0 = tn * BN;
    if (accumulate)
      sload<false>(acc, C, m, p, ldc, row0, col0, ty, tx);
    else
      sacc_zero(acc);
    for (int64_t k0 = 0; k0 < n; k0 += kBKf) {
      __syncthreads();
      for (int e = threadIdx.x; e < BM * kBKf; e += 256) {
        const int r = e / kBKf, k = e % kBKf;
        const int64_t gi = row0 + r, gk = k0 + k;
        const float v = (gi < m && gk < n) ? A[gi * lda + gk] : 0.f;
        sA[(r * kRowB + (((k >> 2) ^ (r & 7)) << 4) + (k & 3) * 4) / 4] = v;
      }
      for (int e = threadIdx.x; e < kBKf * BN; e += 256) {
        const int k = e / BN, c = e % BN;
        const int64_t gk = k0 + k, gj = col0 + c;
        const float v = (gk < n && gj < p) ? B[gk * ldb + gj] : 0.f;
        sB[((c >> 5) * kBoxBf + k * kRowB + ((((c & 31) >> 2) ^ (k & 7)) << 4) + (c & 3) * 4) / 4] = v;
      }
      __syncthreads();
      ffma_slab(acc, sm, sm + BM * kRowB, ty, tx);
    }
    sstore<false>(acc, C, m, p, ldc, row0, col0, ty, tx);
    for (int d = 0; d < peers.nd; ++d)  // fused gather epilogue (see K3's PEER)
      sstore<false>(acc, reinterpret_cast<float*>(peers.dst[d]), m, p, ldc, row0, col0, ty, tx);
  }
}

TileConfig kK3Configs[] = {
    {MOA_KERNEL_SGEMM_FFMA, 128, 128, 32, 6, K3Traits<6>::kThreads, 1, K3Traits<6>::kSmem, 1.0},
};
TileConfig kK3gConfigs[] = {
    {MOA_KERNEL_SGEMM_GENERIC, 128, 128, 32, 1, 256, 1, 128 * kRowB + kBKf * 128 * 4, 0.5},
};

void refine_occupancy() {
  static std::once_flag once;
  std::call_once(once, [] {
    RelaxedCapture relaxed_capture;
    int n = 0;
    auto kern = k_sgemm_ffma<6, false, false>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, K3Traits<6>::kSmem) == cudaSuccess &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, K3Traits<6>::kThreads, K3Traits<6>::kSmem) ==
            cudaSuccess &&
        n > 0)
      kK3Configs[0].ctas_per_sm = n;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_sgemm_generic, 256, 0) == cudaSuccess && n > 0)
      kK3gConfigs[0].ctas_per_sm = n;
    cudaGetLastError();
  });
}

}  // namespace

int sgemm_tile_configs(int kernel, const TileConfig** out) {
  refine_occupancy();
  if (kernel == MOA_KERNEL_SGEMM_FFMA) {
    *out = kK3Configs;
    return 1;
  }
  if (kernel == MOA_KERNEL_SGEMM_GENERIC) {
    *out = kK3gConfigs;
    return 1;
  }
  return tf32_tile_configs(kernel, out);
}

int launch_sgemm_ffma(const moa_plan_t& plan, const GemmArgs& g, cudaStream_t stream) {
  using Tr = K3Traits<6>;
  CUtensorMap ta, tb;
  const int64_t m = g.m, n = g.n, p = g.p;
  if (!encode_2d(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, g.A, m, n, kBKf, Tr::BM, CU_TENSOR_MAP_SWIZZLE_128B, g.lda) ||
      !encode_2d(&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, g.B, n, p, 32, kBKf, CU_TENSOR_MAP_SWIZZLE_128B, g.ldb))
    return MOA_ERR_CUDA;
  float* C = (float*)g.C;
  const bool peer = g.peers && g.peers->nd > 0;
  auto kern = g.accumulate ? (peer ? k_sgemm_ffma<6, true, true> : k_sgemm_ffma<6, true, false>)
                           : (peer ? k_sgemm_ffma<6, false, true> : k_sgemm_ffma<6, false, false>);
  PeerDst peers{};
  if (peer) peers = *g.peers;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [&] {
    RelaxedCapture relaxed_capture;
    for (auto k : {k_sgemm_ffma<6, false, false>, k_sgemm_ffma<6, true, false>, k_sgemm_ffma<6, false, true>,
                   k_sgemm_ffma<6, true, true>})
      if (attr_err == cudaSuccess)
        attr_err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Tr::kSmem);
  });
  if (attr_err != cudaSuccess) {
    set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(attr_err));
    return MOA_ERR_CUDA;
  }
  kern<<<plan.grid, Tr::kThreads, Tr::kSmem, stream>>>(ta, tb, C, m, n, p, g.ldc, plan.tiles_m, plan.tiles_n,
                                                       plan.raster_group, peers);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("k_sgemm_ffma launch: ") + cudaGetErrorString(e));
    return MOA_ERR_CUDA;
  }
  return MOA_OK;
}

int launch_sgemm_generic(const moa_plan_t& plan, const GemmArgs& g, cudaStream_t stream) {
  PeerDst peers{};
  if (g.peers) peers = *g.peers;
  k_sgemm_generic<<<plan.grid, 256, 0, stream>>>((const float*)g.A, (const float*)g.B, (float*)g.C, g.m, g.n, g.p,
                                                 g.lda, g.ldb, g.ldc, g.accumulate, plan.tiles_m, plan.tiles_n,
                                                 plan.raster_group, peers);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("k_sgemm_generic launch: ") + cudaGetErrorString(e));
    return MOA_ERR_CUDA;
  }
  return MOA_OK;
}

}  // namespace moa
