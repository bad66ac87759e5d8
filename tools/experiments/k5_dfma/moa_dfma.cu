// ARCHIVED EXPERIMENT (round 2) — not built, not part of libmoa.so. Compiled into the
// library for one measurement (profiles/r02/small_n_k5_dfma.json, tools/small_n.py):
// the DFMA latency tiles were SLOWER than K1's DMMA latency tiles at every N from 64
// to 1024 (256^3: 7.06 vs 5.79 us graph-timed). Its loop is bound by its shared-memory
// loads, not by the DFMA latency (8 cycles, tools/probe/chain_latency.cu). Kept as the
// evidence behind DESIGN.md's small-N reading; to rebuild it, restore the
// MOA_KERNEL_DGEMM_DFMA plumbing of commit "K5 experiment" (moa_host.cpp choose_dfma).
// moa_dfma.cu — K5: fp64 MoA-ONF GEMM latency tiles on the FP64 SIMT pipe (DFMA).
//
//   C[(i*p)+j] := sum_k A[(i*n)+k] * B[(k*p)+j]      (Eq. 3)
//
// Why it was tried. Parity is bitwise against Fig. 3 ip.c with its update fused
// (reading R3): every element is ONE fma chain, k = 0..n-1 ascending, so the chain
// cannot be split. The hypothesis was that the n/4 dependent DMMA.8x8x4 of that chain
// bound tiny problems; the direct probe later showed a dependent DMMA takes only 26
// cycles (tools/probe/chain_latency.cu), so the hypothesis was wrong, and this kernel
// (bitwise the same chain on DFMA) lost at every size.
//
// Structure: one tile per CTA (grid = tiles, tile t = blockIdx.x in K1's grouped
// raster order). One producer warp streams A row segments and B row boxes with TMA
// in K1's exact stage layout (128B-swizzled 16-k slabs; B by rows, never by
// columns: Fig. 1) through an S-stage mbarrier ring; with all of k
// resident (ceil(n/16) <= S) every load is in flight at once and no stage is
// released. Consumer thread t owns a 2 x TN block of C (row pair t / (BN/TN), column
// group t % (BN/TN)): per k one 16-B A chunk per row (two k at once) and TN/2 16-B B
// chunks, then 2*TN independent fma chains. Programmatic dependent launch as K1.
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

constexpr int kBK = 16;                  // k per slab (one 128-B row segment of A)
constexpr int kRowBytes = kBK * 8;       // 128
constexpr int kBoxBytes = 16 * kRowBytes;  // B box: 16 k-rows x 16 columns

template <int BM, int BN, int TN, int STAGES>
struct K5Traits {
  static constexpr int kConsumers = BM * BN / (2 * TN);
  static constexpr int kConsumerWarps = kConsumers / 32;
  static constexpr int kThreads = kConsumers + 32;  // + one producer warp
  static constexpr int kABytes = BM * kRowBytes;
  static constexpr int kBBytes = BN * kRowBytes;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kSmem = 1024 + STAGES * kStageBytes + 2 * STAGES * 8;
  static_assert(kConsumers % 32 == 0 && BM % 2 == 0 && BN % 16 == 0 && (TN == 2 || TN == 4), "K5 tile shape");
  static_assert(kStageBytes % 1024 == 0, "stages stay 1024-B aligned (128B swizzle)");
};

template <int BM, int BN, int TN, int STAGES, bool ACC, bool PEER>
__global__ void __launch_bounds__(K5Traits<BM, BN, TN, STAGES>::kThreads)
    k_dgemm_dfma(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 double* __restrict__ C, int64_t m, int64_t n, int64_t p, int64_t ldc, int64_t tiles_m,
                 int64_t tiles_n, int group, const __grid_constant__ PeerDst peers) {
  using Tr = K5Traits<BM, BN, TN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t sbase = (raw + 1023u) & ~1023u;
  const uint8_t* sptr = smem_raw + (sbase - raw);
  const uint32_t full0 = sbase + STAGES * Tr::kStageBytes;
  const uint32_t empty0 = full0 + STAGES * 8;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ktiles = (int)((n + kBK - 1) / kBK);
  const bool release = ktiles > STAGES;  // all of k resident: no stage is ever refilled
  int64_t tm, tn;
  tile_coords(blockIdx.x, tiles_m, tiles_n, group, tm, tn);

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, Tr::kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: global accesses after the previous grid

  if (warp == Tr::kConsumerWarps) {
    // ------------------------------- producer ---------------------------------
    if (lane == 0) {
      prefetch_tmap(&tmA);
      prefetch_tmap(&tmB);
      const int row0 = (int)(tm * BM), col0 = (int)(tn * BN);
      int stage = 0;
      uint32_t phase = 0;
      for (int kt = 0; kt < ktiles; ++kt) {
        mbar_wait(empty0 + 8 * stage, phase ^ 1u);
        const uint32_t fb = full0 + 8 * stage;
        mbar_arrive_expect_tx(fb, Tr::kStageBytes);
        const uint32_t sa = sbase + stage * Tr::kStageBytes;
        tma_load_2d(sa, &tmA, fb, kt * kBK, row0);
#pragma unroll
        for (int b = 0; b < BN / 16; ++b) tma_load_2d(sa + Tr::kABytes + b * kBoxBytes, &tmB, fb, col0 + 16 * b, kt * kBK);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    return;
  }

  // -------------------------------- consumers ----------------------------------
  constexpr int kGroups = BN / TN;  // column groups per row pair
  const int r0 = 2 * (tid / kGroups), c0 = TN * (tid % kGroups);
  // A: rows r0, r0+1; 16-B chunk q (k = 2q, 2q+1) of row r at r*128 + ((q ^ (r&7)) << 4)
  const uint32_t aoff0 = r0 * kRowBytes, aoff1 = (r0 + 1) * kRowBytes;
  const int ar0 = r0 & 7, ar1 = (r0 + 1) & 7;
  // B: column pair c (even) of k-row k at (c>>4)*2048 + k*128 + ((((c&15)>>1) ^ (k&7)) << 4)
  uint32_t boff[TN / 2];
  int bq[TN / 2];
#pragma unroll
  for (int h = 0; h < TN / 2; ++h) {
    const int c = c0 + 2 * h;
    boff[h] = (uint32_t)Tr::kABytes + (c >> 4) * kBoxBytes;
    bq[h] = (c & 15) >> 1;
  }
  double acc[2][TN];
  const int64_t grow = tm * BM + r0, gcol = tn * BN + c0;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      acc[i][j] = 0.0;
      if (ACC && grow + i < m && gcol + j < p) acc[i][j] = C[(grow + i) * ldc + gcol + j];
    }
  int stage = 0;
  uint32_t phase = 0;
  for (int kt = 0; kt < ktiles; ++kt) {
    mbar_wait(full0 + 8 * stage, phase);
    const uint8_t* s = sptr + stage * Tr::kStageBytes;
#pragma unroll
    for (int q = 0; q < kBK / 2; ++q) {  // k = 2q, 2q+1 (ascending: every chain is Fig. 3's sigma loop)
      const double2 a0 = *reinterpret_cast<const double2*>(s + aoff0 + ((q ^ ar0) << 4));
      const double2 a1 = *reinterpret_cast<const double2*>(s + aoff1 + ((q ^ ar1) << 4));
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int k = 2 * q + e;
        const double ak0 = e ? a0.y : a0.x, ak1 = e ? a1.y : a1.x;
#pragma unroll
        for (int h = 0; h < TN / 2; ++h) {
          const double2 b = *reinterpret_cast<const double2*>(s + boff[h] + k * kRowBytes + ((bq[h] ^ (k & 7)) << 4));
          acc[0][2 * h] = fma(ak0, b.x, acc[0][2 * h]);
          acc[0][2 * h + 1] = fma(ak0, b.y, acc[0][2 * h + 1]);
          acc[1][2 * h] = fma(ak1, b.x, acc[1][2 * h]);
          acc[1][2 * h + 1] = fma(ak1, b.y, acc[1][2 * h + 1]);
        }
      }
    }
    if (release) {  // WAR across proxies before the producer's next TMA write (see K1)
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(empty0 + 8 * stage);
    }
    if (++stage == STAGES) {
      stage = 0;
      phase ^= 1u;
    }
  }
  // contiguous write-back C[(i*p)+j] := (TMA eligibility: p even, C 16-B aligned)
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    if (grow + i >= m) continue;
#pragma unroll
    for (int h = 0; h < TN / 2; ++h) {
      const int64_t col = gcol + 2 * h;
      if (col >= p) continue;
      const double2 v = make_double2(acc[i][2 * h], acc[i][2 * h + 1]);
      *reinterpret_cast<double2*>(C + (grow + i) * ldc + col) = v;
      if constexpr (PEER)
        for (int d = 0; d < peers.nd; ++d)
          *reinterpret_cast<double2*>(reinterpret_cast<double*>(peers.dst[d]) + (grow + i) * ldc + col) = v;
    }
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <int BM, int BN, int TN, int ST, bool ACC, bool PEER>
cudaError_t k5_attrs() {
  auto kern = k_dgemm_dfma<BM, BN, TN, ST, ACC, PEER>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, K5Traits<BM, BN, TN, ST>::kSmem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  return e;
}

template <int BM, int BN, int TN, int ST>
int launch_k5(const moa_plan_t& plan, const GemmArgs& g, cudaStream_t stream) {
  using Tr = K5Traits<BM, BN, TN, ST>;
  CUtensorMap ta, tb;
  if (!encode_2d(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, g.A, g.m, g.n, 16, BM, CU_TENSOR_MAP_SWIZZLE_128B, g.lda) ||
      !encode_2d(&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, g.B, g.n, g.p, 16, 16, CU_TENSOR_MAP_SWIZZLE_128B, g.ldb))
    return MOA_ERR_CUDA;
  const bool peer = g.peers && g.peers->nd > 0;
  auto kern = g.accumulate ? (peer ? k_dgemm_dfma<BM, BN, TN, ST, true, true> : k_dgemm_dfma<BM, BN, TN, ST, true, false>)
                           : (peer ? k_dgemm_dfma<BM, BN, TN, ST, false, true> : k_dgemm_dfma<BM, BN, TN, ST, false, false>);
  PeerDst peers{};
  if (peer) peers = *g.peers;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [&] {
    RelaxedCapture relaxed_capture;
    attr_err = k5_attrs<BM, BN, TN, ST, false, false>();
    if (attr_err == cudaSuccess) attr_err = k5_attrs<BM, BN, TN, ST, true, false>();
    if (attr_err == cudaSuccess) attr_err = k5_attrs<BM, BN, TN, ST, false, true>();
    if (attr_err == cudaSuccess) attr_err = k5_attrs<BM, BN, TN, ST, true, true>();
  });
  if (attr_err != cudaSuccess) {
    set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(attr_err));
    return MOA_ERR_CUDA;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)plan.tiles);
  cfg.blockDim = dim3(Tr::kThreads);
  cfg.dynamicSmemBytes = Tr::kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ta, tb, (double*)g.C, g.m, g.n, g.p, g.ldc, plan.tiles_m, plan.tiles_n,
                                     (int)plan.raster_group, peers);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("k_dgemm_dfma launch: ") + cudaGetErrorString(e));
    return MOA_ERR_CUDA;
  }
  return MOA_OK;
}

// K5 configs: bm, bn, stages (threads = bm*bn/(2*tn) + 32). 16 stages keep all of
// k <= 256 resident (one-shot); deeper k runs through the ring.
TileConfig kK5Configs[] = {
    // kernel, bm, bn, bk, stages, threads, ctas/SM, smem, eta
    {MOA_KERNEL_DGEMM_DFMA, 16, 32, 16, 16, K5Traits<16, 32, 2, 16>::kThreads, 2, K5Traits<16, 32, 2, 16>::kSmem, 1.0},
    {MOA_KERNEL_DGEMM_DFMA, 8, 32, 16, 16, K5Traits<8, 32, 2, 16>::kThreads, 4, K5Traits<8, 32, 2, 16>::kSmem, 1.0},
    {MOA_KERNEL_DGEMM_DFMA, 16, 64, 16, 8, K5Traits<16, 64, 4, 8>::kThreads, 2, K5Traits<16, 64, 4, 8>::kSmem, 1.0},
};

template <int BM, int BN, int TN, int ST>
int k5_occupancy() {
  if (k5_attrs<BM, BN, TN, ST, false, false>() != cudaSuccess) return 0;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_dgemm_dfma<BM, BN, TN, ST, false, false>,
                                                    K5Traits<BM, BN, TN, ST>::kThreads,
                                                    K5Traits<BM, BN, TN, ST>::kSmem) != cudaSuccess)
    return 0;
  return n;
}

}  // namespace

int dfma_tile_configs(const TileConfig** out) {
  static std::once_flag once;
  std::call_once(once, [] {
    RelaxedCapture relaxed_capture;
    const int o[3] = {k5_occupancy<16, 32, 2, 16>(), k5_occupancy<8, 32, 2, 16>(), k5_occupancy<16, 64, 4, 8>()};
    for (int i = 0; i < 3; ++i)
      if (o[i] > 0) kK5Configs[i].ctas_per_sm = o[i];
    cudaGetLastError();
  });
  *out = kK5Configs;
  return (int)(sizeof(kK5Configs) / sizeof(kK5Configs[0]));
}

int launch_dgemm_dfma(const moa_plan_t& plan, const GemmArgs& g, cudaStream_t stream) {
  if (plan.bm == 16 && plan.bn == 32 && plan.stages == 16) return launch_k5<16, 32, 2, 16>(plan, g, stream);
  if (plan.bm == 8 && plan.bn == 32 && plan.stages == 16) return launch_k5<8, 32, 2, 16>(plan, g, stream);
  if (plan.bm == 16 && plan.bn == 64 && plan.stages == 8) return launch_k5<16, 64, 4, 8>(plan, g, stream);
  set_error("no compiled K5 instance for this plan");
  return MOA_ERR_INVALID_SHAPE;
}

}  // namespace moa
