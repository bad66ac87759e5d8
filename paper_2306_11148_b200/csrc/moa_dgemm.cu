// moa_dgemm.cu — fp64 MoA-ONF GEMM kernels for sm_100a.
//
//   C[(i*p)+j] := sum_k A[(i*n)+k] * B[(k*p)+j]      (Eq. 3)
//
// K1 k_dgemm_tma   : persistent, warp-specialised. A producer warp (a warpgroup
//                    that donates its registers, for the 128x128 tile) streams
//                    the operands with TMA (cp.async.bulk.tensor, 128B swizzle)
//                    into an S-stage shared-memory ring guarded by mbarriers;
//                    1..8 consumer warps run DMMA.8x8x4 (mma.sync m8n8k4 f64) on
//                    register accumulators. Work: dynamically claimed tiles plus
//                    stream-K runs for the partial last wave, whose cut tiles
//                    continue the fma chain from the stored partial (bitwise);
//                    launched with programmatic dependent launch. The PEER
//                    instantiation also stores every final tile to up to 8
//                    further destinations (other ranks' C_full over NVLink):
//                    the all-gather of the row-lifted product fused into the
//                    epilogue (moa_gemm_lifted_gather / moa_gemm_scatter).
// K2 k_dgemm_generic: same arithmetic, plain predicated loads (odd n or p,
//                    pointers not 16-byte aligned — shapes TMA cannot describe).
//
// MoA mapping:
//  * Dimension lifting: i -> (tile row tm, warp row wm, atom a, lane
//    row); j -> (tile col tn, warp col wn, box bx, atom half h, lane col); the
//    sigma loop is split into 16-wide k-slabs ("the sigma loop is broken up
//    creating the block") whose partial sums stay in registers.
//  * Contiguous access: A is staged as BM rows x 16 k of row-major
//    segments (one 128 B run per row), B as 16 k-rows x 16 j boxes — rows of B,
//    never columns (Fig. 1: scalar A[i,k] times row k of B). No
//    transposed copy of anything exists.
//  * Summation order: for every C element, k = 0,1,...,n-1 strictly ascending
//    through k-slabs (ascending), DMMA k-steps (ascending) and the DMMA's
//    internal chain (measured on B200: DMMA.8x8x4 == fma chain k0..k3,
//    profiles/r01_fp64_probe.jsonl). Hence the result equals Fig. 3 ip.c with
//    its update fused (reading R3) bit for bit, and it depends only on n — any
//    row block computed alone equals the same rows of the full product.
//  * Bank conflicts: the DMMA fragment rows/columns are permuted (rho, pi below)
//    so that every ld.shared of a 128B-swizzled tile is conflict-free.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "moa_internal.h"
#include "moa_ptx.cuh"

namespace moa {
namespace {

using namespace ptx;

// Shared-memory fragment loads through plain C++ pointers into the __shared__
// window: the compiler emits LDS.64 / LDS.128, may schedule them freely, and
// still orders them after the mbarrier waits (which clobber "memory").
__device__ __forceinline__ double lds64(const uint8_t* s, uint32_t off) {
  return *reinterpret_cast<const double*>(s + off);
}
__device__ __forceinline__ double2 lds128(const uint8_t* s, uint32_t off) {
  return *reinterpret_cast<const double2*>(s + off);
}
// D = A(8x4) * B(4x8) + C, fp64 tensor core. Lane l: a = A[l>>2][l&3],
// b = B[l&3][l>>2], c/d = row l>>2, cols 2(l&3), 2(l&3)+1.
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// ------------------------- shared-memory tile layout -------------------------
// A stage: BM rows x 16 doubles (128 B per row), TMA SWIZZLE_128B: the 16-byte
//   chunk c of row r lives at chunk c ^ (r & 7).
// B stage: BN/16 boxes, each 16 k-rows x 16 doubles (2 KiB), same swizzle by k.
constexpr int kBK = 16;
constexpr int kRowBytes = kBK * 8;       // 128
constexpr int kBoxBytes = 16 * kRowBytes;  // 2048

// Per-lane fragment offsets (bytes), computed once.
//  rho(g) = ((g&3)<<1)|(g>>2): MMA row g -> physical row inside the 8-row atom.
//  pi(q)  = (q>>1)|((q&1)<<2): MMA col q -> physical 2-double pair inside a box;
//           the "even" atom takes the pair's first double, the "odd" atom the second.
struct FragOffsets {
  uint32_t a[4];  // per k-step s (4 per k-slab)
  uint32_t b[2];  // per (s & 1); add s*512 for the k-row base
  int rr;         // rho(lane>>2)
  int t;          // lane & 3
};
__device__ __forceinline__ FragOffsets make_offsets(int lane) {
  FragOffsets f;
  const int g = lane >> 2, t = lane & 3;
  const int rr = ((g & 3) << 1) | (g >> 2);
  const int piq = (g >> 1) | ((g & 1) << 2);
#pragma unroll
  for (int s = 0; s < 4; ++s) f.a[s] = rr * kRowBytes + ((((2 * s) + (t >> 1)) ^ rr) << 4) + ((t & 1) << 3);
#pragma unroll
  for (int s = 0; s < 2; ++s) f.b[s] = t * kRowBytes + ((piq ^ (4 * s + t)) << 4);
  f.rr = rr;
  f.t = t;
  return f;
}

template <int MA, int NBOX>
struct Acc {
  double v[MA][NBOX][2][2];  // [A atom][box][even/odd atom][C pair]
};

template <int MA, int NBOX>
__device__ __forceinline__ void acc_zero(Acc<MA, NBOX>& c) {
#pragma unroll
  for (int a = 0; a < MA; ++a)
#pragma unroll
    for (int b = 0; b < NBOX; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) c.v[a][b][h][0] = c.v[a][b][h][1] = 0.0;
}

// One 16-wide k-slab: 4 k-steps (ascending) x (MA x 2*NBOX) DMMA atoms.
// a_base: this warp's 8*MA rows of the A stage; b_base: its first B box.
template <int MA, int NBOX>
__device__ __forceinline__ void mma_slab(Acc<MA, NBOX>& c, const uint8_t* a_base, const uint8_t* b_base,
                                         const FragOffsets& f) {
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    double af[MA];
    double2 bf[NBOX];
#pragma unroll
    for (int a = 0; a < MA; ++a) af[a] = lds64(a_base, a * 8 * kRowBytes + f.a[s]);
#pragma unroll
    for (int b = 0; b < NBOX; ++b) bf[b] = lds128(b_base, b * kBoxBytes + s * 4 * kRowBytes + f.b[s & 1]);
#pragma unroll
    for (int a = 0; a < MA; ++a)
#pragma unroll
      for (int b = 0; b < NBOX; ++b) {
        dmma(c.v[a][b][0], af[a], bf[b].x);
        dmma(c.v[a][b][1], af[a], bf[b].y);
      }
  }
}

// Write the warp's 8*MA x (16*NBOX) block of C. Lane holds, for atom a and box b,
// row rho(g) and columns {2t, 2t+1} (pair 0) and {2t+8, 2t+9} (pair 1).
// Accumulate mode ("the addition loop to add up the blocks", across
// launches): start the chain from the C already in memory instead of +0. Because
// DMMA continues an fma chain from its C operand, a sequence of k-panel launches
// reproduces the single-launch result bit for bit. Same fragment map as store_acc.
template <int MA, int NBOX, bool kVec>
__device__ __forceinline__ void load_acc(Acc<MA, NBOX>& c, const double* __restrict__ C, int64_t m, int64_t p,
                                         int64_t ldc, int64_t row0, int64_t col0, const FragOffsets& f) {
#pragma unroll
  for (int a = 0; a < MA; ++a) {
    const int64_t r = row0 + a * 8 + f.rr;
    const double* crow = C + r * ldc;
#pragma unroll
    for (int b = 0; b < NBOX; ++b) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int64_t col = col0 + b * 16 + 2 * f.t + 8 * q;
        // scalar loads straight into the two atoms' accumulators (a double2 load
        // would pair registers of different DMMA operands and cost copies)
        double lo = 0.0, hi = 0.0;
        if (r < m) {
          if (col < p) lo = __ldcg(crow + col);  // L2: may be another CTA's partial
          if (col + 1 < p) hi = __ldcg(crow + col + 1);
        }
        c.v[a][b][0][q] = lo;
        c.v[a][b][1][q] = hi;
      }
    }
  }
}

template <int MA, int NBOX, bool kVec>
__device__ __forceinline__ void store_acc(const Acc<MA, NBOX>& c, double* __restrict__ C, int64_t m, int64_t p,
                                          int64_t ldc, int64_t row0, int64_t col0, const FragOffsets& f) {
#pragma unroll
  for (int a = 0; a < MA; ++a) {
    const int64_t r = row0 + a * 8 + f.rr;
    if (r >= m) continue;
    double* crow = C + r * ldc;
#pragma unroll
    for (int b = 0; b < NBOX; ++b) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int64_t col = col0 + b * 16 + 2 * f.t + 8 * q;
        const double lo = c.v[a][b][0][q], hi = c.v[a][b][1][q];
        if (kVec) {
          if (col < p) *reinterpret_cast<double2*>(crow + col) = make_double2(lo, hi);
        } else {
          if (col < p) crow[col] = lo;
          if (col + 1 < p) crow[col + 1] = hi;
        }
      }
    }
  }
}

#ifdef MOA_K1_PHASES
// PHASE-BREAKDOWN EXPERIMENT (variant builds with -DMOA_K1_PHASES only; the product
// never defines it): per CTA, %globaltimer (ns) at kernel entry, after
// griddepcontrol.wait, at the producer's first TMA issue, and for consumer warp 0 /
// lane 0 the first slab's landing, the summed full-barrier waits, the end of the last
// slab and the end of the store. Read back with moa_k1_phases_read (tools/experiments/phases.py).
__device__ unsigned long long g_ph[1024 * 8];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define MOA_PH(slot, v) \
  do {                 \
    if (blockIdx.x < 1024) g_ph[blockIdx.x * 8 + (slot)] = (v); \
  } while (0)
#else
#define MOA_PH(slot, v) \
  do {                 \
  } while (0)
#endif

// ------------------------------- K1: TMA + WS --------------------------------
// Register file is split per SM sub-partition (warp w -> SMSP w % 4, 16384
// registers each). With 8 consumer warps a lone producer warp would put 3 warps
// on one SMSP and cap every thread at 168 registers (the 64 fp64 accumulators
// alone need 128), so the producer becomes a full warpgroup that gives its
// registers to the consumers with setmaxnreg: per SMSP 1 x 40 + 2 x 232 regs.
constexpr int kK1OneShotGroup = 4;  // k-slabs per barrier of a one-shot latency tile
template <int BM, int BN, int WARPS_M, int WARPS_N, int STAGES>
struct K1Traits {
  static constexpr int kConsumerWarps = WARPS_M * WARPS_N;
  static constexpr int kNBoxW = BN / WARPS_N / 16;
  // Only the 32x64 warp tile (64 accumulators) needs the producer's registers.
  static constexpr int kProducerWarps = (kConsumerWarps >= 8 && kNBoxW == 4) ? 4 : 1;
  // 32x16 warp tiles fit 2 CTAs/SM; the 1-2 warp latency tiles (<= 16 rows per
  // warp) are meant to pack many CTAs per SM
  static constexpr int kMinBlocks = kNBoxW >= 2 ? 1 : (BM / WARPS_M <= 16 ? 8 : 2);
  // One-shot latency tiles: a 16-stage ring holds all of k <= 256 of a tile, so when a
  // CTA owns exactly one tile the producer issues every load up front (one barrier per
  // kK1OneShotGroup slabs) and nothing is ever released or refilled; the consumers run
  // the whole k-chain with kK1OneShotGroup slabs between barrier waits.
  static constexpr bool kOneShotCfg = BM * BN <= 32 * 32 && STAGES >= 16;
  static constexpr bool kSetMaxNReg = kProducerWarps == 4;
  static constexpr int kProducerRegs = 40;  // 40 + 2 x 232 per SMSP; also the CTA pool: 4 x 40 + 8 x 232 = 12 x 168
  static constexpr int kConsumerRegs = 232;
  static constexpr int kThreads = (kConsumerWarps + kProducerWarps) * 32;
  static_assert(!kSetMaxNReg || (kProducerRegs + 2 * kConsumerRegs) * 32 <= 16384, "per-SMSP register budget");
  // setmaxnreg moves registers inside the CTA's pool (every warp starts with the
  // launch count, 65536 / threads rounded down to 8): a consumer .inc beyond what the
  // producers' .dec released waits forever (a hang, not an error)
  static_assert(!kSetMaxNReg || kProducerWarps * kProducerRegs + kConsumerWarps * kConsumerRegs <=
                                    (kProducerWarps + kConsumerWarps) * ((65536 / ((kConsumerWarps + kProducerWarps) * 32)) & ~7),
                "setmaxnreg: consumers ask for more registers than the producers release");
  static constexpr int kNBox = BN / WARPS_N / 16;
  static constexpr int kMA = BM / WARPS_M / 8;  // A atoms (8 rows each) per warp
  static constexpr int kABytes = BM * kRowBytes;
  static constexpr int kBBytes = BN * kRowBytes;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kSmem = 1024 /*align slack*/ + STAGES * kStageBytes + 2 * STAGES * 8;  // + full/empty barriers
  static_assert(BM == 8 * kMA * WARPS_M && (kMA == 1 || kMA == 2 || kMA == 4), "warp tile is 8, 16 or 32 rows");
  static_assert(BN % (16 * WARPS_N) == 0, "warp tile is a whole number of 16-column boxes");
};

// One piece of work for a consumer warp: tile (row0, col0), k-slabs [k0, k1). With
// `load` the chain starts from the C in memory (accumulate mode, or the stored
// low-k partial of a split tile), else from +0: the loads are predicated off by
// passing m = 0, so there is ONE copy of the slab loop in the kernel (a branch
// between load_acc and acc_zero once cost 5.4% in register copies).
template <int MA, int NBOX, int STAGES, int STAGE_BYTES, int A_BYTES>
__device__ __forceinline__ void consume_piece(Acc<MA, NBOX>& acc, uint32_t a_s, uint32_t b_s, uint32_t full0, uint32_t empty0,
                                              int& stage, uint32_t& phase,
                                              double* __restrict__ C, int64_t m, int64_t p, int64_t ldc,
                                              int64_t row0, int64_t col0, int wm, int wn, int k0, int k1, bool load,
                                              const FragOffsets& f, int lane) {
  load_acc<MA, NBOX, true>(acc, C, load ? m : 0, p, ldc, row0 + wm * 8 * MA, col0 + wn * NBOX * 16, f);
#ifdef MOA_K1_PHASES
  unsigned long long waited = 0, tw0 = 0;
  const bool ph = threadIdx.x == 0;
#endif
  for (int kt = k0; kt < k1; ++kt) {
#ifdef MOA_K1_PHASES
    if (ph) tw0 = gtime();
#endif
    mbar_wait(full0 + 8 * stage, phase);  // (ptxas reconverges the spin with BSSY/BSYNC before the DMMAs)
#ifdef MOA_K1_PHASES
    if (ph) {
      const unsigned long long tw1 = gtime();
      waited += tw1 - tw0;
      if (kt == k0) MOA_PH(3, tw1);
    }
#endif
    // a_s / b_s: this warp's A rows and B boxes in stage 0 (shared-window addresses,
    // computed once by the caller and kept opaque); without them ptxas re-derived the
    // window base (S2R SR_CgaCtaId, S2R SR_TID.X and ~20 integer ops) at every slab, on
    // the critical path between the stage wait and the first fragment loads
    const uint32_t so = (uint32_t)stage * STAGE_BYTES;
    mma_slab(acc, static_cast<const uint8_t*>(__cvta_shared_to_generic(a_s + so)),
             static_cast<const uint8_t*>(__cvta_shared_to_generic(b_s + so)), f);
    // WAR across proxies: these generic-proxy LDS reads must be ordered before the
    // producer's next TMA (async-proxy) write of this stage. The arrive's .release
    // alone does not do it (ptxas even hoists the arrive above the slab's last
    // DMMAs): without this fence whole warp tiles were computed from overwritten
    // operands, rarely under dynamic scheduling, often under stream-K.
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * stage);
    if (++stage == STAGES) {
      stage = 0;
      phase ^= 1u;
    }
  }
#ifdef MOA_K1_PHASES
  if (ph) {
    MOA_PH(4, waited);
    MOA_PH(5, gtime());
  }
#endif
  store_acc<MA, NBOX, true>(acc, C, m, p, ldc, row0 + wm * 8 * MA, col0 + wn * NBOX * 16, f);
#ifdef MOA_K1_PHASES
  if (ph) MOA_PH(6, gtime());
#endif
}

// ACC: start every tile's chain from the C in memory (moa_gemm_acc k-panel chains).
//
// Work assignment: every CTA walks its own static schedule (StaticSched: whole
// tiles cta, cta + G, ... below the stream-K region, then its stream-K run r = cta),
// computed identically by the producer and by every consumer warp, so nothing about
// the schedule crosses shared memory (round 1 published piece descriptors with
// plain shared stores ordered by the stage mbarrier: correct, but the one hazard
// compute-sanitizer racecheck reported, since it does not model mbarriers). The
// wave gate (producer) keeps the CTAs of a wave in k-lockstep, which round 1's
// dynamic tile claiming only approximated.
// launch mode bits (host -> K1)
constexpr int kK1WaveGate = 2;  // wave gate (see the producer)

// One CTA's static schedule: whole tiles cta, cta + G, ... below
// `first` (the stream-K region's start, or all tiles), then its stream-K run r = cta:
// head first, whole run tiles, tail last (the order the hand-off argument of
// moa_ptx.cuh needs).
struct StaticSched {
  // tile indices fit in 32 bits: C (>= 256 fp64 elements per tile) fits in HBM
  int32_t t, first, G, w, hb, ta, f1;
  int32_t hk, tk, ktiles, st;
  __device__ __forceinline__ StaticSched(int64_t tiles, int ktiles_, int64_t G_, int64_t cta, bool sk)
      : t((int32_t)cta), first((int32_t)(sk ? sk_first_tile(tiles, G_) : tiles)), G((int32_t)G_), w(0), hb(0),
        ta(0), f1(0), hk(0), tk(0), ktiles(ktiles_), st(sk ? 0 : 3) {
    if (sk) {
      const SkRun q = sk_run(tiles, ktiles_, G_, cta);
      hb = (int32_t)q.hb, ta = (int32_t)q.ta, w = (int32_t)q.f0, f1 = (int32_t)q.f1, hk = q.hk, tk = q.tk;
    }
  }
  __device__ __forceinline__ bool next(int64_t& tile, int& k0, int& k1, int& run) {
    if (t < first) {
      tile = t;
      t += G;
      k0 = 0, k1 = ktiles, run = -1;
      return true;
    }
    const int r = t % G;  // = cta
    if (st == 0) {  // head of the run
      st = 1;
      if (hk > 0) {
        tile = hb, k0 = 0, k1 = hk, run = r;
        return true;
      }
    }
    if (st == 1) {  // whole tiles of the run, then its tail
      if (w < f1) {
        tile = w++, k0 = 0, k1 = ktiles, run = r;
        return true;
      }
      st = 2;
      if (tk > 0) {
        tile = ta, k0 = tk, k1 = ktiles, run = r;
        return true;
      }
    }
    st = 3;
    return false;
  }
};

//
// PEER: the fused GEMM -> all-gather epilogue (moa_gemm_lifted_gather). Every FINAL
// tile (whole tile, or the tail of a stream-K cut tile) is also stored, straight
// from the accumulator registers, to each peers.dst[d] at the same (row, col) —
// NVLink peer stores into the other ranks' C_full, overlapping the remaining
// tiles' DMMA work; stream-K head partials stay local.
template <int BM, int BN, int WARPS_M, int WARPS_N, int STAGES, bool ACC, bool PEER>
__global__ void __launch_bounds__(K1Traits<BM, BN, WARPS_M, WARPS_N, STAGES>::kThreads,
                                  K1Traits<BM, BN, WARPS_M, WARPS_N, STAGES>::kMinBlocks)
    k_dgemm_tma(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                double* __restrict__ C, int64_t m, int64_t n, int64_t p, int64_t ldc,
                int64_t tiles_m, int64_t tiles_n, int group, unsigned int* __restrict__ flags,
                unsigned int* __restrict__ issued, const __grid_constant__ PeerDst peers, int mode) {
  using Tr = K1Traits<BM, BN, WARPS_M, WARPS_N, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t sbase = (raw + 1023u) & ~1023u;  // SWIZZLE_128B needs 1024-B alignment
  const uint8_t* sptr = smem_raw + (sbase - raw);
  const uint32_t full0 = sbase + STAGES * Tr::kStageBytes;
  const uint32_t empty0 = full0 + STAGES * 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ktiles = (int)((n + kBK - 1) / kBK);
#ifdef MOA_K1_PHASES
  if (threadIdx.x == 0) MOA_PH(0, gtime());
#endif

  // Programmatic dependent launch: this prologue may run while the previous grid in
  // the stream drains; griddepcontrol.wait (below) orders every global-memory access
  // after that grid's completion, so stream semantics are unchanged. Each thread
  // signals launch_dependents only when it is done, so the next grid's CTAs are
  // placed as this grid's SMs free up (signalling at the start let small CTAs of the
  // next grids pile onto busy SMs: N=512 went from 15 to 23 us).
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, Tr::kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef MOA_K1_PHASES
  if (threadIdx.x == 0) MOA_PH(1, gtime());
#endif

  if (warp >= Tr::kConsumerWarps) {
    // ----------------------------- producer ---------------------------------
    if constexpr (Tr::kSetMaxNReg) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(Tr::kProducerRegs));
    if (warp == Tr::kConsumerWarps && lane == 0) {
      prefetch_tmap(&tmA);
      prefetch_tmap(&tmB);
      if constexpr (Tr::kOneShotCfg) {
        if (ktiles <= STAGES && tiles_m * tiles_n <= (int64_t)gridDim.x && !flags) {  // one-shot (see K1Traits)
          if (blockIdx.x < tiles_m * tiles_n) {
            int64_t tm, tn;
            tile_coords32(blockIdx.x, tiles_m, tiles_n, group, tm, tn);
            const int row0 = (int)(tm * BM), col0 = (int)(tn * BN);
            for (int g = 0; g * kK1OneShotGroup < ktiles; ++g) {
              const int k0 = g * kK1OneShotGroup, k1 = min(ktiles, k0 + kK1OneShotGroup);
              const uint32_t fb = full0 + 8 * g;
              mbar_arrive_expect_tx(fb, (k1 - k0) * Tr::kStageBytes);
              for (int kt = k0; kt < k1; ++kt) {
                const uint32_t sa = sbase + kt * Tr::kStageBytes;
                tma_load_2d(sa, &tmA, fb, kt * kBK, row0);
#pragma unroll
                for (int b = 0; b < BN / 16; ++b)
                  tma_load_2d(sa + Tr::kABytes + b * kBoxBytes, &tmB, fb, col0 + 16 * b, kt * kBK);
              }
            }
          }
          asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
          return;
        }
      }
      int stage = 0;
      uint32_t phase = 0;
      auto emit = [&](int64_t t, int k0, int k1, int run) {
        int64_t tm, tn;
        if constexpr (BM * BN <= 32 * 32)
          tile_coords32(t, tiles_m, tiles_n, group, tm, tn);
        else
          tile_coords(t, tiles_m, tiles_n, group, tm, tn);
        const int row0 = (int)(tm * BM), col0 = (int)(tn * BN);
        for (int kt = k0; kt < k1; ++kt) {
          mbar_wait(empty0 + 8 * stage, phase ^ 1u);
          const uint32_t fb = full0 + 8 * stage;
#ifdef MOA_K1_PHASES
          if (kt == 0) MOA_PH(2, gtime());
#endif
          mbar_arrive_expect_tx(fb, Tr::kStageBytes);
          const uint32_t sa = sbase + stage * Tr::kStageBytes;
          tma_load_2d(sa, &tmA, fb, kt * kBK, row0);
#pragma unroll
          for (int b = 0; b < BN / 16; ++b)
            tma_load_2d(sa + Tr::kABytes + b * kBoxBytes, &tmB, fb, col0 + 16 * b, kt * kBK);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      };
      const int64_t tiles = tiles_m * tiles_n, G = gridDim.x;
      // Wave gate: the tiles of wave t/G start only once every tile of the earlier
      // waves has had all its loads issued, so the CTAs of a wave walk k in step and
      // share each A/B k-slab through L2 instead of drifting apart over many waves
      // (which re-read the panels from DRAM). The last issue precedes the last
      // consume by the ring depth, so the gate opens inside the producer's lead.
      const bool gate = (mode & kK1WaveGate) && issued;
      StaticSched sc(tiles, ktiles, G, blockIdx.x, flags != nullptr);
      int64_t t;
      int k0, k1, run;
      while (sc.next(t, k0, k1, run)) {
        if (gate) wave_gate(issued, (unsigned)min(t / G * G, (int64_t)sc.first));
        emit(t, k0, k1, run);
        if (gate && run < 0) atomicAdd(issued, 1u);  // all loads of a whole tile issued
      }
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    return;
  }

  // ------------------------------- consumers ---------------------------------
  if constexpr (Tr::kSetMaxNReg) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(Tr::kConsumerRegs));
  const int wm = warp % WARPS_M, wn = warp / WARPS_M;
  FragOffsets f = make_offsets(lane);
  // Opaque copies: computed once, kept live. Without this ptxas rematerialised the
  // offsets (S2R tid + ~25 integer ops) in every slab.
#pragma unroll
  for (int s = 0; s < 4; ++s) asm volatile("" : "+r"(f.a[s]));
  asm volatile("" : "+r"(f.b[0]), "+r"(f.b[1]));
  uint32_t a_s = sbase + wm * 8 * Tr::kMA * kRowBytes, b_s = sbase + Tr::kABytes + wn * Tr::kNBox * kBoxBytes;
  asm volatile("" : "+r"(a_s), "+r"(b_s));
  Acc<Tr::kMA, Tr::kNBox> acc;
  if constexpr (Tr::kOneShotCfg) {
    if (ktiles <= STAGES && tiles_m * tiles_n <= (int64_t)gridDim.x && !flags) {  // one-shot (see K1Traits)
      if (blockIdx.x < tiles_m * tiles_n) {
        int64_t tm, tn;
        tile_coords32(blockIdx.x, tiles_m, tiles_n, group, tm, tn);
        const int64_t r0 = tm * BM + wm * 8 * Tr::kMA, c0 = tn * BN + wn * Tr::kNBox * 16;
        load_acc<Tr::kMA, Tr::kNBox, true>(acc, C, ACC ? m : 0, p, ldc, r0, c0, f);
        for (int g = 0; g * kK1OneShotGroup < ktiles; ++g) {
          mbar_wait(full0 + 8 * g, 0);
#pragma unroll
          for (int j = 0; j < kK1OneShotGroup; ++j) {
            const int kt = g * kK1OneShotGroup + j;
            if (kt < ktiles) {
              const uint8_t* sa = sptr + kt * Tr::kStageBytes;
              mma_slab(acc, sa + wm * 8 * Tr::kMA * kRowBytes, sa + Tr::kABytes + wn * Tr::kNBox * kBoxBytes, f);
            }
          }
        }
        store_acc<Tr::kMA, Tr::kNBox, true>(acc, C, m, p, ldc, r0, c0, f);
        if constexpr (PEER)
          for (int d = 0; d < peers.nd; ++d)
            store_acc<Tr::kMA, Tr::kNBox, true>(acc, reinterpret_cast<double*>(peers.dst[d]), m, p, ldc, r0, c0, f);
      }
      asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
      return;
    }
  }
  int stage = 0;
  uint32_t phase = 0;
  StaticSched sc(tiles_m * tiles_n, ktiles, gridDim.x, blockIdx.x, flags != nullptr);
  for (;;) {
    int64_t tm, tn;
    int k0, k1, run;
    int64_t t;
    if (!sc.next(t, k0, k1, run)) break;
    // (the 64-bit map: a 32-bit one was measured 0.6% slower at 8192^3 through the
    // consumers' code generation, profiles/r02/ab_bisect*.jsonl)
    if constexpr (BM * BN <= 32 * 32)  // latency tiles (moa_ptx.cuh tile_coords32)
      tile_coords32(t, tiles_m, tiles_n, group, tm, tn);
    else
      tile_coords(t, tiles_m, tiles_n, group, tm, tn);
    const bool head = k1 < ktiles, tail = k0 > 0;  // stream-K split pieces
    if (tail) split_wait(flags + run, Tr::kConsumerWarps, lane);
    consume_piece<Tr::kMA, Tr::kNBox, STAGES, Tr::kStageBytes, Tr::kABytes>(
        acc, a_s, b_s, full0, empty0, stage, phase, C, m, p, ldc, tm * BM, tn * BN, wm, wn, k0, k1, ACC || tail, f, lane);
    if (head) split_signal(flags + run + 1, lane);  // low-k partial of this tile -> run + 1
    if (tail) split_release(flags + run, 2 * Tr::kConsumerWarps, lane);
    if constexpr (PEER) {
      if (!head)
        for (int d = 0; d < peers.nd; ++d)
          store_acc<Tr::kMA, Tr::kNBox, true>(acc, reinterpret_cast<double*>(peers.dst[d]), m, p, ldc,
                                              tm * BM + wm * 8 * Tr::kMA, tn * BN + wn * Tr::kNBox * 16, f);
    }
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ------------------------------ K2: generic ----------------------------------
template <int BM, int BN, int WARPS_M, int WARPS_N>
__global__ void __launch_bounds__(WARPS_M* WARPS_N * 32)
    k_dgemm_generic(const double* __restrict__ A, const double* __restrict__ B, double* __restrict__ C, int64_t m,
                    int64_t n, int64_t p, int64_t lda, int64_t ldb, int64_t ldc, int accumulate, int64_t tiles_m,
                    int64_t tiles_n, int group, const __grid_constant__ PeerDst peers) {
  constexpr int kNBox = BN / WARPS_N / 16;
  constexpr int kThreads = WARPS_M * WARPS_N * 32;
  __shared__ __align__(1024) uint8_t sm[(BM + BN) * kRowBytes];
  const uint8_t* sa = sm;
  const uint8_t* sb = sm + BM * kRowBytes;
  double* sA = reinterpret_cast<double*>(sm);
  double* sB = reinterpret_cast<double*>(sm + BM * kRowBytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp % WARPS_M, wn = warp / WARPS_M;
  const FragOffsets f = make_offsets(lane);
  const int64_t tiles = tiles_m * tiles_n;
  Acc<4, kNBox> acc;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    int64_t tm, tn;
    tile_coords(t, tiles_m, tiles_n, group, tm, tn);
    const int64_t row0 = tm * BM, col0 = tn * BN;
    if (accumulate)
      load_acc<4, kNBox, false>(acc, C, m, p, ldc, row0 + wm * 32, col0 + wn * kNBox * 16, f);
    else
      acc_zero(acc);
    for (int64_t k0 = 0; k0 < n; k0 += kBK) {
      __syncthreads();
      for (int e = threadIdx.x; e < BM * kBK; e += kThreads) {  // A: row r, k
        const int r = e / kBK, k = e % kBK;
        const int64_t gi = row0 + r, gk = k0 + k;
        const double v = (gi < m && gk < n) ? A[gi * lda + gk] : 0.0;
        sA[(r * kRowBytes + (((k >> 1) ^ (r & 7)) << 4) + ((k & 1) << 3)) / 8] = v;
      }
      for (int e = threadIdx.x; e < kBK * BN; e += kThreads) {  // B: k-row, col
        const int k = e / BN, c = e % BN;
        const int64_t gk = k0 + k, gj = col0 + c;
        const double v = (gk < n && gj < p) ? B[gk * ldb + gj] : 0.0;
        const int box = c >> 4, cc = c & 15;
        sB[(box * kBoxBytes + k * kRowBytes + (((cc >> 1) ^ (k & 7)) << 4) + ((cc & 1) << 3)) / 8] = v;
      }
      __syncthreads();
      mma_slab(acc, sa + wm * 32 * kRowBytes, sb + wn * kNBox * kBoxBytes, f);
    }
    store_acc<4, kNBox, false>(acc, C, m, p, ldc, row0 + wm * 32, col0 + wn * kNBox * 16, f);
    for (int d = 0; d < peers.nd; ++d)  // fused gather epilogue (see K1's PEER)
      store_acc<4, kNBox, false>(acc, reinterpret_cast<double*>(peers.dst[d]), m, p, ldc, row0 + wm * 32,
                                 col0 + wn * kNBox * 16, f);
  }
}

// ------------------------------ host helpers ---------------------------------
bool encode_2d_f64(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  return encode_2d(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, base, rows, cols, 16, box_rows, CU_TENSOR_MAP_SWIZZLE_128B,
                   ld);
}

// Opt in to the full dynamic smem per CTA and the maximum shared-memory carveout:
// without the carveout the driver picked a smaller L1/smem split and the small
// tiles fit fewer CTAs per SM than their smem allows (32x32x3: 6 instead of 8).
template <int BM, int BN, int WM, int WN, int ST, bool ACC, bool PEER>
cudaError_t k1_attrs() {
  auto kern = k_dgemm_tma<BM, BN, WM, WN, ST, ACC, PEER>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       K1Traits<BM, BN, WM, WN, ST>::kSmem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  return e;
}

// The wave gate pays where CTA drift would otherwise cost DRAM re-reads: launches of
// many waves. Measured: 32768^3 (443 waves) DRAM 2.6 TB -> 418 GB, -15% J/GEMM, +0.2%
// time; 16384^3 (110 waves) 72 -> 55 GB, -3.5% J, equal time; 8192^3 (27.7 waves) no
// traffic change and 0.5% slower gated, shallow k (65536x512x512, 13.8 waves) 0.1-0.3%
// slower gated (profiles/r02/wave_gate.jsonl, ab_gate_shallow.jsonl). So it is on from
// kK1GateWaves whole-tile waves up. MOA_K1_WAVE_GATE=0 / =1 force it off / on (A/B).
constexpr int64_t kK1GateWaves = 48;
int k1_wave_gate_mode() {  // 0 off, 1 on, 2 by size
  static const int mode = [] {
    const char* e = getenv("MOA_K1_WAVE_GATE");
    return (e && e[0] == '0') ? 0 : (e && e[0] == '1') ? 1 : 2;
  }();
  return mode;
}

template <int BM, int BN, int WM, int WN, int ST>
int launch_k1(const moa_plan_t& plan, const GemmArgs& g, cudaStream_t stream) {
  using Tr = K1Traits<BM, BN, WM, WN, ST>;
  CUtensorMap ta, tb;
  const int64_t m = g.m, n = g.n, p = g.p;
  if (!encode_2d_f64(&ta, g.A, m, n, g.lda, BM) || !encode_2d_f64(&tb, g.B, n, p, g.ldb, 16)) return MOA_ERR_CUDA;
  double* C = (double*)g.C;
  const bool peer = g.peers && g.peers->nd > 0;
  auto kern = g.accumulate
                  ? (peer ? k_dgemm_tma<BM, BN, WM, WN, ST, true, true> : k_dgemm_tma<BM, BN, WM, WN, ST, true, false>)
                  : (peer ? k_dgemm_tma<BM, BN, WM, WN, ST, false, true> : k_dgemm_tma<BM, BN, WM, WN, ST, false, false>);
  PeerDst peers{};
  if (peer) peers = *g.peers;
  static std::once_flag once;  // per instantiation
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [&] {
    RelaxedCapture relaxed_capture;
    attr_err = k1_attrs<BM, BN, WM, WN, ST, false, false>();
    if (attr_err == cudaSuccess) attr_err = k1_attrs<BM, BN, WM, WN, ST, true, false>();
    if (attr_err == cudaSuccess) attr_err = k1_attrs<BM, BN, WM, WN, ST, false, true>();
    if (attr_err == cudaSuccess) attr_err = k1_attrs<BM, BN, WM, WN, ST, true, true>();
  });
  if (attr_err != cudaSuccess) {
    set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(attr_err));
    return MOA_ERR_CUDA;
  }
  // Schedule (see the kernel): whole tiles by static stride, plus stream-K runs when
  // the last wave is partial; a counter carries the wave gate's issue count.
  unsigned int *flags = nullptr, *ctr = nullptr;
  const int gmode = k1_wave_gate_mode();
  bool gate = false;
  if (plan.tiles > plan.grid) {
    const bool sk = use_stream_k(plan.tiles, plan.grid);
    if (sk && !acquire_split_flags((unsigned)plan.grid + 1, stream, &flags)) return MOA_ERR_CUDA;
    const int64_t first = sk ? sk_first_tile(plan.tiles, plan.grid) : plan.tiles;
    // the gate's issue counter, when there are at least two waves of whole tiles
    gate = gmode == 1 ? first >= 2 * plan.grid : gmode == 2 && first >= kK1GateWaves * plan.grid;
    if (gate && !acquire_tile_counter(stream, &ctr)) return MOA_ERR_CUDA;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)plan.grid);
  cfg.blockDim = dim3(Tr::kThreads);
  cfg.dynamicSmemBytes = Tr::kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (see the kernel prologue)
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // one tile per CTA and all of k resident in the ring: no stage is ever refilled
  int mode = 0;
  if (ctr && gate) mode |= kK1WaveGate;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ta, tb, C, m, n, p, g.ldc, plan.tiles_m, plan.tiles_n,
                                     (int)plan.raster_group, flags, ctr, peers, mode);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("k_dgemm_tma launch: ") + cudaGetErrorString(e));
    return MOA_ERR_CUDA;
  }
  return MOA_OK;
}

// The chooser's candidate lifted blocks. ctas_per_sm is refined at first use
// from the occupancy API (registers are what limit it; see K1Traits). eta is the
// per-tile efficiency relative to 128x128, measured once at N=16384 where wave
// quantisation vanishes (tools/small_n.py -> profiles/r01_small_n.json: 0.9806 /
// 0.9614 / 0.9574 / 0.9665 of peak) — a property of the tile config, not a
// per-shape tuning. 64x32 (4-warp CTAs) is compiled for the block-size experiment
// but not offered to the chooser (eta 0): with one CTA per SM it leaves one warp per
// sub-partition and is erratic (N=768: 44 vs 31 us for 64x64; N=640: 28.7 vs 26.8),
// and the latency tiles below cover the sizes where its finer grain helped.
TileConfig kK1Configs[] = {
    // kernel, bm, bn, bk, stages, threads, ctas/SM, smem, eta
    {MOA_KERNEL_DGEMM_TMA, 128, 128, 16, 6, K1Traits<128, 128, 4, 2, 6>::kThreads, 1, K1Traits<128, 128, 4, 2, 6>::kSmem, 1.00},
    {MOA_KERNEL_DGEMM_TMA, 128, 64, 16, 4, K1Traits<128, 64, 4, 2, 4>::kThreads, 1, K1Traits<128, 64, 4, 2, 4>::kSmem, 0.980},
    {MOA_KERNEL_DGEMM_TMA, 64, 64, 16, 4, K1Traits<64, 64, 2, 4, 4>::kThreads, 2, K1Traits<64, 64, 2, 4, 4>::kSmem, 0.976},
    {MOA_KERNEL_DGEMM_TMA, 64, 32, 16, 4, K1Traits<64, 32, 2, 2, 4>::kThreads, 4, K1Traits<64, 32, 2, 2, 4>::kSmem, 0.0},
    // latency tiles (16x16 outputs per warp): eta here is the latency-regime factor;
    // the chooser considers them only for tiny problems (moa_host.cpp choose()).
    // 16x32 first: it wins the ties (N=512: 13.2 vs 22.3 us for 16x16). (A 16-stage
    // one-shot form, all of k <= 256 resident, was measured and dropped: 256^3 5.92 vs
    // 5.79 us for 16x16, 512^3 24.7 vs 13.2 us: profiles/r02/small_n_k5_dfma.json.)
    {MOA_KERNEL_DGEMM_TMA, 16, 32, 16, 4, K1Traits<16, 32, 1, 2, 4>::kThreads, 8, K1Traits<16, 32, 1, 2, 4>::kSmem, 1.0},
    {MOA_KERNEL_DGEMM_TMA, 16, 16, 16, 4, K1Traits<16, 16, 1, 1, 4>::kThreads, 8, K1Traits<16, 16, 1, 1, 4>::kSmem, 1.0},
    // latency tiles with 8x16 warp tiles (2 DMMA chains per warp, spread over more SM
    // sub-partitions); 8 stages ("stages" also tells them apart in a plan)
    {MOA_KERNEL_DGEMM_TMA, 16, 32, 16, 8, K1Traits<16, 32, 2, 2, 8>::kThreads, 4, K1Traits<16, 32, 2, 2, 8>::kSmem, 0.0},
    {MOA_KERNEL_DGEMM_TMA, 16, 16, 16, 8, K1Traits<16, 16, 2, 1, 8>::kThreads, 8, K1Traits<16, 16, 2, 1, 8>::kSmem, 0.0},
    // their one-shot twins (16 stages: all of k <= 256 resident, no stage release)
    {MOA_KERNEL_DGEMM_TMA, 16, 32, 16, 16, K1Traits<16, 32, 2, 2, 16>::kThreads, 2, K1Traits<16, 32, 2, 2, 16>::kSmem, 0.0},
    {MOA_KERNEL_DGEMM_TMA, 16, 16, 16, 16, K1Traits<16, 16, 2, 1, 16>::kThreads, 3, K1Traits<16, 16, 2, 1, 16>::kSmem, 0.0},
};
TileConfig kK2Configs[] = {
    {MOA_KERNEL_DGEMM_GENERIC, 64, 64, 16, 1, 128, 4, (64 + 64) * kRowBytes, 0.5},
};

template <int BM, int BN, int WM, int WN, int ST>
int k1_occupancy() {
  using Tr = K1Traits<BM, BN, WM, WN, ST>;
  auto kern = k_dgemm_tma<BM, BN, WM, WN, ST, false, false>;
  if (k1_attrs<BM, BN, WM, WN, ST, false, false>() != cudaSuccess) return 0;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, Tr::kThreads, Tr::kSmem) != cudaSuccess) return 0;
  return n;
}

void refine_occupancy() {
  static std::once_flag once;
  std::call_once(once, [] {
    RelaxedCapture relaxed_capture;
    int o[10] = {k1_occupancy<128, 128, 4, 2, 6>(),  k1_occupancy<128, 64, 4, 2, 4>(),  k1_occupancy<64, 64, 2, 4, 4>(),
                 k1_occupancy<64, 32, 2, 2, 4>(),    k1_occupancy<16, 32, 1, 2, 4>(),    k1_occupancy<16, 16, 1, 1, 4>(),
                 k1_occupancy<16, 32, 2, 2, 8>(),    k1_occupancy<16, 16, 2, 1, 8>(),    k1_occupancy<16, 32, 2, 2, 16>(),
                 k1_occupancy<16, 16, 2, 1, 16>()};
    for (int i = 0; i < 10; ++i)
      if (o[i] > 0) kK1Configs[i].ctas_per_sm = o[i];
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_dgemm_generic<64, 64, 2, 2>, 128, 0) == cudaSuccess && n > 0)
      kK2Configs[0].ctas_per_sm = n;
    cudaGetLastError();
  });
}

}  // namespace

int dgemm_tile_configs(int kernel, const TileConfig** out) {
  refine_occupancy();
  if (kernel == MOA_KERNEL_DGEMM_TMA) {
    *out = kK1Configs;
    return (int)(sizeof(kK1Configs) / sizeof(kK1Configs[0]));
  }
  if (kernel == MOA_KERNEL_DGEMM_GENERIC) {
    *out = kK2Configs;
    return 1;
  }
  *out = nullptr;
  return 0;
}

int launch_dgemm_tma(const moa_plan_t& plan, const GemmArgs& g, cudaStream_t stream) {
  if (plan.bm == 128 && plan.bn == 128 && plan.stages == 6) return launch_k1<128, 128, 4, 2, 6>(plan, g, stream);
  if (plan.bm == 128 && plan.bn == 64 && plan.stages == 4) return launch_k1<128, 64, 4, 2, 4>(plan, g, stream);
  if (plan.bm == 64 && plan.bn == 64 && plan.stages == 4) return launch_k1<64, 64, 2, 4, 4>(plan, g, stream);
  if (plan.bm == 64 && plan.bn == 32 && plan.stages == 4) return launch_k1<64, 32, 2, 2, 4>(plan, g, stream);
  if (plan.bm == 16 && plan.bn == 32 && plan.stages == 4) return launch_k1<16, 32, 1, 2, 4>(plan, g, stream);
  if (plan.bm == 16 && plan.bn == 16 && plan.stages == 4) return launch_k1<16, 16, 1, 1, 4>(plan, g, stream);
  if (plan.bm == 16 && plan.bn == 32 && plan.stages == 8) return launch_k1<16, 32, 2, 2, 8>(plan, g, stream);
  if (plan.bm == 16 && plan.bn == 16 && plan.stages == 8) return launch_k1<16, 16, 2, 1, 8>(plan, g, stream);
  if (plan.bm == 16 && plan.bn == 32 && plan.stages == 16) return launch_k1<16, 32, 2, 2, 16>(plan, g, stream);
  if (plan.bm == 16 && plan.bn == 16 && plan.stages == 16) return launch_k1<16, 16, 2, 1, 16>(plan, g, stream);
  set_error("no compiled K1 instance for this plan");
  return MOA_ERR_INVALID_SHAPE;
}

int launch_dgemm_generic(const moa_plan_t& plan, const GemmArgs& g, cudaStream_t stream) {
  PeerDst peers{};
  if (g.peers) peers = *g.peers;
  k_dgemm_generic<64, 64, 2, 2><<<plan.grid, 128, 0, stream>>>(
      (const double*)g.A, (const double*)g.B, (double*)g.C, g.m, g.n, g.p, g.lda, g.ldb, g.ldc, g.accumulate,
      plan.tiles_m, plan.tiles_n, plan.raster_group, peers);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("k_dgemm_generic launch: ") + cudaGetErrorString(e));
    return MOA_ERR_CUDA;
  }
  return MOA_OK;
}

}  // namespace moa

#ifdef MOA_K1_PHASES
extern "C" int moa_k1_phases_read(unsigned long long* host, int n) {
  if (n > 1024 * 8) n = 1024 * 8;
  return (int)cudaMemcpyFromSymbol(host, moa::g_ph, sizeof(unsigned long long) * (size_t)n);
}
extern "C" int moa_k1_phases_clear() {
  static unsigned long long z[1024 * 8] = {};
  return (int)cudaMemcpyToSymbol(moa::g_ph, z, sizeof(z));
}
#endif
