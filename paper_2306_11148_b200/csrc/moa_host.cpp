// moa_host.cpp — the C-ABI host layer of libmoa.so (declared in include/moa.h):
// argument validation, the static block plan, psi / row-lifting helpers,
// kernel dispatch, the NCCL-backed row-lifted path and error reporting.
//
// Paper references: PAPER.md lines P:n (see include/moa.h for the per-entry
// citations). Readings R1..R16: DESIGN.md §Readings.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges cost nothing unless a profiler attaches

#include <climits>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "moa.h"
#include "moa_internal.h"

// Library-owned communicator: the NCCL communicator plus a side stream and events
// used to pipeline the broadcast of B's k-panels against the lifted compute.
constexpr int kMaxPanels = 16;
constexpr int kPipeCTAs = 4;
struct moa_comm_s {
  ncclComm_t nccl = nullptr;
  int nranks = 0;
  int rank = 0;
  int device = 0;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_start = nullptr;
  cudaEvent_t ev_panel[kMaxPanels] = {};
  // 2-D lifting: row / column sub-communicators for the last grid shape used
  int grid_rows = 0, grid_cols = 0;
  ncclComm_t row_comm = nullptr, col_comm = nullptr;
  // Pipelined B panels (after the first) travel on a split of the communicator whose
  // kernels are limited to kPipeCTAs CTAs; the GEMMs they overlap leave that many
  // SMs free (see gemm_reserving).
  ncclComm_t pipe = nullptr;
  // Symmetric windows (moa_comm_alloc_window) for the fused GEMM -> all-gather:
  // ncclMemAlloc'd memory registered on this communicator, with every rank's copy
  // resolved to an address in this process.
  struct Window {
    void* ptr = nullptr;
    size_t bytes = 0;
    ncclWindow_t win = nullptr;
    std::vector<void*> peer;  // peer[r] = rank r's copy
  };
  std::vector<Window> windows;
  int* barrier_buf = nullptr;  // two ints: [0] the barrier all-reduce's operand, [1] moa_comm_agree's
};

namespace moa {

namespace {
thread_local std::string g_last_error;

// NVTX range around the host-side issue of one step of a lifted call (exchange,
// compute, gather), so a profiler timeline (nsys / ncu --nvtx) attributes the
// stream work each step enqueues.
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

std::mutex g_dev_mu;
std::map<int, DeviceShape> g_devs;

int elem_size(int dtype) {
  switch (dtype) {
    case MOA_F64: return 8;
    case MOA_F32: return 4;
    case MOA_F32_3XTF32: return 4;
    default: return 0;
  }
}

bool mul_ok(int64_t a, int64_t b, int64_t* out) {
  return !__builtin_mul_overflow(a, b, out);
}

int cuda_fail(cudaError_t e, const char* what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return MOA_ERR_CUDA;
}

int get_device_shape(int device, DeviceShape* out) {
  if (device < 0) {
    cudaError_t e = cudaGetDevice(&device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  }
  {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    auto it = g_devs.find(device);
    if (it != g_devs.end()) {
      *out = it->second;
      return MOA_OK;
    }
  }
  DeviceShape d;
  d.device = device;
  cudaError_t e;
  int v = 0;
  RelaxedCapture relaxed_capture;  // first call may be inside graph capture
  if ((e = cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, device)) != cudaSuccess)
    return cuda_fail(e, "cudaDeviceGetAttribute(SM count)");
  cudaDeviceGetAttribute(&d.cc_major, cudaDevAttrComputeCapabilityMajor, device);
  cudaDeviceGetAttribute(&d.cc_minor, cudaDevAttrComputeCapabilityMinor, device);
  cudaDeviceGetAttribute(&d.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  cudaDeviceGetAttribute(&d.smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
  cudaDeviceGetAttribute(&d.regs_per_sm, cudaDevAttrMaxRegistersPerMultiprocessor, device);
  cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, device);
  d.l2_bytes = v;
  std::lock_guard<std::mutex> lk(g_dev_mu);
  g_devs[device] = d;
  *out = d;
  return MOA_OK;
}

// Byte span [lo, hi) of a rows x cols matrix with row stride ld (elements).
void span(const void* base, int64_t rows, int64_t cols, int64_t ld, int es, uintptr_t* lo, uintptr_t* hi) {
  *lo = (uintptr_t)base;
  *hi = *lo + (uintptr_t)(rows > 0 && cols > 0 ? ((rows - 1) * ld + cols) * es : 0);
}

// Per-device resources of the pipelined host path (created once, owned by the
// library): two copy streams and the events that chain panels across streams.
constexpr int kMaxHostPanels = 32;
struct HostPipe {
  std::mutex mu;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t ev0 = nullptr;
  cudaEvent_t evA[kMaxHostPanels] = {};
  cudaEvent_t evB[kMaxHostPanels] = {};
  cudaEvent_t evC[kMaxHostPanels] = {};
};
std::mutex g_pipe_mu;
std::map<int, HostPipe*> g_pipes;

int host_pipe(int device, HostPipe** out) {
  std::lock_guard<std::mutex> lk(g_pipe_mu);
  auto it = g_pipes.find(device);
  if (it != g_pipes.end()) {
    *out = it->second;
    return MOA_OK;
  }
  auto* hp = new HostPipe;
  cudaError_t e = cudaStreamCreateWithFlags(&hp->h2d, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&hp->d2h, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&hp->ev0, cudaEventDisableTiming);
  for (int i = 0; i < kMaxHostPanels && e == cudaSuccess; ++i) {
    e = cudaEventCreateWithFlags(&hp->evA[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&hp->evB[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&hp->evC[i], cudaEventDisableTiming);
  }
  if (e != cudaSuccess) return cuda_fail(e, "host pipeline streams/events");  // leaked on failure: process is broken
  g_pipes[device] = hp;
  *out = hp;
  return MOA_OK;
}

// Validation shared by every GEMM entry point (before any CUDA call). Row-major
// operands with leading dimensions lda >= n, ldb >= p, ldc >= p (elements).
int validate_g(const GemmArgs& g, int dtype) {
  const int64_t m = g.m, n = g.n, p = g.p;
  if (m < 0 || n < 0 || p < 0) {
    set_error("negative extent");
    return MOA_ERR_INVALID_SHAPE;
  }
  const int es = elem_size(dtype);
  if (es == 0) {
    set_error("unknown dtype");
    return MOA_ERR_INVALID_DTYPE;
  }
  if (g.lda < (n > 1 ? n : 1) || g.ldb < (p > 1 ? p : 1) || g.ldc < (p > 1 ? p : 1)) {
    set_error("leading dimension smaller than the row length");
    return MOA_ERR_INVALID_SHAPE;
  }
  int64_t t;
  if (!mul_ok(m, g.lda, &t) || !mul_ok(t, es, &t) || !mul_ok(n, g.ldb, &t) || !mul_ok(t, es, &t) ||
      !mul_ok(m, g.ldc, &t) || !mul_ok(t, es, &t) || !mul_ok(m, p, &t) || !mul_ok(m, n, &t) || !mul_ok(n, p, &t)) {
    set_error("extent product overflows int64");
    return MOA_ERR_INVALID_SHAPE;
  }
  if ((m * n > 0 && !g.A) || (n * p > 0 && !g.B) || (m * p > 0 && !g.C)) {
    set_error("NULL pointer for a non-empty operand");
    return MOA_ERR_NULL_POINTER;
  }
  auto mis = [es](const void* q) { return q && (reinterpret_cast<uintptr_t>(q) % (uintptr_t)es) != 0; };
  if (mis(g.A) || mis(g.B) || mis(g.C)) {
    set_error("pointer not aligned to the element size");
    return MOA_ERR_MISALIGNED;
  }
  uintptr_t a0, a1, b0, b1, c0, c1;
  span(g.A, m, n, g.lda, es, &a0, &a1);
  span(g.B, n, p, g.ldb, es, &b0, &b1);
  span(g.C, m, p, g.ldc, es, &c0, &c1);
  auto ov = [](uintptr_t x0, uintptr_t x1, uintptr_t y0, uintptr_t y1) { return x0 < x1 && y0 < y1 && x0 < y1 && y0 < x1; };
  if (ov(c0, c1, a0, a1) || ov(c0, c1, b0, b1)) {
    set_error("C overlaps A or B (':=' needs a distinct output)");
    return MOA_ERR_ALIASING;
  }
  return MOA_OK;
}

GemmArgs dense(int64_t m, int64_t n, int64_t p, const void* A, const void* B, void* C) {
  return GemmArgs{m, n, p, A, B, C, n > 0 ? n : 1, p > 0 ? p : 1, p > 0 ? p : 1, 0};
}

int validate(int64_t m, int64_t n, int64_t p, const void* A, const void* B, const void* C, int dtype) {
  return validate_g(dense(m, n, p, A, B, const_cast<void*>(C)), dtype);
}

// Is this call describable by the TMA kernels? (row strides multiple of 16 B,
// bases 16-B aligned, coordinates fit the tensor map's int32.)
// The extra C destinations of the fused-gather epilogue are written with the same
// 16-byte vector stores as C (K1 double2, K3 float4), so they must be 16-B aligned
// too; an 8-B-aligned fp64 destination routes the call to the generic kernels, which
// store one element at a time (same bits).
bool tma_eligible(const GemmArgs& g, int es) {
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15u) == 0; };
  const int per16 = 16 / es;
  bool ok = (g.lda % per16 == 0) && (g.ldb % per16 == 0) && (g.ldc % per16 == 0) && (g.p % per16 == 0) && al16(g.A) &&
            al16(g.B) && al16(g.C) && g.m < INT32_MAX && g.n < INT32_MAX && g.p < INT32_MAX;
  for (int d = 0; ok && g.peers && d < g.peers->nd; ++d) ok = al16(g.peers->dst[d]);
  return ok;
}

// Persistent grid. K1 (stream-K runs, moa_ptx.cuh sk_run) needs grid <= tiles and all
// CTAs resident: a whole number of CTAs per SM up to the occupancy, so every SM
// carries the same share of the balanced work. Other kernels: min(tiles, slots).
int32_t grid_for(int kernel, int64_t tiles, int sms, int ctas_per_sm, int64_t tile_area) {
  const int64_t slots = (int64_t)sms * ctas_per_sm;
  // latency tiles (<= 32x32 outputs, 1-2 warps): one resident CTA per tile
  if (kernel != MOA_KERNEL_DGEMM_TMA || tiles < sms || tiles >= slots || tile_area <= 32 * 32)
    return (int32_t)(tiles < slots ? tiles : slots);
  return (int32_t)((int64_t)sms * (tiles / sms));
}

// The static chooser: among the compiled tile configs of
// `kernel`, pick the one with the best predicted SM-level efficiency
//   eff = (m*p) / (waves * sms * bm*bn) * eta,   waves = ceil(tiles / sms)
// (for K1 stream-K plans: (m*p) / (tiles * bm*bn) * eta * 0.99, no wave loss;
// for the K1 latency tiles, tiny problems only: the longest chain per SM sub-partition),
// i.e. the lifted block (bm x bn) "as close as possible" to filling every SM's
// fp64 pipe for a whole number of waves. No measurement, no autotuning.
int choose(int kernel, int64_t m, int64_t n, int64_t p, const DeviceShape& ds, moa_plan_t* out) {
  const TileConfig* cfgs = nullptr;
  int nc = 0;
  if (kernel == MOA_KERNEL_DGEMM_TMA || kernel == MOA_KERNEL_DGEMM_GENERIC)
    nc = dgemm_tile_configs(kernel, &cfgs);
  else
    nc = sgemm_tile_configs(kernel, &cfgs);
  if (nc <= 0) {
    set_error("no tile configuration compiled for this kernel");
    return MOA_ERR_INVALID_DTYPE;
  }
  double best = -1.0;
  int bi = 0;
  bool ruled = false;
  // Tiny problems (fewer 64x32 tiles than SMs): the latency tiles, by a rule read off
  // the measured sweep (profiles/r02/small_n_latency.json, graph-timed, every pick the
  // fastest compiled tile at N = 64...512): 16x16 CTAs of two 8x16 warps while there
  // are at most 2.75 tiles per SM, then 16x32 CTAs of four 8x16 warps up to 2 per SM,
  // then 16x32 CTAs of two 16x16 warps. (Spreading a CTA's outputs over more warps
  // puts more SM sub-partitions on the short k-chains: 256^3 4.45 vs 5.18 us.)
  if (kernel == MOA_KERNEL_DGEMM_TMA && (double)m * (double)p < (double)ds.sms * 64.0 * 32.0) {
    const int64_t t16 = ((m + 15) / 16) * ((p + 15) / 16), t32 = ((m + 15) / 16) * ((p + 31) / 32);
    int want_bn = 4 * t16 <= 11LL * ds.sms ? 16 : 32;
    int want_st = (want_bn == 16 || t32 <= 2LL * ds.sms) ? 8 : 4;
    // All of k in one 16-stage ring (n <= 256) and one tile per resident CTA: the
    // one-shot twins of the 8x16-warp tiles (K1Traits::kOneShotCfg: every load issued up
    // front, no stage release). Their time is the operand stream into the busiest SM
    // (each CTA loads its (bm + bn) x n operands once, all at the start) followed by the
    // k-chain, so between the two the one with fewer bytes into the busiest SM wins:
    // ceil(tiles / SMs) x (bm + bn). Measured (profiles/r02/small_n_oneshot.json,
    // graph-timed): N = 64 / 128 / 192 take 16x16 (1.84 / 2.52 / 2.86 us), N = 256 takes
    // 16x32 (3.56 us; 16x16 4.25; the ring-fed tiles before: 4.42).
    if (want_st == 8 && (n + 15) / 16 <= 16) {
      auto slots = [&](int bn) -> int64_t {
        for (int i = 0; i < nc; ++i)
          if (cfgs[i].bm == 16 && cfgs[i].bn == bn && cfgs[i].stages == 16 && cfgs[i].smem_bytes <= ds.smem_optin)
            return (int64_t)ds.sms * cfgs[i].ctas_per_sm;
        return 0;
      };
      const bool ok16 = t16 <= slots(16), ok32 = t32 <= slots(32);
      const int64_t b16 = (t16 + ds.sms - 1) / ds.sms * 32, b32 = (t32 + ds.sms - 1) / ds.sms * 48;
      if (ok32 && (!ok16 || b32 < b16)) {
        want_bn = 32;
        want_st = 16;
      } else if (ok16) {
        want_bn = 16;
        want_st = 16;
      }
    }
    for (int i = 0; i < nc; ++i)
      if (cfgs[i].bm == 16 && cfgs[i].bn == want_bn && cfgs[i].stages == want_st && cfgs[i].smem_bytes <= ds.smem_optin) {
        ruled = true;
        bi = i;
      }
  }
  for (int i = 0; i < nc && !ruled; ++i) {
    const TileConfig& c = cfgs[i];
    if (c.smem_bytes > ds.smem_optin) continue;
    double eta = c.eta;
    if (eta <= 0.0) {
      // A 32-column tile (K1 64x32) is offered only where every 64-column tile would
      // waste columns (p mod 64 in (0, 32]): thin-p shapes, e.g. m = 2^20, n = p = 32,
      // where 128x64 does twice the DMMA work (177 vs 90.6 us; 64x32 reaches 5.9 TB/s,
      // 91% of HBM: profiles/r01_skinny_hbm.jsonl). Its eta there is its large-N
      // efficiency relative to 128x128 (N=2048: 0.95), so near-square shapes keep the
      // wide tiles.
      const int64_t c32 = (p + 31) / 32 * 32, c64 = (p + 63) / 64 * 64;
      if (!(c.kernel == MOA_KERNEL_DGEMM_TMA && c.bn == 32 && c.bm * c.bn > 32 * 32 && c32 < c64)) continue;
      eta = 0.95;
    }
    const int64_t tm = (m + c.bm - 1) / c.bm, tn = (p + c.bn - 1) / c.bn, tiles = tm * tn;
    const int64_t waves = (tiles + ds.sms - 1) / ds.sms;
    double eff = (double)m * (double)p / ((double)waves * ds.sms * (double)c.bm * c.bn) * eta;
    if (c.kernel == MOA_KERNEL_DGEMM_TMA && (int64_t)c.bm * c.bn <= 32 * 32) {
      // Latency tiles (16x16 outputs per warp, one resident CTA per tile): only for
      // tiny problems (fewer 64x32 tiles than SMs), where the time is the longest
      // DMMA chain per SM sub-partition: ceil(warps / (4 SMs)) warps of 16x16 each.
      // For thin p (<= 32 columns: one 16x32 tile spans the row) the 16x32 tiles stay
      // candidates up to 2x that size at 0.85 of the model: 16384 x {64, 512, 4096} x 32
      // run 5.7 / 23.3 / 165 us with them vs 9.7 / 28.6 / 180 us with 64x32 stream-K
      // (profiles/r01_thin_p.jsonl; at 30000 x 128 x 32 64x32 is ahead again).
      // (Extending the gate to every tile picked 16x16 tiles far too often.)
      const double mp = (double)m * (double)p, one = (double)ds.sms * 64.0 * 32.0;
      const bool thin = c.bn == 32 && p <= 32 && mp < 2.0 * one;
      if (mp >= one && !thin) continue;
      const int64_t warps = tiles * ((int64_t)c.bm * c.bn / 256), smsp = 4LL * ds.sms;
      eff = mp / ((double)smsp * (double)((warps + smsp - 1) / smsp) * 256.0) * eta * (mp < one ? 1.0 : 0.85);
    }
    // K1 stream-K plans balance the last wave (every SM gets the same k-slabs); the
    // cut tiles cost a partial store + reload and an extra pipeline fill: -1%, and
    // each run of R k-slabs pays about 4 slabs of hand-off, which only matters for
    // shallow k (n = 64: R ~ 7 slabs; 256x64x8192 took 19.3 us with 128x64 stream-K
    // vs 14.2 us with one wave of 128x128 tiles).
    const int32_t grid = grid_for(c.kernel, tiles, ds.sms, c.ctas_per_sm, (int64_t)c.bm * c.bn);
    if (c.kernel == MOA_KERNEL_DGEMM_TMA && use_stream_k(tiles, grid)) {
      const double run = (double)tiles * (double)((n + c.bk - 1) / c.bk) / (double)grid;
      eff = (double)m * (double)p / ((double)tiles * c.bm * c.bn) * eta * 0.99 * run / (run + 4.0);
      // a 4-warp 64x32 CTA alone on an SM (stream-K grid = SMs) leaves one warp per
      // sub-partition: N = 1024 ran 98 vs 72 us with the same tiles two-plus per SM
      if (grid <= ds.sms && (int64_t)c.bm * c.bn <= 64 * 32) eff *= 0.75;
      // likewise a config built for two CTAs per SM (64x64: 8 warps of 32x16) that the
      // stream-K grid leaves alone on its SM. Measured against the model: 64x64 alone
      // at 1024^3 ran 29.0 TF/s (model 0.932, i.e. x0.84 of it) and 1024x4096x1024 31.6
      // (model 0.957, x0.89); one wave of 128x64 tiles (model 0.848) ran 29.7 and 30.5.
      // x0.89 ranks both pairs right (profiles/r02/ab_midn_grid.jsonl, ab_tile_80x96.jsonl)
      else if (grid <= ds.sms && c.ctas_per_sm >= 2) eff *= 0.89;
    }
    if (eff > best + 1e-12) {
      best = eff;
      bi = i;
    }
  }
  const TileConfig& c = cfgs[bi];
  memset(out, 0, sizeof(*out));
  out->kernel = c.kernel;
  out->bm = c.bm;
  out->bn = c.bn;
  out->bk = c.bk;
  out->stages = c.stages;
  out->threads = c.threads;
  out->ctas_per_sm = c.ctas_per_sm;
  out->tiles_m = (m + c.bm - 1) / c.bm;
  out->tiles_n = (p + c.bn - 1) / c.bn;
  out->tiles = out->tiles_m * out->tiles_n;
  out->grid = grid_for(c.kernel, out->tiles, ds.sms, c.ctas_per_sm, (int64_t)c.bm * c.bn);
  out->raster_group = (int32_t)(out->tiles_m < 8 ? out->tiles_m : 8);
  if (out->raster_group < 1) out->raster_group = 1;
  out->smem_bytes = c.smem_bytes;
  out->sms = ds.sms;
  return MOA_OK;
}

int tile_configs_for(int kernel, const TileConfig** cfgs) {
  if (kernel == MOA_KERNEL_DGEMM_TMA || kernel == MOA_KERNEL_DGEMM_GENERIC) return dgemm_tile_configs(kernel, cfgs);
  return sgemm_tile_configs(kernel, cfgs);
}

int plan_impl(int64_t m, int64_t n, int64_t p, int dtype, const DeviceShape& ds, bool tma_ok, moa_plan_t* out) {
  memset(out, 0, sizeof(*out));
  out->sms = ds.sms;
  if (m == 0 || p == 0) {
    out->kernel = MOA_KERNEL_NONE;
    return MOA_OK;
  }
  if (n == 0) {
    out->kernel = MOA_KERNEL_ZERO_FILL;
    return MOA_OK;
  }
  int kernel;
  if (dtype == MOA_F64)
    kernel = tma_ok ? MOA_KERNEL_DGEMM_TMA : MOA_KERNEL_DGEMM_GENERIC;
  else if (dtype == MOA_F32)
    kernel = tma_ok ? MOA_KERNEL_SGEMM_FFMA : MOA_KERNEL_SGEMM_GENERIC;
  else if (dtype == MOA_F32_3XTF32)  // shapes TMA cannot describe fall back to the (more exact) fp32 kernel
    kernel = tma_ok ? MOA_KERNEL_SGEMM_3XTF32 : MOA_KERNEL_SGEMM_GENERIC;
  else {
    set_error("unknown dtype");
    return MOA_ERR_INVALID_DTYPE;
  }
  return choose(kernel, m, n, p, ds, out);
}

int check_device(const DeviceShape& ds) {
  if (ds.cc_major != 10 || ds.cc_minor != 0) {
    set_error("libmoa.so is compiled for sm_100a only (B200); device is sm_" + std::to_string(ds.cc_major) +
              std::to_string(ds.cc_minor));
    return MOA_ERR_UNSUPPORTED_DEVICE;
  }
  return MOA_OK;
}

int run_plan(const moa_plan_t& plan, const GemmArgs& g, int dtype, cudaStream_t s) {
  switch (plan.kernel) {
    case MOA_KERNEL_NONE: return MOA_OK;
    case MOA_KERNEL_ZERO_FILL: {  // empty sum: C := 0, or C := C + 0 (nothing) when accumulating
      if (g.accumulate) return MOA_OK;
      const size_t es = (size_t)elem_size(dtype);
      cudaError_t e = cudaMemset2DAsync(g.C, (size_t)g.ldc * es, 0, (size_t)g.p * es, (size_t)g.m, s);
      for (int d = 0; g.peers && d < g.peers->nd && e == cudaSuccess; ++d)
        e = cudaMemset2DAsync(g.peers->dst[d], (size_t)g.ldc * es, 0, (size_t)g.p * es, (size_t)g.m, s);
      return e == cudaSuccess ? MOA_OK : cuda_fail(e, "cudaMemset2DAsync");
    }
    case MOA_KERNEL_DGEMM_TMA: return launch_dgemm_tma(plan, g, s);
    case MOA_KERNEL_DGEMM_GENERIC: return launch_dgemm_generic(plan, g, s);
    case MOA_KERNEL_SGEMM_FFMA: return launch_sgemm_ffma(plan, g, s);
    case MOA_KERNEL_SGEMM_GENERIC: return launch_sgemm_generic(plan, g, s);
    case MOA_KERNEL_SGEMM_3XTF32: return launch_sgemm_3xtf32(plan, g, s);
    default: set_error("bad plan kernel id"); return MOA_ERR_INVALID_SHAPE;
  }
}

// The common GEMM path: validate, plan (optionally honouring an explicit tile
// choice), launch.
int gemm_impl(const GemmArgs& g, int dtype, const moa_plan_t* plan, cudaStream_t stream) {
  Nvtx range("moa gemm");
  int rc = validate_g(g, dtype);
  if (rc) return rc;
  DeviceShape ds;
  if ((rc = get_device_shape(-1, &ds))) return rc;
  if ((rc = check_device(ds))) return rc;
  moa_plan_t pl;
  if ((rc = plan_impl(g.m, g.n, g.p, dtype, ds, tma_eligible(g, elem_size(dtype)), &pl))) return rc;
  if (plan && pl.kernel == plan->kernel) {
    // honour an explicit tile choice (the block-size experiment) if it is a compiled config
    const TileConfig* cfgs = nullptr;
    int nc = tile_configs_for(pl.kernel, &cfgs);
    bool found = false;
    for (int i = 0; i < nc && !found; ++i)
      if (cfgs[i].bm == plan->bm && cfgs[i].bn == plan->bn && cfgs[i].stages == plan->stages) {
        pl.bm = cfgs[i].bm;
        pl.bn = cfgs[i].bn;
        pl.stages = cfgs[i].stages;
        pl.threads = cfgs[i].threads;
        pl.ctas_per_sm = cfgs[i].ctas_per_sm;
        pl.smem_bytes = cfgs[i].smem_bytes;
        pl.tiles_m = (g.m + pl.bm - 1) / pl.bm;
        pl.tiles_n = (g.p + pl.bn - 1) / pl.bn;
        pl.tiles = pl.tiles_m * pl.tiles_n;
        pl.grid = grid_for(pl.kernel, pl.tiles, ds.sms, pl.ctas_per_sm, (int64_t)pl.bm * pl.bn);
        if (plan->grid > 0 && plan->grid < pl.grid) pl.grid = plan->grid;
        if (plan->raster_group > 0) pl.raster_group = plan->raster_group;
        found = true;
      }
    if (!found) {
      set_error("requested tile configuration is not compiled");
      return MOA_ERR_INVALID_SHAPE;
    }
  } else if (plan && pl.kernel != MOA_KERNEL_NONE && pl.kernel != MOA_KERNEL_ZERO_FILL) {
    set_error("plan kernel does not match the kernel this call requires");
    return MOA_ERR_INVALID_SHAPE;
  }
  return run_plan(pl, g, dtype, stream);
}

ncclDataType_t nccl_type(int dtype) { return dtype == MOA_F64 ? ncclFloat64 : ncclFloat32; }

int nccl_fail(ncclResult_t r, const char* what) {
  set_error(std::string(what) + ": " + ncclGetErrorString(r));
  return MOA_ERR_NCCL;
}

}  // namespace

void set_error(const std::string& s) { g_last_error = s; }

}  // namespace moa

using namespace moa;

extern "C" {

int moa_abi_version(void) { return MOA_ABI_VERSION; }

const char* moa_last_error(void) { return g_last_error.c_str(); }

const char* moa_status_string(int status) {
  switch (status) {
    case MOA_OK: return "MOA_OK";
    case MOA_ERR_INVALID_SHAPE: return "MOA_ERR_INVALID_SHAPE";
    case MOA_ERR_INVALID_DTYPE: return "MOA_ERR_INVALID_DTYPE";
    case MOA_ERR_NULL_POINTER: return "MOA_ERR_NULL_POINTER";
    case MOA_ERR_ALIASING: return "MOA_ERR_ALIASING";
    case MOA_ERR_MISALIGNED: return "MOA_ERR_MISALIGNED";
    case MOA_ERR_INVALID_INDEX: return "MOA_ERR_INVALID_INDEX";
    case MOA_ERR_CUDA: return "MOA_ERR_CUDA";
    case MOA_ERR_NCCL: return "MOA_ERR_NCCL";
    case MOA_ERR_UNSUPPORTED_DEVICE: return "MOA_ERR_UNSUPPORTED_DEVICE";
    case MOA_ERR_NOT_REGISTERED: return "MOA_ERR_NOT_REGISTERED";
    default: return "MOA_ERR_UNKNOWN";
  }
}

int moa_psi(int rank, const int64_t* shape, int q, const int64_t* idx, int64_t* offset, int64_t* count) {
  if (!offset || !count || (rank > 0 && !shape) || (q > 0 && !idx)) {
    set_error("NULL argument");
    return MOA_ERR_NULL_POINTER;
  }
  if (rank < 0 || q < 0 || q > rank) {
    set_error("index longer than the shape");
    return MOA_ERR_INVALID_INDEX;
  }
  for (int d = 0; d < rank; ++d)
    if (shape[d] < 0) {
      set_error("negative extent");
      return MOA_ERR_INVALID_SHAPE;
    }
  for (int d = 0; d < q; ++d)
    if (idx[d] < 0 || idx[d] >= shape[d]) {
      set_error("index out of bounds (0 <=* i <* rho xi)");
      return MOA_ERR_INVALID_INDEX;
    }
  // count = pi(shape[q..rank)); offset = gamma_row(idx ++ zeros) by Horner.
  int64_t cnt = 1;
  for (int d = q; d < rank; ++d)
    if (!mul_ok(cnt, shape[d], &cnt)) {
      set_error("shape product overflows int64");
      return MOA_ERR_INVALID_SHAPE;
    }
  int64_t off = 0;
  for (int d = 0; d < rank; ++d) {
    const int64_t i = d < q ? idx[d] : 0;
    if (!mul_ok(off, shape[d], &off) || __builtin_add_overflow(off, i, &off)) {
      set_error("offset overflows int64");
      return MOA_ERR_INVALID_SHAPE;
    }
  }
  if (cnt == 0) off = 0;
  *offset = off;
  *count = cnt;
  return MOA_OK;
}

int moa_lift_rows(int64_t m, int nparts, int part, int64_t* row0, int64_t* rows) {
  if (!row0 || !rows) {
    set_error("NULL argument");
    return MOA_ERR_NULL_POINTER;
  }
  if (m < 0 || nparts <= 0 || part < 0 || part >= nparts) {
    set_error("bad row-lifting arguments");
    return MOA_ERR_INVALID_SHAPE;
  }
  const int64_t q = m / nparts, r = m % nparts;
  *rows = q + (part < r ? 1 : 0);
  *row0 = (int64_t)part * q + (part < r ? part : r);
  return MOA_OK;
}

int moa_select_block_paper(int64_t l1_budget_bytes, int elem_bytes, int64_t* b) {
  if (!b) {
    set_error("NULL argument");
    return MOA_ERR_NULL_POINTER;
  }
  if (elem_bytes <= 0 || l1_budget_bytes < 3LL * elem_bytes) {
    set_error("budget too small for three 1x1 blocks");
    return MOA_ERR_INVALID_SHAPE;
  }
  int64_t s = 1;
  while (s < (1LL << 30) && 3 * (2 * s) * (2 * s) * (int64_t)elem_bytes <= l1_budget_bytes) s *= 2;
  *b = s;
  return MOA_OK;
}

int moa_plan(int64_t m, int64_t n, int64_t p, int dtype, int device, moa_plan_t* out) {
  if (!out) {
    set_error("NULL plan");
    return MOA_ERR_NULL_POINTER;
  }
  if (m < 0 || n < 0 || p < 0) {
    set_error("negative extent");
    return MOA_ERR_INVALID_SHAPE;
  }
  if (elem_size(dtype) == 0) {
    set_error("unknown dtype");
    return MOA_ERR_INVALID_DTYPE;
  }
  DeviceShape ds;
  int rc = get_device_shape(device, &ds);
  if (rc) return rc;
  const int per16 = 16 / elem_size(dtype);
  const bool tma_ok = n % per16 == 0 && p % per16 == 0 && m < INT32_MAX && n < INT32_MAX && p < INT32_MAX;
  return plan_impl(m, n, p, dtype, ds, tma_ok, out);
}

int moa_gemm_with_plan(int64_t m, int64_t n, int64_t p, const void* A, const void* B, void* C, int dtype,
                       const moa_plan_t* plan, void* stream) {
  return gemm_impl(dense(m, n, p, A, B, C), dtype, plan, (cudaStream_t)stream);
}

int moa_gemm(int64_t m, int64_t n, int64_t p, const void* A, const void* B, void* C, int dtype, void* stream) {
  return gemm_impl(dense(m, n, p, A, B, C), dtype, nullptr, (cudaStream_t)stream);
}

int moa_gemm_acc(int64_t m, int64_t n, int64_t p, const void* A, int64_t lda, const void* B, int64_t ldb, void* C,
                 int64_t ldc, int accumulate, int dtype, void* stream) {
  return gemm_impl(GemmArgs{m, n, p, A, B, C, lda, ldb, ldc, accumulate ? 1 : 0}, dtype, nullptr,
                   (cudaStream_t)stream);
}

static int gemm_reserving(const GemmArgs& g, int dtype, cudaStream_t s, int reserve);
static int pipe_comm(moa_comm_t comm, ncclComm_t* out);
static int issue_nccl(moa_comm_t comm, const moa_coll_t& o, void* data, const void* send, int dtype, cudaStream_t s);
namespace {
int host_panel_bounds(int64_t n, int dtype, bool comm, bool first_chain, int64_t* kb);
std::vector<moa_coll_t> plan_vec(int variant, int64_t m, int64_t n, int64_t p, int dtype, int G, int rank, int gr,
                                 int gc, int npanels, int flags);
}  // namespace

// The end-to-end pipeline of moa_gemm_host; with a communicator, the rank's rows
// of the row-lifted product (moa_gemm_lifted_host): B's k-panels cross the host
// link on rank 0 only and reach every rank by an NCCL broadcast per panel on the
// communicator's side stream, so the exchange of B is pipelined with the host
// copies and with the compute of row panel 0.
static int gemm_host_impl(int64_t m, int64_t n, int64_t p, const void* A_host, const void* B_host, void* C_host,
                          void* A_dev, void* B_dev, void* C_dev, int dtype, void* stream, moa_comm_t comm) {
  int rc = validate(m, n, p, A_dev, B_dev, C_dev, dtype);
  if (rc) return rc;
  const int64_t es = elem_size(dtype);
  const bool b_root = !comm || comm->rank == 0;  // this rank reads B from the host
  if ((m * n > 0 && !A_host) || (n * p > 0 && b_root && !B_host) || (m * p > 0 && !C_host)) {
    set_error("NULL host pointer for a non-empty operand");
    return MOA_ERR_NULL_POINTER;
  }
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  DeviceShape ds;
  if ((rc = get_device_shape(-1, &ds))) return rc;
  HostPipe* hp = nullptr;
  if ((rc = host_pipe(ds.device, &hp))) return rc;
  std::lock_guard<std::mutex> lk(hp->mu);
  // Row lifting inside one GPU (rows of C depend only on the same rows of
  // A, Fig. 1): A streams in row panels on a copy stream while earlier panels
  // compute on `stream`, and each finished C panel streams back on a second copy
  // stream. Panels are whole tile rows sized to ~7 waves of tiles each (static), so
  // the panel GEMMs lose no wave efficiency; results are bitwise the one-call ones.
  moa_plan_t pl;
  if ((rc = moa_plan(m, n, p, dtype, ds.device, &pl))) return rc;
  // Static schedule from the hardware shape (no measurement):
  //  * row panel 0 is computed as a chain over KB = 8 k-panels of B (accumulate,
  //    bitwise the one-call result for f64/f32) that start as soon as A0 and the
  //    first B k-panel have landed; it is sized so its compute lasts about as long
  //    as B takes to cross the host link: rows0 ~ peak * esize / (2 * link), independent
  //    of n and p (fp64: 37 TF/s * 8 B / (2 * 52 GB/s) ~ 2.9K rows);
  //  * the middle rows go in panels of ~7 waves of tiles (no wave loss), each
  //    starting when its A rows have landed, after all of B;
  //  * a short last panel (4 tile rows) trims the final D2H tail.
  //  * deep k (n >= 24576, one device, B in 16 k-panels): A0 crosses in column blocks,
  //    each just before the B k-panel it meets, so compute starts after one column
  //    block and one B panel instead of all of A0 (32768^3: e2e 1963.5 -> 1948.8 ms,
  //    profiles/r02/e2e_a0cols.jsonl); A0 gets one more tile row because its blocks
  //    now share the link with B. (At 8192^3 the strided copies lost: round 1.)
  const bool chain = n >= 512 && dtype != MOA_F32_3XTF32;
  const bool a0cols_k = !comm && n >= 24576;
  const int64_t bm = pl.bm > 0 ? pl.bm : 128;
  int64_t bnd[kMaxHostPanels + 1];
  int64_t P = 0;
  bnd[0] = 0;
  if (pl.kernel != MOA_KERNEL_NONE && pl.tiles > 0) {
    int64_t rows0 = 0;
    if (chain) {
      const double peak = dtype == MOA_F64 ? 37.0e12 : 61.0e12, link = 52.0e9;
      rows0 = ((int64_t)(peak * es / (2.0 * link)) + bm - 1) / bm * bm + (a0cols_k ? bm : 0);
      if (rows0 > m / 2) rows0 = 0;  // too small a problem to pipeline this way
    }
    const int64_t per = (ds.sms * 7 / (pl.tiles_n > 0 ? pl.tiles_n : 1) + 1) * bm;  // ~7 waves of tiles
    const int64_t last = (m - rows0 > 2 * per) ? 4 * bm : 0;
    if (rows0 > 0) bnd[++P] = rows0;
    const int64_t rest = m - rows0 - last;
    int64_t k = (rest + per - 1) / per;
    if (k < 1) k = 1;
    if (k > kMaxHostPanels - P - 1) k = kMaxHostPanels - P - 1;
    for (int64_t j = 1; j <= k; ++j) bnd[P + j] = j == k ? rows0 + rest : rows0 + (((rest / bm) * j / k) * bm);
    P += k;
    if (last > 0) bnd[++P] = m;
  } else {
    bnd[++P] = m;
  }
  const bool first_chain = chain && P > 1 && bnd[1] < m;
  // With a communicator the number of B k-panels (= broadcasts) must be the same on
  // every rank, so it depends only on (n, dtype), never on this rank's row count; a
  // rank without a row-panel split still chains its single panel over them (bitwise
  // the same result). The broadcasts are the exchange plan's (MOA_XPLAN_ROWS_HOST).
  int64_t kb[kMaxPanels + 1];
  const int64_t KB = host_panel_bounds(n, dtype, comm != nullptr, first_chain, kb);
  const std::vector<moa_coll_t> xops =
      comm ? plan_vec(MOA_XPLAN_ROWS_HOST, m, n, p, dtype, comm->nranks, comm->rank, 0, 0, 0, 0)
           : std::vector<moa_coll_t>();
  if ((e = cudaEventRecord(hp->ev0, s)) != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
  if ((e = cudaStreamWaitEvent(hp->h2d, hp->ev0, 0)) != cudaSuccess) return cuda_fail(e, "cudaStreamWaitEvent");
  if ((e = cudaStreamWaitEvent(hp->d2h, hp->ev0, 0)) != cudaSuccess) return cuda_fail(e, "cudaStreamWaitEvent");
  auto h2d_rows = [&](const void* hsrc, void* ddst, int64_t r0, int64_t rows, int64_t rowlen) -> cudaError_t {
    if (rows * rowlen <= 0) return cudaSuccess;
    return cudaMemcpyAsync((char*)ddst + r0 * rowlen * es, (const char*)hsrc + r0 * rowlen * es,
                           (size_t)(rows * rowlen * es), cudaMemcpyHostToDevice, hp->h2d);
  };
  // copy order on the H2D engine: A panel 0 (or, deep k, its column blocks interleaved
  // with B's k-panels), B's k-panels, A panels 1..P-1
  const bool a0cols = a0cols_k && first_chain;
  if (!a0cols && (e = h2d_rows(A_host, A_dev, bnd[0], bnd[1] - bnd[0], n)) != cudaSuccess)
    return cuda_fail(e, "H2D A panel");
  if ((e = cudaEventRecord(hp->evA[0], hp->h2d)) != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
  if (comm && (e = cudaStreamWaitEvent(comm->side, hp->ev0, 0)) != cudaSuccess)
    return cuda_fail(e, "cudaStreamWaitEvent");
  // evB[j] (the event compute waits on for B's k-panel j): after its H2D copy, or
  // with a communicator after its broadcast from rank 0 (every processor
  // reads all of B), issued in the same order on every rank
  cudaEvent_t* evB = comm ? comm->ev_panel : hp->evB;
  bool pipe_used = false;  // NCCL panels in flight on the CTA-limited comm: leave SMs free
  for (int64_t j = 0; j < KB; ++j) {
    if (a0cols && kb[j + 1] > kb[j] &&
        (e = cudaMemcpy2DAsync((char*)A_dev + kb[j] * es, (size_t)(n * es), (const char*)A_host + kb[j] * es,
                               (size_t)(n * es), (size_t)((kb[j + 1] - kb[j]) * es), (size_t)bnd[1],
                               cudaMemcpyHostToDevice, hp->h2d)) != cudaSuccess)
      return cuda_fail(e, "H2D A panel 0 column block");
    if (b_root) {
      if ((e = h2d_rows(B_host, B_dev, kb[j], kb[j + 1] - kb[j], p)) != cudaSuccess) return cuda_fail(e, "H2D B panel");
      if ((e = cudaEventRecord(hp->evB[j], hp->h2d)) != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
    }
    if (comm) {
      if (b_root && (e = cudaStreamWaitEvent(comm->side, hp->evB[j], 0)) != cudaSuccess)
        return cuda_fail(e, "cudaStreamWaitEvent");
      for (const auto& o : xops)
        if (o.panel == j) {
          if ((rc = issue_nccl(comm, o, B_dev, nullptr, dtype, comm->side))) return rc;
          pipe_used = pipe_used || o.comm == MOA_COMM_PIPE;
        }
      if ((e = cudaEventRecord(comm->ev_panel[j], comm->side)) != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
    }
  }
  for (int64_t i = 1; i < P; ++i) {
    if ((e = h2d_rows(A_host, A_dev, bnd[i], bnd[i + 1] - bnd[i], n)) != cudaSuccess) return cuda_fail(e, "H2D A panel");
    if ((e = cudaEventRecord(hp->evA[i], hp->h2d)) != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
  }
  for (int64_t i = 0; i < P; ++i) {
    const int64_t r0 = bnd[i], rows = bnd[i + 1] - bnd[i];
    if ((e = cudaStreamWaitEvent(s, hp->evA[i], 0)) != cudaSuccess) return cuda_fail(e, "cudaStreamWaitEvent");
    // (without a communicator, evA[i >= 1] follows all of B on the H2D stream)
    if (comm && i > 0 && (e = cudaStreamWaitEvent(s, evB[KB - 1], 0)) != cudaSuccess)
      return cuda_fail(e, "cudaStreamWaitEvent");
    if (i == 0) {
      for (int64_t j = 0; j < KB; ++j) {
        if ((e = cudaStreamWaitEvent(s, evB[j], 0)) != cudaSuccess) return cuda_fail(e, "cudaStreamWaitEvent");
        if (j > 0 && kb[j + 1] == kb[j]) continue;
        const GemmArgs g{rows, kb[j + 1] - kb[j], p, (const char*)A_dev + (r0 * n + kb[j]) * es, (const char*)B_dev + kb[j] * p * es,
                         (char*)C_dev + r0 * p * es, n > 0 ? n : 1, p > 0 ? p : 1, p > 0 ? p : 1, j > 0 ? 1 : 0};
        // with a communicator, later B panels are still being broadcast: leave SMs free
        if ((rc = gemm_reserving(g, dtype, s, pipe_used && j < KB - 1 ? kPipeCTAs : 0))) return rc;
      }
    } else if ((rc = moa_gemm(rows, n, p, (const char*)A_dev + r0 * n * es, B_dev, (char*)C_dev + r0 * p * es, dtype,
                              stream))) {
      return rc;
    }
    if ((e = cudaEventRecord(hp->evC[i], s)) != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
    if ((e = cudaStreamWaitEvent(hp->d2h, hp->evC[i], 0)) != cudaSuccess) return cuda_fail(e, "cudaStreamWaitEvent");
    if (rows * p > 0 &&
        (e = cudaMemcpyAsync((char*)C_host + r0 * p * es, (const char*)C_dev + r0 * p * es, (size_t)(rows * p * es),
                             cudaMemcpyDeviceToHost, hp->d2h)) != cudaSuccess)
      return cuda_fail(e, "D2H C panel");
  }
  if ((e = cudaStreamSynchronize(hp->d2h)) != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize(d2h)");
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
  return MOA_OK;
}

int moa_gemm_host(int64_t m, int64_t n, int64_t p, const void* A_host, const void* B_host, void* C_host,
                  void* A_dev, void* B_dev, void* C_dev, int dtype, void* stream) {
  return gemm_host_impl(m, n, p, A_host, B_host, C_host, A_dev, B_dev, C_dev, dtype, stream, nullptr);
}

int moa_gemm_lifted_host(int64_t m, int64_t n, int64_t p, const void* A_host, const void* B_host, void* C_host,
                         void* A_dev, void* B_dev, void* C_dev, int dtype, void* stream, moa_comm_t comm) {
  if (!comm) {
    set_error("NULL communicator");
    return MOA_ERR_NULL_POINTER;
  }
  if (m < 0) {
    set_error("negative extent");
    return MOA_ERR_INVALID_SHAPE;
  }
  int64_t row0 = 0, rows = 0;
  int rc = moa_lift_rows(m, comm->nranks, comm->rank, &row0, &rows);
  if (rc) return rc;
  return gemm_host_impl(rows, n, p, A_host, B_host, C_host, A_dev, B_dev, C_dev, dtype, stream, comm);
}

int moa_comm_get_unique_id(unsigned char id[128]) {
  if (!id) {
    set_error("NULL id");
    return MOA_ERR_NULL_POINTER;
  }
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
  ncclUniqueId u;
  ncclResult_t r = ncclGetUniqueId(&u);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(id, &u, 128);
  return MOA_OK;
}

int moa_comm_init(int nranks, int rank, const unsigned char id[128], int device, moa_comm_t* comm) {
  if (!id || !comm) {
    set_error("NULL argument");
    return MOA_ERR_NULL_POINTER;
  }
  if (nranks <= 0 || rank < 0 || rank >= nranks) {
    set_error("bad rank/nranks");
    return MOA_ERR_INVALID_SHAPE;
  }
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  ncclUniqueId u;
  memcpy(&u, id, 128);
  auto* c = new moa_comm_s;
  ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_fail(r, "ncclCommInitRank");
  }
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  if ((e = cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming)) != cudaSuccess) {
    ncclCommDestroy(c->nccl);
    delete c;
    return cuda_fail(e, "side stream / event");
  }
  for (int i = 0; i < kMaxPanels; ++i)
    if ((e = cudaEventCreateWithFlags(&c->ev_panel[i], cudaEventDisableTiming)) != cudaSuccess) {
      ncclCommDestroy(c->nccl);
      delete c;
      return cuda_fail(e, "panel events");
    }
  if ((e = cudaMalloc(&c->barrier_buf, 2 * sizeof(int))) != cudaSuccess ||
      (e = cudaMemset(c->barrier_buf, 0, 2 * sizeof(int))) != cudaSuccess) {
    ncclCommDestroy(c->nccl);
    delete c;
    return cuda_fail(e, "barrier buffer");
  }
  *comm = c;
  return MOA_OK;
}

int moa_comm_destroy(moa_comm_t comm) {
  if (!comm) return MOA_OK;
  if (comm->row_comm) ncclCommDestroy(comm->row_comm);
  if (comm->col_comm) ncclCommDestroy(comm->col_comm);
  if (comm->pipe) ncclCommDestroy(comm->pipe);
  if (comm->side) cudaStreamSynchronize(comm->side);
  for (auto& w : comm->windows) {
    cudaDeviceSynchronize();  // no kernel may still be storing into the window
    ncclCommWindowDeregister(comm->nccl, w.win);
    ncclMemFree(w.ptr);
  }
  comm->windows.clear();
  if (comm->barrier_buf) cudaFree(comm->barrier_buf);
  for (int i = 0; i < kMaxPanels; ++i)
    if (comm->ev_panel[i]) cudaEventDestroy(comm->ev_panel[i]);
  if (comm->ev_start) cudaEventDestroy(comm->ev_start);
  if (comm->side) cudaStreamDestroy(comm->side);
  ncclResult_t r = ncclCommDestroy(comm->nccl);
  delete comm;
  return r == ncclSuccess ? MOA_OK : nccl_fail(r, "ncclCommDestroy");
}

static int validate_elementwise(const void* A, int64_t na, const void* B, int64_t nb, const void* C, int64_t nc,
                                int dtype) {
  const int es = elem_size(dtype);
  if (es == 0 || dtype == MOA_F32_3XTF32) {
    set_error("dtype must be MOA_F64 or MOA_F32");
    return MOA_ERR_INVALID_DTYPE;
  }
  if ((na > 0 && !A) || (nb > 0 && !B) || (nc > 0 && !C)) {
    set_error("NULL pointer for a non-empty operand");
    return MOA_ERR_NULL_POINTER;
  }
  auto mis = [es](const void* q) { return q && (reinterpret_cast<uintptr_t>(q) % (uintptr_t)es) != 0; };
  if (mis(A) || mis(B) || mis(C)) {
    set_error("pointer not aligned to the element size");
    return MOA_ERR_MISALIGNED;
  }
  auto ov = [es](const void* x, int64_t xn, const void* y, int64_t yn) {
    if (xn <= 0 || yn <= 0) return false;
    uintptr_t a0 = (uintptr_t)x, a1 = a0 + (uintptr_t)(xn * es), b0 = (uintptr_t)y, b1 = b0 + (uintptr_t)(yn * es);
    return a0 < b1 && b0 < a1;
  };
  if (ov(C, nc, A, na) || ov(C, nc, B, nb)) {
    set_error("C overlaps an input");
    return MOA_ERR_ALIASING;
  }
  return MOA_OK;
}

int moa_hadamard(int64_t m, int64_t n, const void* A, const void* B, void* C, int dtype, void* stream) {
  int64_t mn;
  if (m < 0 || n < 0 || !mul_ok(m, n, &mn) || !mul_ok(mn, 8, &mn)) {
    set_error("bad extents");
    return MOA_ERR_INVALID_SHAPE;
  }
  mn = m * n;
  int rc = validate_elementwise(A, mn, B, mn, C, mn, dtype);
  if (rc) return rc;
  if (mn == 0) return MOA_OK;
  DeviceShape ds;
  if ((rc = get_device_shape(-1, &ds)) || (rc = check_device(ds))) return rc;
  return launch_hadamard(m, n, A, B, C, dtype, (cudaStream_t)stream);
}

int moa_kron(int64_t m, int64_t n, int64_t p, int64_t q, const void* A, const void* B, void* C, int dtype,
             void* stream) {
  int64_t mn, pq, out, t;
  if (m < 0 || n < 0 || p < 0 || q < 0 || !mul_ok(m, n, &mn) || !mul_ok(p, q, &pq) || !mul_ok(mn, pq, &out) ||
      !mul_ok(out, 8, &t)) {
    set_error("bad extents");
    return MOA_ERR_INVALID_SHAPE;
  }
  int rc = validate_elementwise(A, mn, B, pq, C, out, dtype);
  if (rc) return rc;
  if (out == 0) return MOA_OK;
  DeviceShape ds;
  if ((rc = get_device_shape(-1, &ds)) || (rc = check_device(ds))) return rc;
  return launch_kron(m, n, p, q, A, B, C, dtype, (cudaStream_t)stream);
}

int moa_lift_panels(int64_t n, int64_t p, int dtype, int nranks) {
  // Static choice (no autotuning): pipeline only when B actually travels; aim for
  // <= 512 MiB per panel (a panel's broadcast then hides behind the previous
  // panel's compute), at most 8 panels (each extra panel re-reads/writes C once).
  if (nranks <= 1 || n <= 0 || p <= 0) return 1;
  const int64_t bytes = n * p * elem_size(dtype);
  int64_t k = (bytes + (512ll << 20) - 1) / (512ll << 20);
  if (k > 8) k = 8;
  if (k > n / 64) k = n / 64;
  return k < 1 ? 1 : (int)k;
}

int moa_pull_panels(int64_t n, int64_t* bnd) {
  // A small first panel (little exposed before compute starts), then doubling: the
  // pull of panel j+1 (twice panel j's rows) overlaps panel j's compute, which at the
  // configs[4] shapes runs ~1.4x longer than the pull. Boundaries are
  // multiples of 32 rows of B (TMA alignment of the A column slice).
  if (n < 64) {
    if (bnd) {
      bnd[0] = 0;
      bnd[1] = n > 0 ? n : 0;
    }
    return 1;
  }
  int64_t first = (n / 64) / 32 * 32;
  if (first < 32) first = 32;
  int K = 0;
  int64_t b = 0;
  if (bnd) bnd[0] = 0;
  while (b < n) {
    int64_t next = K == 0 ? first : 2 * b;
    if (next >= n || K == kMaxPanels - 1) next = n;
    b = next;
    ++K;
    if (bnd) bnd[K] = b;
  }
  return K;
}

// A GEMM that leaves `reserve` SMs free for a concurrent collective. A persistent
// K1 grid takes every SM's registers and shared memory (one 384-thread CTA with
// 168..232 registers per thread and ~193 KiB of smem), so an NCCL kernel launched
// next to it could not start until the GEMM had ended: the "overlapped" broadcast
// would in fact serialise. The pipe communicator's kernels use at most kPipeCTAs
// CTAs, and this GEMM's grid is capped at (SMs - reserve) x CTAs-per-SM. Every
// kernel's work assignment is grid-size independent (persistent tile loops, and
// stream-K runs of R >= K slabs since tiles >= grid), so the result is unchanged.
static int gemm_reserving(const GemmArgs& g, int dtype, cudaStream_t s, int reserve) {
  int rc = validate_g(g, dtype);
  if (rc) return rc;
  DeviceShape ds;
  if ((rc = get_device_shape(-1, &ds)) || (rc = check_device(ds))) return rc;
  moa_plan_t pl;
  if ((rc = plan_impl(g.m, g.n, g.p, dtype, ds, tma_eligible(g, elem_size(dtype)), &pl))) return rc;
  if (reserve > 0 && pl.grid > 0 && ds.sms > reserve) {
    const int64_t cap = (int64_t)(ds.sms - reserve) * (pl.ctas_per_sm > 0 ? pl.ctas_per_sm : 1);
    if (pl.grid > cap) pl.grid = (int32_t)cap;
  }
  return run_plan(pl, g, dtype, s);
}

static int pipe_comm(moa_comm_t comm, ncclComm_t* out) {
  if (!comm->pipe) {
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.minCTAs = 1;
    cfg.maxCTAs = kPipeCTAs;
    ncclResult_t r = ncclCommSplit(comm->nccl, 0, comm->rank, &comm->pipe, &cfg);
    if (r != ncclSuccess) {
      comm->pipe = nullptr;
      return nccl_fail(r, "ncclCommSplit(pipe)");
    }
  }
  *out = comm->pipe;
  return MOA_OK;
}

// ----------------------------- the exchange plan (row a7) -----------------------------

namespace {

// k-panel boundaries of the NCCL-pipelined exchange: multiples of 32 rows of B (TMA
// alignment of the A column slice), as equal as possible. Each panel of B is ONE
// contiguous byte range (rows k0..k1 of a row-major B — MoA order). Returns K.
int nccl_panel_bounds(int64_t n, int K, int64_t* bnd) {
  if (K < 1) K = 1;
  if (K > kMaxPanels) K = kMaxPanels;
  if (n < K) K = n > 0 ? (int)n : 1;
  for (int j = 0; j <= K; ++j) bnd[j] = j == K ? n : (n * j / K) / 32 * 32;
  return K;
}

// Panel boundaries of moa_gemm_lifted_host's B chain (static: 8 k-panels when the
// first row panel is chained over B, see gemm_host_impl; 16 for deep k, n >= 24576,
// where B's first panel is the larger part of the pipeline's head: 32768^3 fp64 e2e
// 1972-1977 -> 1966-1968 ms, profiles/r02/e2e_kb.jsonl). A function of (n, dtype)
// only, so every rank of moa_gemm_lifted_host issues the same broadcasts.
int host_panel_bounds(int64_t n, int dtype, bool comm, bool first_chain, int64_t* kb) {
  const bool chain = n >= 512 && dtype != MOA_F32_3XTF32;
  const int KB = (comm ? chain : first_chain) ? (n >= 24576 ? 16 : 8) : 1;
  for (int j = 0; j <= KB; ++j) kb[j] = j == KB ? n : (n * j / KB) / 32 * 32;
  return KB;
}

struct PlanOut {
  moa_coll_t* ops;
  int max_ops;
  int n = 0;
  void add(int op, int comm, int root, int group, int operand, int phase, int panel, int64_t offset, int64_t count) {
    if (n < max_ops) {
      moa_coll_t& o = ops[n];
      o.op = op;
      o.comm = comm;
      o.root = root;
      o.group = group;
      o.operand = operand;
      o.phase = phase;
      o.panel = panel;
      o.reserved = 0;
      o.offset = offset;
      o.count = count;
    }
    ++n;
  }
};

// The plan itself. Arguments are validated by the caller (moa_exchange_plan or an
// executor); every branch depends only on the arguments, never on pointers.
void build_plan(int variant, int64_t m, int64_t n, int64_t p, int dtype, int G, int rank, int grid_rows,
                int grid_cols, int npanels, int flags, PlanOut* out) {
  if (G <= 1) return;  // nothing travels on a 1-rank communicator
  const bool fused = flags & MOA_XF_FUSED_GATHER, gather = (flags & MOA_XF_GATHER) && !fused,
             direct = flags & MOA_XF_DIRECT_B, pull = (flags & MOA_XF_PULL_B) && !direct;
  int64_t bnd[kMaxPanels + 1];
  switch (variant) {
    case MOA_XPLAN_ROWS: {
      if (m * p == 0 && n * p == 0) return;
      // entry barrier: (fused) no rank stores into a peer's C_full before the peer
      // reached this call; (pull, direct) rank 0's B is final before anyone reads it
      if (fused || pull || direct) out->add(MOA_COLL_BARRIER, MOA_COMM_WORLD, -1, 0, MOA_OPERAND_C, 0, -1, 0, 1);
      // (direct: B never moves as a collective — every rank's GEMM reads rank 0's copy
      // through its TMA loads over NVLink)
      if (n * p > 0 && !direct) {
        if (pull) {
          // every processor reads all of B: ranks g > 0 pull it from rank 0
          if (rank != 0) {
            const int K = moa_pull_panels(n, bnd);
            for (int j = 0; j < K; ++j)
              out->add(MOA_COLL_PULL, MOA_COMM_WORLD, 0, 0, MOA_OPERAND_B, 1, j, bnd[j] * p, (bnd[j + 1] - bnd[j]) * p);
          }
        } else {
          const int K = nccl_panel_bounds(n, npanels > 0 ? npanels : moa_lift_panels(n, p, dtype, G), bnd);
          for (int j = 0; j < K; ++j)
            if (bnd[j + 1] > bnd[j] || K == 1)
              out->add(MOA_COLL_BROADCAST, j == 0 ? MOA_COMM_WORLD : MOA_COMM_PIPE, 0, 0, MOA_OPERAND_B, 1, j,
                       bnd[j] * p, (bnd[j + 1] - bnd[j]) * p);
        }
      }
      if (gather && m * p > 0) {
        if (m % G == 0) {
          out->add(MOA_COLL_ALLGATHER, MOA_COMM_WORLD, -1, 0, MOA_OPERAND_C, 2, -1, 0, (m / G) * p);
        } else {
          for (int g = 0; g < G; ++g) {
            int64_t r0, rg;
            moa_lift_rows(m, G, g, &r0, &rg);
            if (rg > 0) out->add(MOA_COLL_BROADCAST, MOA_COMM_WORLD, g, 1, MOA_OPERAND_C, 2, -1, r0 * p, rg * p);
          }
        }
      }
      // exit barrier: (fused) every peer store is complete; (pull, direct) every read
      // of rank 0's B is complete before rank 0 may change it
      if (fused || pull || direct) out->add(MOA_COLL_BARRIER, MOA_COMM_WORLD, -1, 0, MOA_OPERAND_C, 2, -1, 0, 1);
      return;
    }
    case MOA_XPLAN_ROWS_HOST: {
      int64_t kb[kMaxPanels + 1];
      const int KB = host_panel_bounds(n, dtype, true, false, kb);
      for (int j = 0; j < KB; ++j)
        if (kb[j + 1] > kb[j])
          out->add(MOA_COLL_BROADCAST, j == 0 ? MOA_COMM_WORLD : MOA_COMM_PIPE, 0, 0, MOA_OPERAND_B, 1, j, kb[j] * p,
                   (kb[j + 1] - kb[j]) * p);
      return;
    }
    case MOA_XPLAN_COLS: {
      if (fused) out->add(MOA_COLL_BARRIER, MOA_COMM_WORLD, -1, 0, MOA_OPERAND_C, 0, -1, 0, 1);
      // every processor needs all of A (ip_cols.c reads A[(i*shr0)+sigma] with no
      // column-group index): ONE in-place broadcast from rank 0
      if (m * n > 0) out->add(MOA_COLL_BROADCAST, MOA_COMM_WORLD, 0, 0, MOA_OPERAND_A, 0, -1, 0, m * n);
      if (fused) out->add(MOA_COLL_BARRIER, MOA_COMM_WORLD, -1, 0, MOA_OPERAND_C, 2, -1, 0, 1);
      if (gather && m * p > 0)
        for (int g = 0; g < G; ++g) {  // rank g's column block travels through the workspace
          int64_t c0, cg;
          moa_lift_rows(p, G, g, &c0, &cg);
          if (cg > 0) out->add(MOA_COLL_BROADCAST, MOA_COMM_WORLD, g, 0, MOA_OPERAND_C, 2, -1, c0, m * cg);
        }
      return;
    }
    case MOA_XPLAN_2D: {
      const int r = rank / grid_cols, c = rank % grid_cols;
      int64_t row0, rows, col0, cols;
      moa_lift_rows(m, grid_rows, r, &row0, &rows);
      moa_lift_rows(p, grid_cols, c, &col0, &cols);
      if (fused) out->add(MOA_COLL_BARRIER, MOA_COMM_WORLD, -1, 0, MOA_OPERAND_C, 0, -1, 0, 1);
      // A's row panel along the process row (root: column 0), B's column panel along
      // the process column (root: row 0): Figs. 4 and 5 together
      if (grid_cols > 1 && rows * n > 0) out->add(MOA_COLL_BROADCAST, MOA_COMM_ROW, 0, 0, MOA_OPERAND_A, 0, -1, 0, rows * n);
      if (grid_rows > 1 && n * cols > 0) out->add(MOA_COLL_BROADCAST, MOA_COMM_COL, 0, 0, MOA_OPERAND_B, 0, -1, 0, n * cols);
      if (fused) out->add(MOA_COLL_BARRIER, MOA_COMM_WORLD, -1, 0, MOA_OPERAND_C, 2, -1, 0, 1);
      return;
    }
    default: return;
  }
}

std::vector<moa_coll_t> plan_vec(int variant, int64_t m, int64_t n, int64_t p, int dtype, int G, int rank, int gr,
                                 int gc, int npanels, int flags) {
  PlanOut cnt{nullptr, 0};
  build_plan(variant, m, n, p, dtype, G, rank, gr, gc, npanels, flags, &cnt);
  std::vector<moa_coll_t> v((size_t)cnt.n);
  PlanOut out{v.data(), cnt.n};
  build_plan(variant, m, n, p, dtype, G, rank, gr, gc, npanels, flags, &out);
  return v;
}

}  // namespace

int moa_exchange_plan(int variant, int64_t m, int64_t n, int64_t p, int dtype, int nranks, int rank, int grid_rows,
                      int grid_cols, int npanels, int flags, moa_coll_t* ops, int max_ops, int* nops) {
  if (!nops || (max_ops > 0 && !ops)) {
    set_error("NULL argument");
    return MOA_ERR_NULL_POINTER;
  }
  if (variant < MOA_XPLAN_ROWS || variant > MOA_XPLAN_2D || m < 0 || n < 0 || p < 0 || nranks <= 0 || rank < 0 ||
      rank >= nranks || npanels < 0 || npanels > kMaxPanels || max_ops < 0 ||
      (variant == MOA_XPLAN_2D && (grid_rows <= 0 || grid_cols <= 0 || grid_rows * grid_cols != nranks))) {
    set_error("bad exchange-plan arguments");
    return MOA_ERR_INVALID_SHAPE;
  }
  if (elem_size(dtype) == 0) {
    set_error("unknown dtype");
    return MOA_ERR_INVALID_DTYPE;
  }
  int64_t t;
  if (!mul_ok(m, n, &t) || !mul_ok(n, p, &t) || !mul_ok(m, p, &t)) {
    set_error("extent product overflows int64");
    return MOA_ERR_INVALID_SHAPE;
  }
  PlanOut out{ops, max_ops};
  build_plan(variant, m, n, p, dtype, nranks, rank, grid_rows, grid_cols, npanels, flags, &out);
  *nops = out.n;
  if (out.n > max_ops) {
    set_error("ops array too small");
    return MOA_ERR_INVALID_SHAPE;
  }
  return MOA_OK;
}

// ---------------------------------- executors ----------------------------------

static const moa_comm_s::Window* find_window(moa_comm_t comm, const void* ptr, int64_t bytes);

// Barrier of the fused gather / pulled exchange: a one-element all-reduce on the
// stream. When it completes on rank r, every rank has finished the work it enqueued
// before it (for the exit barrier: its GEMM, whose peer stores are complete at
// kernel end, and its pulls, which its last GEMM waited for).
static int stream_barrier(moa_comm_t comm, cudaStream_t s) {
  if (comm->nranks <= 1) return MOA_OK;
  ncclResult_t r = ncclAllReduce(comm->barrier_buf, comm->barrier_buf, 1, ncclInt32, ncclMax, comm->nccl, s);
  return r == ncclSuccess ? MOA_OK : nccl_fail(r, "ncclAllReduce(barrier)");
}

static int split_2d(moa_comm_t comm, int grid_rows, int grid_cols) {
  if (comm->grid_rows == grid_rows && comm->grid_cols == grid_cols) return MOA_OK;
  const int r = comm->rank / grid_cols, c = comm->rank % grid_cols;
  if (comm->row_comm) ncclCommDestroy(comm->row_comm);
  if (comm->col_comm) ncclCommDestroy(comm->col_comm);
  comm->row_comm = comm->col_comm = nullptr;
  comm->grid_rows = comm->grid_cols = 0;
  ncclResult_t q = ncclCommSplit(comm->nccl, r, c, &comm->row_comm, nullptr);
  if (q == ncclSuccess) q = ncclCommSplit(comm->nccl, c, r, &comm->col_comm, nullptr);
  if (q != ncclSuccess) return nccl_fail(q, "ncclCommSplit(2-D grid)");
  comm->grid_rows = grid_rows;
  comm->grid_cols = grid_cols;
  return MOA_OK;
}

static int comm_of(moa_comm_t comm, int kind, ncclComm_t* out) {
  switch (kind) {
    case MOA_COMM_WORLD: *out = comm->nccl; return MOA_OK;
    case MOA_COMM_PIPE: return pipe_comm(comm, out);
    case MOA_COMM_ROW: *out = comm->row_comm; break;
    case MOA_COMM_COL: *out = comm->col_comm; break;
    default: *out = nullptr;
  }
  if (!*out) {
    set_error("sub-communicator missing for an exchange op");
    return MOA_ERR_NCCL;
  }
  return MOA_OK;
}

// Issue one NCCL op of a plan on stream s. `data` is the destination operand (the
// op's offset applies to it); `send` (broadcast roots only, may be NULL) is where a
// root's data comes from when it is not in place.
static int issue_nccl(moa_comm_t comm, const moa_coll_t& o, void* data, const void* send, int dtype, cudaStream_t s) {
  const int64_t es = elem_size(dtype);
  const ncclDataType_t ty = nccl_type(dtype);
  if (o.op == MOA_COLL_BARRIER) return stream_barrier(comm, s);
  ncclComm_t nc;
  int rc = comm_of(comm, o.comm, &nc);
  if (rc) return rc;
  char* dst = (char*)data + o.offset * es;
  ncclResult_t r;
  if (o.op == MOA_COLL_BROADCAST)
    r = ncclBroadcast(send ? send : dst, dst, (size_t)o.count, ty, o.root, nc, s);
  else if (o.op == MOA_COLL_ALLGATHER)
    r = ncclAllGather(send, dst, (size_t)o.count, ty, nc, s);
  else {
    set_error("not an NCCL op");
    return MOA_ERR_INVALID_SHAPE;
  }
  return r == ncclSuccess ? MOA_OK : nccl_fail(r, o.op == MOA_COLL_BROADCAST ? "ncclBroadcast" : "ncclAllGather");
}

// Row lifting: the plan's collectives around this rank's compute (Fig. 4 ip_rows.c,
// k = rank), shared by moa_gemm_lifted_ex and moa_gemm_lifted_gather. `last_peers`
// (fused gather) goes to the launch that writes the FINAL C, i.e. the last k-panel.
static int lifted_rows_exec(int64_t m, int64_t n, int64_t p, int64_t rows, const void* A_local, void* B,
                            void* C_local, void* C_full, int dtype, cudaStream_t s, moa_comm_t comm, int npanels,
                            int flags, const PeerDst* last_peers) {
  const int64_t es = elem_size(dtype);
  const int G = comm->nranks;
  const bool direct = flags & MOA_XF_DIRECT_B, pull = (flags & MOA_XF_PULL_B) && !direct;
  const std::vector<moa_coll_t> ops =
      plan_vec(MOA_XPLAN_ROWS, m, n, p, dtype, G, comm->rank, 0, 0, npanels, flags);
  // compute panels: the same boundaries as the plan's B ops (or one panel where no B
  // arrives: rank 0 of a pulled exchange computes its rows in one launch)
  int64_t bnd[kMaxPanels + 1];
  int K;
  if (pull)
    K = (G > 1 && comm->rank != 0) ? moa_pull_panels(n, bnd) : (bnd[0] = 0, bnd[1] = n, 1);
  else if (direct)
    K = (bnd[0] = 0, bnd[1] = n, 1);
  else
    K = nccl_panel_bounds(n, npanels > 0 ? npanels : moa_lift_panels(n, p, dtype, G), bnd);
  const moa_comm_s::Window* bwin = (pull || direct) ? find_window(comm, B, n * p * es) : nullptr;
  if ((pull || direct) && n * p > 0 && !bwin) {
    set_error("B is not inside a window of the communicator");
    return MOA_ERR_NOT_REGISTERED;
  }
  // direct: the GEMM's B operand is rank 0's copy, addressed through this process's
  // mapping of rank 0's window (NVLink load/store); rank 0 reads its own
  const void* Bsrc = B;
  if (direct && n * p > 0 && G > 1 && comm->rank != 0)
    Bsrc = (const char*)bwin->peer[0] + ((uintptr_t)B - (uintptr_t)bwin->ptr);
  cudaError_t e;
  int rc;
  Nvtx whole("moa lifted rows");
  // phase 0: entry barrier
  for (const auto& o : ops)
    if (o.phase == 0 && (rc = issue_nccl(comm, o, nullptr, nullptr, dtype, s))) return rc;
  Nvtx exch("moa exchange B");
  // phase 1: B's k-panels, on the side stream (when compute overlaps them) with one
  // event per panel, else on the compute stream
  bool has[kMaxPanels] = {};
  bool reserve_sms = false;  // NCCL panel broadcasts in flight need SMs of their own
  const bool side = K > 1;
  if (side) {
    if ((e = cudaEventRecord(comm->ev_start, s)) != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
    if ((e = cudaStreamWaitEvent(comm->side, comm->ev_start, 0)) != cudaSuccess)
      return cuda_fail(e, "cudaStreamWaitEvent");
  }
  for (const auto& o : ops) {
    if (o.phase != 1) continue;
    cudaStream_t os = side ? comm->side : s;
    if (o.op == MOA_COLL_PULL) {
      // copy-engine read of rank 0's copy over NVLink: no SMs, no NCCL kernel
      const uintptr_t off = (uintptr_t)B - (uintptr_t)bwin->ptr + (uintptr_t)(o.offset * es);
      e = cudaMemcpyAsync((char*)B + o.offset * es, (const char*)bwin->peer[(size_t)o.root] + off,
                          (size_t)(o.count * es), cudaMemcpyDeviceToDevice, os);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(pull B panel)");
    } else {
      if ((rc = issue_nccl(comm, o, B, nullptr, dtype, os))) return rc;
      if (o.comm == MOA_COMM_PIPE) reserve_sms = true;
    }
    if (side && o.panel >= 0 && o.panel < K) {
      if ((e = cudaEventRecord(comm->ev_panel[o.panel], os)) != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
      has[o.panel] = true;
    }
  }
  nvtxRangePop();  // (end of "moa exchange B": its ops are enqueued)
  nvtxRangePushA("moa lifted compute");
  // the lifted compute: this rank's rows of C, panel by panel. Panel j > 0 continues
  // every element's fma chain from panel j-1's C, so the result is bitwise the
  // one-launch result ("the addition loop to add up the blocks").
  for (int j = 0; j < K; ++j) {
    const int64_t k0 = bnd[j], k1 = bnd[j + 1];
    if (has[j] && (e = cudaStreamWaitEvent(s, comm->ev_panel[j], 0)) != cudaSuccess)
      return cuda_fail(e, "cudaStreamWaitEvent");
    if (k1 <= k0 && j > 0) continue;
    GemmArgs g{rows, k1 - k0, p, (const char*)A_local + k0 * es, (const char*)Bsrc + k0 * p * es, C_local,
               n > 0 ? n : 1, p > 0 ? p : 1, p > 0 ? p : 1, j > 0 ? 1 : 0};
    if (j == K - 1) g.peers = last_peers;  // the final panel writes the final C
    if ((rc = gemm_reserving(g, dtype, s, reserve_sms && j < K - 1 ? kPipeCTAs : 0))) return rc;
  }
  nvtxRangePop();
  nvtxRangePushA("moa gather C / exit barrier");  // (popped by exch's destructor)
  // phase 2: gather of C (reading R14) / exit barrier
  int group = 0;
  for (size_t i = 0; i < ops.size(); ++i) {
    const auto& o = ops[i];
    if (o.phase != 2) continue;
    if (o.group != group) {
      if (group && ncclGroupEnd() != ncclSuccess) return nccl_fail(ncclInternalError, "ncclGroupEnd");
      if (o.group && ncclGroupStart() != ncclSuccess) return nccl_fail(ncclInternalError, "ncclGroupStart");
      group = o.group;
    }
    const void* send = o.op == MOA_COLL_ALLGATHER ? C_local : (o.root == comm->rank ? C_local : nullptr);
    if ((rc = issue_nccl(comm, o, o.op == MOA_COLL_BARRIER ? nullptr : C_full, send, dtype, s))) {
      if (group) ncclGroupEnd();
      return rc;
    }
  }
  if (group) {
    ncclResult_t r = ncclGroupEnd();
    if (r != ncclSuccess) return nccl_fail(r, "ncclGroupEnd");
  }
  if ((flags & MOA_XF_GATHER) && !(flags & MOA_XF_FUSED_GATHER) && G == 1 && m * p > 0) {
    e = cudaMemcpyAsync(C_full, C_local, (size_t)(m * p * es), cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(C_full)");
  }
  return MOA_OK;
}

static bool overlap_bytes(const void* x, int64_t xb, const void* y, int64_t yb) {
  if (!x || !y || xb <= 0 || yb <= 0) return false;
  uintptr_t a0 = (uintptr_t)x, a1 = a0 + (uintptr_t)xb, b0 = (uintptr_t)y, b1 = b0 + (uintptr_t)yb;
  return a0 < b1 && b0 < a1;
}

int moa_gemm_lifted_ex(int64_t m, int64_t n, int64_t p, const void* A_local, void* B, void* C_local, void* C_full,
                       int dtype, void* stream, moa_comm_t comm, int npanels) {
  if (!comm) {
    set_error("NULL communicator");
    return MOA_ERR_NULL_POINTER;
  }
  if (m < 0) {
    set_error("negative extent");
    return MOA_ERR_INVALID_SHAPE;
  }
  if (npanels < 0 || npanels > kMaxPanels) {
    set_error("npanels out of range");
    return MOA_ERR_INVALID_SHAPE;
  }
  int64_t row0 = 0, rows = 0;
  int rc = moa_lift_rows(m, comm->nranks, comm->rank, &row0, &rows);
  if (rc) return rc;
  if ((rc = validate(rows, n, p, A_local, B, C_local, dtype))) return rc;
  const int64_t es = elem_size(dtype);
  if (C_full && (reinterpret_cast<uintptr_t>(C_full) % (uintptr_t)es) != 0) {
    set_error("C_full not aligned to the element size");
    return MOA_ERR_MISALIGNED;
  }
  if (C_full && (overlap_bytes(C_full, m * p * es, B, n * p * es) || overlap_bytes(C_full, m * p * es, A_local, rows * n * es) ||
                 overlap_bytes(C_full, m * p * es, C_local, rows * p * es))) {
    set_error("C_full overlaps another operand");
    return MOA_ERR_ALIASING;
  }
  // B inside a symmetric window (every rank): the exchange is copy-engine pulls
  int flags = C_full ? MOA_XF_GATHER : 0;
  if (comm->nranks > 1 && n * p > 0 && find_window(comm, B, n * p * es)) flags |= MOA_XF_PULL_B;
  return lifted_rows_exec(m, n, p, rows, A_local, B, C_local, C_full, dtype, (cudaStream_t)stream, comm, npanels,
                          flags, nullptr);
}

int moa_gemm_lifted_direct(int64_t m, int64_t n, int64_t p, const void* A_local, void* B, void* C_local,
                           void* C_full, int dtype, void* stream, moa_comm_t comm) {
  if (!comm) {
    set_error("NULL communicator");
    return MOA_ERR_NULL_POINTER;
  }
  if (m < 0) {
    set_error("negative extent");
    return MOA_ERR_INVALID_SHAPE;
  }
  int64_t row0 = 0, rows = 0;
  int rc = moa_lift_rows(m, comm->nranks, comm->rank, &row0, &rows);
  if (rc) return rc;
  if ((rc = validate(rows, n, p, A_local, B, C_local, dtype))) return rc;
  const int64_t es = elem_size(dtype);
  if (n * p > 0 && !find_window(comm, B, n * p * es)) {
    set_error("moa_gemm_lifted_direct: B must lie inside a window from moa_comm_alloc_window on every rank");
    return MOA_ERR_NOT_REGISTERED;
  }
  if (C_full && (reinterpret_cast<uintptr_t>(C_full) % (uintptr_t)es) != 0) {
    set_error("C_full not aligned to the element size");
    return MOA_ERR_MISALIGNED;
  }
  if (C_full && (overlap_bytes(C_full, m * p * es, B, n * p * es) || overlap_bytes(C_full, m * p * es, A_local, rows * n * es) ||
                 overlap_bytes(C_full, m * p * es, C_local, rows * p * es))) {
    set_error("C_full overlaps another operand");
    return MOA_ERR_ALIASING;
  }
  const int flags = (C_full ? MOA_XF_GATHER : 0) | MOA_XF_DIRECT_B;
  return lifted_rows_exec(m, n, p, rows, A_local, B, C_local, C_full, dtype, (cudaStream_t)stream, comm, 0, flags,
                          nullptr);
}

int moa_gemm_lifted_cols(int64_t m, int64_t n, int64_t p, void* A, const void* B_local, void* C_local, void* C_full,
                         void* workspace, int dtype, void* stream, moa_comm_t comm) {
  if (!comm) {
    set_error("NULL communicator");
    return MOA_ERR_NULL_POINTER;
  }
  if (p < 0) {
    set_error("negative extent");
    return MOA_ERR_INVALID_SHAPE;
  }
  const int G = comm->nranks;
  int64_t col0 = 0, cols = 0;
  int rc = moa_lift_rows(p, G, comm->rank, &col0, &cols);  // the split of the j axis
  if (rc) return rc;
  if ((rc = validate(m, n, cols, A, B_local, C_local, dtype))) return rc;
  const int64_t es = elem_size(dtype);
  // C_full inside a symmetric window (moa_comm_alloc_window), any dtype: the gather is
  // fused into the GEMM epilogue — this rank's column block is computed straight into
  // its columns of C_full (row stride p) and stored by the same epilogue into every
  // peer's C_full over NVLink; no workspace, no per-rank broadcasts of C.
  const moa_comm_s::Window* win =
      (C_full && m * p > 0 && G - 1 <= kMaxPeerDst)
          ? find_window(comm, C_full, m * p * es)
          : nullptr;
  if (C_full && m * p > 0 && !win) {
    if ((reinterpret_cast<uintptr_t>(C_full) % (uintptr_t)es) != 0) {
      set_error("C_full not aligned to the element size");
      return MOA_ERR_MISALIGNED;
    }
    if (G > 1 && !workspace) {
      set_error("gathering column blocks needs a workspace of m * ceil(p / G) elements");
      return MOA_ERR_NULL_POINTER;
    }
  }
  const int flags = win ? MOA_XF_FUSED_GATHER : (C_full && m * p > 0 ? MOA_XF_GATHER : 0);
  const std::vector<moa_coll_t> ops = plan_vec(MOA_XPLAN_COLS, m, n, p, dtype, G, comm->rank, 0, 0, 0, flags);
  cudaStream_t s = (cudaStream_t)stream;
  for (const auto& o : ops)  // phase 0: (entry barrier,) the broadcast of A
    if (o.phase == 0 && (rc = issue_nccl(comm, o, A, nullptr, dtype, s))) return rc;
  if (win) {
    PeerDst pd{};
    const uintptr_t off = (uintptr_t)C_full - (uintptr_t)win->ptr + (uintptr_t)(col0 * es);
    for (int r = 0; r < G; ++r)
      if (r != comm->rank && cols > 0) pd.dst[pd.nd++] = (char*)win->peer[(size_t)r] + off;
    GemmArgs g{m, n, cols, A, B_local, (char*)C_full + col0 * es, n > 0 ? n : 1, cols > 0 ? cols : 1, p, 0};
    g.peers = &pd;
    if (cols > 0 && (rc = gemm_impl(g, dtype, nullptr, s))) return rc;
    if (m * cols > 0) {  // C_local receives the block as documented (local strided copy)
      cudaError_t e = cudaMemcpy2DAsync(C_local, (size_t)(cols * es), (const char*)C_full + col0 * es, (size_t)(p * es),
                                        (size_t)(cols * es), (size_t)m, cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy2DAsync(C_local)");
    }
  } else if ((rc = moa_gemm(m, n, cols, A, B_local, C_local, dtype, stream))) {
    // this rank's column block: C[:, col0:col0+cols] = A • B[:, col0:col0+cols]
    return rc;
  }
  // phase 2: (exit barrier) or rank g's block through the workspace, then a strided
  // 2-D copy places it at columns [col0_g, col0_g + cols_g) of C_full
  for (const auto& o : ops) {
    if (o.phase != 2) continue;
    if (o.op == MOA_COLL_BARRIER) {
      if ((rc = stream_barrier(comm, s))) return rc;
      continue;
    }
    moa_coll_t w = o;
    w.offset = 0;  // the block lands at the start of the workspace
    if ((rc = issue_nccl(comm, w, workspace, o.root == comm->rank ? C_local : nullptr, dtype, s))) return rc;
    const int64_t cg = o.count / (m > 0 ? m : 1);
    cudaError_t e = cudaMemcpy2DAsync((char*)C_full + o.offset * es, (size_t)(p * es), workspace, (size_t)(cg * es),
                                      (size_t)(cg * es), (size_t)m, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy2DAsync(C_full)");
  }
  if (!win && C_full && m * p > 0 && G == 1) {
    cudaError_t e = cudaMemcpy2DAsync(C_full, (size_t)(p * es), C_local, (size_t)(cols * es), (size_t)(cols * es),
                                      (size_t)m, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy2DAsync(C_full)");
  }
  return MOA_OK;
}

static int lifted_2d_impl(int64_t m, int64_t n, int64_t p, int grid_rows, int grid_cols, void* A_panel,
                          void* B_panel, void* C_block, void* C_full, int dtype, void* stream, moa_comm_t comm) {
  if (!comm) {
    set_error("NULL communicator");
    return MOA_ERR_NULL_POINTER;
  }
  if (grid_rows <= 0 || grid_cols <= 0 || grid_rows * grid_cols != comm->nranks || m < 0 || p < 0) {
    set_error("grid_rows * grid_cols must equal the number of ranks");
    return MOA_ERR_INVALID_SHAPE;
  }
  const int r = comm->rank / grid_cols, c = comm->rank % grid_cols;
  int64_t row0, rows, col0, cols;
  int rc = moa_lift_rows(m, grid_rows, r, &row0, &rows);
  if (!rc) rc = moa_lift_rows(p, grid_cols, c, &col0, &cols);
  if (rc) return rc;
  if ((rc = validate(rows, n, cols, A_panel, B_panel, C_block, dtype))) return rc;
  const int64_t es = elem_size(dtype);
  const moa_comm_s::Window* win = nullptr;
  if (C_full && m * p > 0) {  // the fused gather: C_full must be a symmetric window
    if (comm->nranks - 1 > kMaxPeerDst) {
      set_error("moa_gemm_lifted_2d_gather: at most 9 ranks (one NVLink node)");
      return MOA_ERR_INVALID_SHAPE;
    }
    if (!(win = find_window(comm, C_full, m * p * es))) {
      set_error("C_full is not inside a window from moa_comm_alloc_window (of m*p elements)");
      return MOA_ERR_NOT_REGISTERED;
    }
  }
  cudaStream_t s = (cudaStream_t)stream;
  const std::vector<moa_coll_t> ops = plan_vec(MOA_XPLAN_2D, m, n, p, dtype, comm->nranks, comm->rank, grid_rows,
                                               grid_cols, 0, win ? MOA_XF_FUSED_GATHER : 0);
  if (comm->nranks > 1 && (rc = split_2d(comm, grid_rows, grid_cols))) return rc;  // collective, cached
  for (const auto& o : ops)
    if (o.phase == 0 && (rc = issue_nccl(comm, o, o.operand == MOA_OPERAND_A ? A_panel : B_panel, nullptr, dtype, s)))
      return rc;
  if (!win) return moa_gemm(rows, n, cols, A_panel, B_panel, C_block, dtype, stream);
  // fused gather: the block is computed into C_full at (row0, col0) with row stride p
  // and stored by the same epilogue into every other rank's C_full at that offset
  PeerDst pd{};
  const uintptr_t off = (uintptr_t)C_full - (uintptr_t)win->ptr + (uintptr_t)((row0 * p + col0) * es);
  for (int q = 0; q < comm->nranks; ++q)
    if (q != comm->rank && rows * cols > 0) pd.dst[pd.nd++] = (char*)win->peer[(size_t)q] + off;
  GemmArgs g{rows, n, cols, A_panel, B_panel, (char*)C_full + (row0 * p + col0) * es, n > 0 ? n : 1,
             cols > 0 ? cols : 1, p, 0};
  g.peers = &pd;
  if (rows * cols > 0 && (rc = gemm_impl(g, dtype, nullptr, s))) return rc;
  if (rows * cols > 0) {
    cudaError_t e = cudaMemcpy2DAsync(C_block, (size_t)(cols * es), (const char*)C_full + (row0 * p + col0) * es,
                                      (size_t)(p * es), (size_t)(cols * es), (size_t)rows, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy2DAsync(C_block)");
  }
  for (const auto& o : ops)  // exit barrier: every rank's epilogue stores are complete
    if (o.phase == 2 && (rc = issue_nccl(comm, o, nullptr, nullptr, dtype, s))) return rc;
  return MOA_OK;
}

int moa_gemm_lifted_2d(int64_t m, int64_t n, int64_t p, int grid_rows, int grid_cols, void* A_panel, void* B_panel,
                       void* C_block, int dtype, void* stream, moa_comm_t comm) {
  return lifted_2d_impl(m, n, p, grid_rows, grid_cols, A_panel, B_panel, C_block, nullptr, dtype, stream, comm);
}

int moa_gemm_lifted_2d_gather(int64_t m, int64_t n, int64_t p, int grid_rows, int grid_cols, void* A_panel,
                              void* B_panel, void* C_block, void* C_full, int dtype, void* stream, moa_comm_t comm) {
  if (comm && m * p > 0 && !C_full) {
    set_error("NULL C_full");
    return MOA_ERR_NULL_POINTER;
  }
  return lifted_2d_impl(m, n, p, grid_rows, grid_cols, A_panel, B_panel, C_block, C_full, dtype, stream, comm);
}

int moa_gemm_lifted(int64_t m, int64_t n, int64_t p, const void* A_local, void* B, void* C_local, void* C_full,
                    int dtype, void* stream, moa_comm_t comm) {
  return moa_gemm_lifted_ex(m, n, p, A_local, B, C_local, C_full, dtype, stream, comm, 0);
}

int moa_comm_agree(moa_comm_t comm, int local_status, int* global_status) {
  if (!comm || !global_status) {
    set_error("NULL argument");
    return MOA_ERR_NULL_POINTER;
  }
  if (comm->nranks <= 1) {
    *global_status = local_status;
    return MOA_OK;
  }
  int* d = comm->barrier_buf + 1;
  cudaError_t e = cudaMemcpyAsync(d, &local_status, sizeof(int), cudaMemcpyHostToDevice, comm->side);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(agree)");
  ncclResult_t r = ncclAllReduce(d, d, 1, ncclInt32, ncclMax, comm->nccl, comm->side);
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce(agree)");
  int out = 0;
  if ((e = cudaMemcpyAsync(&out, d, sizeof(int), cudaMemcpyDeviceToHost, comm->side)) != cudaSuccess ||
      (e = cudaStreamSynchronize(comm->side)) != cudaSuccess)
    return cuda_fail(e, "agree");
  *global_status = out;
  return MOA_OK;
}

}  // extern "C"

// ----------------------- fused GEMM -> all-gather (NEXT-1) -----------------------

int moa_gemm_scatter(int64_t m, int64_t n, int64_t p, const void* A, int64_t lda, const void* B, int64_t ldb,
                     void* C, int64_t ldc, int accumulate, int ndst, void* const* dst, int dtype, void* stream) {
  if (ndst < 0 || ndst > kMaxPeerDst) {
    set_error("ndst out of range [0, 8]");
    return MOA_ERR_INVALID_SHAPE;
  }
  GemmArgs g{m, n, p, A, B, C, lda, ldb, ldc, accumulate ? 1 : 0};
  int rc = validate_g(g, dtype);
  if (rc) return rc;
  const int64_t es = elem_size(dtype);
  if (ndst > 0 && m * p > 0 && !dst) {
    set_error("NULL dst array");
    return MOA_ERR_NULL_POINTER;
  }
  PeerDst pd{};
  pd.nd = m * p > 0 ? ndst : 0;
  const int64_t cb = m * p > 0 ? ((m - 1) * ldc + p) * es : 0;  // byte span of one strided m x p block
  for (int d = 0; d < pd.nd; ++d) {
    void* q = dst[d];
    if (!q) {
      set_error("NULL destination");
      return MOA_ERR_NULL_POINTER;
    }
    // element alignment is the contract; 16-byte alignment (with C's) selects the TMA
    // kernels' vector-store epilogue, anything else the generic kernels (tma_eligible)
    if (reinterpret_cast<uintptr_t>(q) % (uintptr_t)es) {
      set_error("destination not aligned to the element size");
      return MOA_ERR_MISALIGNED;
    }
    const int64_t ab = m * n > 0 ? ((m - 1) * lda + n) * es : 0, bb = n * p > 0 ? ((n - 1) * ldb + p) * es : 0;
    bool bad = overlap_bytes(q, cb, A, ab) || overlap_bytes(q, cb, B, bb) || overlap_bytes(q, cb, C, cb);
    for (int e2 = 0; e2 < d && !bad; ++e2) bad = overlap_bytes(q, cb, dst[e2], cb);
    if (bad) {
      set_error("destination overlaps an operand or another destination");
      return MOA_ERR_ALIASING;
    }
    pd.dst[d] = q;
  }
  g.peers = &pd;
  return gemm_impl(g, dtype, nullptr, (cudaStream_t)stream);
}

int moa_comm_alloc_window(moa_comm_t comm, size_t bytes, void** ptr) {
  if (!comm || !ptr) {
    set_error("NULL communicator or output pointer");
    return MOA_ERR_NULL_POINTER;
  }
  if (bytes == 0) {
    set_error("zero-byte window");
    return MOA_ERR_INVALID_SHAPE;
  }
  // every rank must be load/store-reachable (one NVLink/NVSwitch domain)
  if (lsa_team_size(comm->nccl) != comm->nranks) {
    set_error("not every rank is NVLink load/store-reachable (LSA team smaller than the communicator)");
    return MOA_ERR_NCCL;
  }
  // allocate on the communicator's device; the caller's current device is restored
  struct DeviceGuard {
    int prev = -1;
    ~DeviceGuard() {
      if (prev >= 0) cudaSetDevice(prev);
    }
  } guard;
  cudaError_t e = cudaGetDevice(&guard.prev);
  if (e == cudaSuccess) e = cudaSetDevice(comm->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  const size_t sz = (bytes + NCCL_WIN_REQUIRED_ALIGNMENT - 1) / NCCL_WIN_REQUIRED_ALIGNMENT * NCCL_WIN_REQUIRED_ALIGNMENT;
  moa_comm_s::Window w;
  w.bytes = bytes;
  ncclResult_t r = ncclMemAlloc(&w.ptr, sz);
  if (r != ncclSuccess) return nccl_fail(r, "ncclMemAlloc");
  r = ncclCommWindowRegister(comm->nccl, w.ptr, sz, &w.win, NCCL_WIN_COLL_SYMMETRIC);
  if (r != ncclSuccess) {
    ncclMemFree(w.ptr);
    return nccl_fail(r, "ncclCommWindowRegister");
  }
  w.peer.assign((size_t)comm->nranks, nullptr);
  // (rank r's own entry is NCCL's flat LSA mapping of the same physical memory: a
  // different virtual address than w.ptr)
  int rc = resolve_window_peers((void*)w.win, comm->nranks, w.peer.data());
  if (rc) {
    ncclCommWindowDeregister(comm->nccl, w.win);
    ncclMemFree(w.ptr);
    return rc;
  }
  comm->windows.push_back(w);
  *ptr = w.ptr;
  return MOA_OK;
}

int moa_comm_free_window(moa_comm_t comm, void* ptr) {
  if (!comm || !ptr) {
    set_error("NULL communicator or pointer");
    return MOA_ERR_NULL_POINTER;
  }
  for (size_t i = 0; i < comm->windows.size(); ++i)
    if (comm->windows[i].ptr == ptr) {
      cudaError_t e = cudaDeviceSynchronize();
      ncclResult_t r = ncclCommWindowDeregister(comm->nccl, comm->windows[i].win);
      ncclResult_t r2 = ncclMemFree(ptr);
      comm->windows.erase(comm->windows.begin() + (long)i);
      if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceSynchronize");
      if (r != ncclSuccess) return nccl_fail(r, "ncclCommWindowDeregister");
      if (r2 != ncclSuccess) return nccl_fail(r2, "ncclMemFree");
      return MOA_OK;
    }
  set_error("pointer is not a window of this communicator");
  return MOA_ERR_NOT_REGISTERED;
}

int moa_comm_window_peer(moa_comm_t comm, const void* ptr, int peer, void** out) {
  if (!comm || !ptr || !out) {
    set_error("NULL argument");
    return MOA_ERR_NULL_POINTER;
  }
  if (peer < 0 || peer >= comm->nranks) {
    set_error("peer out of range");
    return MOA_ERR_INVALID_INDEX;
  }
  for (const auto& w : comm->windows) {
    const uintptr_t a = (uintptr_t)ptr, b = (uintptr_t)w.ptr;
    if (a >= b && a < b + w.bytes) {
      *out = (char*)w.peer[(size_t)peer] + (a - b);
      return MOA_OK;
    }
  }
  set_error("pointer is not inside a window of this communicator");
  return MOA_ERR_NOT_REGISTERED;
}

// The window (moa_comm_alloc_window) holding [ptr, ptr + bytes), or nullptr.
static const moa_comm_s::Window* find_window(moa_comm_t comm, const void* ptr, int64_t bytes) {
  for (const auto& w : comm->windows) {
    const uintptr_t a = (uintptr_t)ptr, b = (uintptr_t)w.ptr;
    if (a >= b && a + (uintptr_t)bytes <= b + w.bytes) return &w;
  }
  return nullptr;
}

int moa_gemm_lifted_gather(int64_t m, int64_t n, int64_t p, const void* A_local, void* B, void* C_full, int dtype,
                           void* stream, moa_comm_t comm, int npanels) {
  if (!comm) {
    set_error("NULL communicator");
    return MOA_ERR_NULL_POINTER;
  }
  if (m < 0 || n < 0 || p < 0) {
    set_error("negative extent");
    return MOA_ERR_INVALID_SHAPE;
  }
  if (npanels < 0 || npanels > kMaxPanels) {
    set_error("npanels out of range");
    return MOA_ERR_INVALID_SHAPE;
  }
  if (comm->nranks - 1 > kMaxPeerDst) {
    set_error("moa_gemm_lifted_gather: at most 9 ranks (one NVLink node)");
    return MOA_ERR_INVALID_SHAPE;
  }
  int64_t row0 = 0, rows = 0;
  int rc = moa_lift_rows(m, comm->nranks, comm->rank, &row0, &rows);
  if (rc) return rc;
  const int64_t es = elem_size(dtype);
  int64_t mp;
  if (!mul_ok(m, p, &mp) || !mul_ok(mp, es, &mp)) {
    set_error("m*p overflows");
    return MOA_ERR_INVALID_SHAPE;
  }
  // C_full must lie inside one of this communicator's symmetric windows
  const moa_comm_s::Window* win = nullptr;
  if (mp > 0) {
    if (!C_full) {
      set_error("NULL C_full");
      return MOA_ERR_NULL_POINTER;
    }
    win = find_window(comm, C_full, mp);
    if (!win) {
      set_error("C_full is not inside a window from moa_comm_alloc_window (of m*p elements)");
      return MOA_ERR_NOT_REGISTERED;
    }
  }
  char* c_local = mp > 0 ? (char*)C_full + row0 * p * es : nullptr;
  if ((rc = validate(rows, n, p, A_local, B, c_local, dtype))) return rc;
  if (overlap_bytes(C_full, mp, B, n * p * es) || overlap_bytes(C_full, mp, A_local, rows * n * es)) {
    set_error("C_full overlaps another operand");
    return MOA_ERR_ALIASING;
  }
  if (mp == 0 && (n * p == 0 || comm->nranks == 1)) return MOA_OK;
  // peers: every other rank's copy of C_full, at this rank's rows
  PeerDst pd{};
  if (win && rows > 0) {
    const uintptr_t off = (uintptr_t)C_full - (uintptr_t)win->ptr + (uintptr_t)(row0 * p * es);
    for (int r = 0; r < comm->nranks; ++r)
      if (r != comm->rank) pd.dst[pd.nd++] = (char*)win->peer[(size_t)r] + off;
  }
  int flags = MOA_XF_FUSED_GATHER;
  if (comm->nranks > 1 && n * p > 0 && find_window(comm, B, n * p * es)) flags |= MOA_XF_PULL_B;
  return lifted_rows_exec(m, n, p, rows, A_local, B, c_local, nullptr, dtype, (cudaStream_t)stream, comm, npanels,
                          flags, pd.nd ? &pd : nullptr);
}
