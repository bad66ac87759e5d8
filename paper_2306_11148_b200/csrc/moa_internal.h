// moa_internal.h — product-internal interface between the C-ABI host layer
// (moa_host.cpp) and the kernel translation units. Not part of the ABI.
#pragma once
#include <cstdint>
#include <string>

#include <cuda_runtime.h>

#include "moa.h"

namespace moa {

// One-time library setup (pool allocation, kernel attributes, occupancy queries)
// may run during the caller's first call, which may be inside CUDA-graph stream
// capture. Those calls are not stream work, so the thread switches to relaxed
// capture mode for their duration (restored on scope exit).
struct RelaxedCapture {
  cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
  RelaxedCapture() { cudaThreadExchangeStreamCaptureMode(&mode); }
  ~RelaxedCapture() { cudaThreadExchangeStreamCaptureMode(&mode); }
  RelaxedCapture(const RelaxedCapture&) = delete;
  RelaxedCapture& operator=(const RelaxedCapture&) = delete;
};


// Per-device properties the static plan reads (cached, mutex-guarded).
struct DeviceShape {
  int device = -1;
  int sms = 0;
  int cc_major = 0, cc_minor = 0;
  int smem_optin = 0;          // sharedMemPerBlockOptin
  int smem_per_sm = 0;         // sharedMemPerMultiprocessor
  int regs_per_sm = 0;
  int64_t l2_bytes = 0;
};

// Thread-local error detail for moa_last_error().
void set_error(const std::string& s);

// One GEMM call as the kernels see it: row-major operands with leading dimensions
// (elements) lda >= n, ldb >= p, ldc >= p; accumulate != 0 continues the chain
// from the C in memory (C := C + A•B, each element's fma chain extended in k order).
// Extra destinations of the FINAL C tile (the fused GEMM -> all-gather epilogue of
// moa_gemm_lifted_gather): each dst[d] is an m x p row-major block with the same
// leading dimension as C, typically a peer GPU's C_full rows reached over NVLink
// (an NCCL symmetric-window address). Partial (stream-K head) values never go there.
constexpr int kMaxPeerDst = 8;
struct PeerDst {
  int nd;
  void* dst[kMaxPeerDst];
};

struct GemmArgs {
  int64_t m, n, p;
  const void* A;
  const void* B;
  void* C;
  int64_t lda, ldb, ldc;
  int accumulate;
  const PeerDst* peers = nullptr;  // fp64 only (K1/K2 epilogues); nullptr or nd == 0: none
};

// Kernel launchers (moa_dgemm.cu / moa_sgemm.cu / moa_tf32.cu). Arguments are
// validated by the host layer; the plan is a valid output of the chooser.
int launch_dgemm_tma(const moa_plan_t& plan, const GemmArgs& g, cudaStream_t stream);
int launch_dgemm_generic(const moa_plan_t& plan, const GemmArgs& g, cudaStream_t stream);
int launch_sgemm_ffma(const moa_plan_t& plan, const GemmArgs& g, cudaStream_t stream);
int launch_sgemm_generic(const moa_plan_t& plan, const GemmArgs& g, cudaStream_t stream);
int launch_sgemm_3xtf32(const moa_plan_t& plan, const GemmArgs& g, cudaStream_t stream);

// moa_window.cu: out[r] = this process's address of rank r's copy of an NCCL
// symmetric window (ncclWindow_t passed as void*). Synchronous.
int resolve_window_peers(void* win, int nranks, void** out);
// Size of NCCL's load/store-accessible (NVLink) team of a communicator (ncclComm_t).
int lsa_team_size(void* comm);

// ipophp siblings (moa_ipophp.cu); dense row-major operands, validated by the host.
int launch_hadamard(int64_t m, int64_t n, const void* A, const void* B, void* C, int dtype, cudaStream_t s);
int launch_kron(int64_t m, int64_t n, int64_t p, int64_t q, const void* A, const void* B, void* C, int dtype,
                cudaStream_t s);

// Static tile configurations compiled into the library (the chooser's candidates).
struct TileConfig {
  int kernel;
  int bm, bn, bk, stages, threads, ctas_per_sm, smem_bytes;
  double eta;  // per-tile efficiency prior (smaller tiles: more smem/L2 traffic per flop)
};
// Return the number of configs for a kernel id and fill *out (static storage).
#ifdef __CUDACC__
#define MOA_HD __host__ __device__
#else
#define MOA_HD
#endif
// K1 schedule choice (host chooser + launcher): the stream-K runs are used
// whenever the last wave is partial (moa_ptx.cuh sk_first_tile / sk_run).
MOA_HD inline bool use_stream_k(int64_t tiles, int64_t grid) {
  return grid > 0 && tiles > grid && tiles % grid != 0;
}

int dgemm_tile_configs(int kernel, const TileConfig** out);  // moa_dgemm.cu
int sgemm_tile_configs(int kernel, const TileConfig** out);  // moa_sgemm.cu
int tf32_tile_configs(int kernel, const TileConfig** out);   // moa_tf32.cu

}  // namespace moa
