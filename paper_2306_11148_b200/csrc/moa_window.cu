// moa_window.cu — peer addresses of an NCCL symmetric window, for the fused
// GEMM -> all-gather epilogue (moa_gemm_lifted_gather).
//
// The row-lifted product has every rank g owning rows [row0_g, row0_g + rows_g) of
// C (Fig. 4 ip_rows.c); the optional gather of C (reading R14) lands
// every rank's rows in every rank's C_full. With C_full allocated by ncclMemAlloc
// and registered as a symmetric window, each rank's copy is load/store-reachable
// from every GPU of the NVLink/NVSwitch domain (the "LSA" team): K1's epilogue
// stores its final C tiles straight into the peers' copies. The addresses are
// resolved once per window with NCCL's device API (ncclGetPeerPointer) and cached
// on the host; the GEMM kernels receive them as plain pointers.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include "moa_internal.h"

namespace moa {
namespace {

__global__ void k_window_peers(ncclWindow_t w, int nranks, void** out) {
  const int r = (int)threadIdx.x;
  if (r < nranks) out[r] = ncclGetPeerPointer(w, 0, r);
}

}  // namespace

int lsa_team_size(void* comm) { return ncclTeamLsa((ncclComm_t)comm).nRanks; }

// out[r] = the address, in this process, of byte 0 of rank r's copy of window w.
// Synchronous (one tiny kernel + a copy on a private stream).
int resolve_window_peers(void* win, int nranks, void** out) {
  if (nranks <= 0 || nranks > 64) {
    set_error("resolve_window_peers: bad nranks");
    return MOA_ERR_INVALID_SHAPE;
  }
  RelaxedCapture relaxed_capture;
  cudaStream_t s = nullptr;
  void** d = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&d, sizeof(void*) * (size_t)nranks);
  if (e == cudaSuccess) {
    k_window_peers<<<1, 64, 0, s>>>((ncclWindow_t)win, nranks, d);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, d, sizeof(void*) * (size_t)nranks, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (d) cudaFree(d);
  if (s) cudaStreamDestroy(s);
  if (e != cudaSuccess) {
    set_error(std::string("resolve_window_peers: ") + cudaGetErrorString(e));
    return MOA_ERR_CUDA;
  }
  return MOA_OK;
}

}  // namespace moa
