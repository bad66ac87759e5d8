// Probe: can this box create an NVLS multicast object (CUDA driver multicast API) with
// one device, and does a multimem.st through its multicast address land in the bound
// memory? (Feasibility of a multimem.st variant of K1's fused-gather epilogue on a
// single-GPU lease.) Prints one JSON line.
#include <cstdio>
#include <cstring>
#include <cuda.h>
#include <cuda_runtime.h>

__global__ void k_mm(double* mc, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (2 * i + 1 < n) {
    const double a = 1.0 + i, b = -2.0 * i;
    const float2 x = *reinterpret_cast<const float2*>(&a), y = *reinterpret_cast<const float2*>(&b);
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + 2 * i), "f"(x.x),
                 "f"(x.y), "f"(y.x), "f"(y.y)
                 : "memory");
  }
}

#define CK(x)                                                                         \
  do {                                                                                \
    CUresult r_ = (x);                                                                \
    if (r_ != CUDA_SUCCESS) {                                                         \
      const char* s_ = nullptr;                                                       \
      cuGetErrorString(r_, &s_);                                                      \
      printf("{\"probe\":\"multicast\",\"step\":\"%s\",\"error\":\"%s\"}\n", #x, s_ ? s_ : "?"); \
      return 0;                                                                       \
    }                                                                                 \
  } while (0)

int main() {
  cudaFree(0);
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  int mc = 0;
  CK(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  if (!mc) {
    printf("{\"probe\":\"multicast\",\"supported\":0}\n");
    return 0;
  }
  const size_t n = 1 << 20, bytes = n * sizeof(double);
  CUmulticastObjectProp mp;
  memset(&mp, 0, sizeof(mp));
  mp.numDevices = 1;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  mp.size = (bytes + gran - 1) / gran * gran;
  CUmemGenericAllocationHandle mh, ph;
  // handle types tried in turn (the export type only matters for sharing across
  // processes): none, fabric, POSIX fd
  CUresult cr = CUDA_ERROR_INVALID_VALUE;
  const char* used = "";
  const CUmemAllocationHandleType types[3] = {CU_MEM_HANDLE_TYPE_NONE, CU_MEM_HANDLE_TYPE_FABRIC,
                                              CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR};
  const char* names[3] = {"none", "fabric", "posix_fd"};
  for (int i = 0; i < 3 && cr != CUDA_SUCCESS; ++i) {
    mp.handleTypes = types[i];
    cr = cuMulticastCreate(&mh, &mp);
    const char* es = nullptr;
    cuGetErrorString(cr, &es);
    printf("{\"probe\":\"multicast\",\"create_handle_type\":\"%s\",\"result\":\"%s\"}\n", names[i], es ? es : "?");
    used = names[i];
  }
  (void)used;
  CK(cr);
  CK(cuMulticastAddDevice(mh, dev));
  CUmemAllocationProp ap;
  memset(&ap, 0, sizeof(ap));
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  CK(cuMemCreate(&ph, mp.size, &ap, 0));
  CK(cuMulticastBindMem(mh, 0, ph, 0, mp.size, 0));
  CUdeviceptr uc = 0, mcp = 0;
  CK(cuMemAddressReserve(&uc, mp.size, gran, 0, 0));
  CK(cuMemMap(uc, mp.size, 0, ph, 0));
  CK(cuMemAddressReserve(&mcp, mp.size, gran, 0, 0));
  CK(cuMemMap(mcp, mp.size, 0, mh, 0));
  CUmemAccessDesc ad;
  ad.location = ap.location;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uc, mp.size, &ad, 1));
  CK(cuMemSetAccess(mcp, mp.size, &ad, 1));
  k_mm<<<(int)(n / 2 / 256), 256>>>(reinterpret_cast<double*>(mcp), (int)n);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("{\"probe\":\"multicast\",\"supported\":1,\"kernel\":\"%s\"}\n", cudaGetErrorString(e));
    return 0;
  }
  double h[8];
  cudaMemcpy(h, reinterpret_cast<void*>(uc), sizeof(h), cudaMemcpyDeviceToHost);
  const bool ok = h[0] == 1.0 && h[1] == 0.0 && h[2] == 2.0 && h[3] == -2.0 && h[6] == 4.0 && h[7] == -6.0;
  printf("{\"probe\":\"multicast\",\"supported\":1,\"granularity\":%zu,\"multimem_st_lands\":%s}\n", gran,
         ok ? "true" : "false");
  return 0;
}
