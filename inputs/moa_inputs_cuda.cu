// Device implementation of the counter-based input generator (see moa_inputs.h).
// Written independently of moa_inputs.c; tests/test_inputs.py checks both give
// identical bits. Grid-stride, one element per thread per iteration.
#include <cuda_runtime.h>
#include "moa_inputs.h"

namespace {
__device__ __forceinline__ uint64_t d_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <typename T>
__global__ void k_fill(T* __restrict__ dst, int64_t count, uint64_t key, int kind, int64_t start) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += stride) {
    uint64_t h = d_mix64(key + ((uint64_t)(start + t) + 1ull) * 0x9E3779B97F4A7C15ull);
    T v;
    if (kind == MOA_GEN_INT) v = (T)((int)(h % 9ull) - 4);
    else if (sizeof(T) == 8) v = (T)((double)(h >> 11) * 0x1.0p-53 * 2.0 - 1.0);
    else v = (T)((float)(h >> 40) * 0x1.0p-24f * 2.0f - 1.0f);
    dst[t] = v;
  }
}

template <typename T>
int fill(T* dst, int64_t count, uint64_t seed, uint64_t id, int kind, int64_t start, void* stream) {
  if (count <= 0) return 0;
  uint64_t z = seed * 0x9E3779B97F4A7C15ull + (id << 56) + 0x632BE59BD9B4E019ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  uint64_t key = z ^ (z >> 31);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = (count + 255) / 256;
  int64_t cap = (int64_t)sms * 8;
  if (blocks > cap) blocks = cap;
  k_fill<T><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(dst, count, key, kind, start);
  return (int)cudaGetLastError();
}
}  // namespace

extern "C" int moa_gen_fill_f64_device(double* dst, int64_t count, uint64_t seed, uint64_t id, int kind,
                                       int64_t start, void* stream) {
  return fill<double>(dst, count, seed, id, kind, start, stream);
}
extern "C" int moa_gen_fill_f32_device(float* dst, int64_t count, uint64_t seed, uint64_t id, int kind,
                                       int64_t start, void* stream) {
  return fill<float>(dst, count, seed, id, kind, start, stream);
}
