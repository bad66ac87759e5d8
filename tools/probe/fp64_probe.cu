// Throwaway-style microbenchmark kept in-tree as evidence: measures the sm_100a
// fp64 tensor (DMMA.8x8x4) and fp64 FMA (DFMA) issue-limited peaks, FFMA/FFMA2
// peaks, and characterises the rounding of one mma.sync.m8n8k4.f64 against
// fma-chain / exact-sum models (SURVEY §8(c) pin P12). Not part of the library.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

template <int NACC>
__global__ void k_dmma(double* out, int iters, double seed) {
  double acc0[NACC], acc1[NACC];
  double a = seed + threadIdx.x * 1e-3, b = seed * 0.5 + threadIdx.x * 1e-4;
#pragma unroll
  for (int i = 0; i < NACC; ++i) { acc0[i] = 0.0; acc1[i] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma(acc0[i], acc1[i], a, b, acc0[i], acc1[i]);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc0[i] + acc1[i];
  if (s == 12345.678) out[0] = s;
}

template <int NCH>
__global__ void k_dfma(double* out, int iters, double seed) {
  double acc[NCH];
  double a = seed + threadIdx.x * 1e-3, b = seed * 0.5;
#pragma unroll
  for (int i = 0; i < NCH; ++i) acc[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) acc[i] = fma(a, acc[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NCH; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

template <int NCH>
__global__ void k_ffma(float* out, int iters, float seed) {
  float acc[NCH];
  float a = seed + threadIdx.x * 1e-3f, b = seed * 0.5f;
#pragma unroll
  for (int i = 0; i < NCH; ++i) acc[i] = (float)i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) acc[i] = fmaf(a, acc[i], b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < NCH; ++i) s += acc[i];
  if (s == 12345.678f) out[0] = s;
}

template <int NCH>
__global__ void k_ffma2(float* out, int iters, float seed) {
  float2 acc[NCH];
  float2 a = make_float2(seed + threadIdx.x * 1e-3f, seed - 1.f);
  float2 b = make_float2(seed * 0.5f, seed * 0.25f);
#pragma unroll
  for (int i = 0; i < NCH; ++i) acc[i] = make_float2((float)i, (float)-i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      unsigned long long r, x = *reinterpret_cast<unsigned long long*>(&acc[i]);
      unsigned long long aa = *reinterpret_cast<unsigned long long*>(&a);
      unsigned long long bb = *reinterpret_cast<unsigned long long*>(&b);
      asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(aa), "l"(x), "l"(bb));
      acc[i] = *reinterpret_cast<float2*>(&r);
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < NCH; ++i) s += acc[i].x + acc[i].y;
  if (s == 12345.678f) out[0] = s;
}

__device__ __forceinline__ uint64_t splitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ double urand(uint64_t c) {
  return (double)(splitmix(c) >> 11) * 0x1.0p-53 * 2.0 - 1.0;
}

// double-double helpers for the exact-sum model
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = a + b; double bb = s - a; e = (a - (s - bb)) + (b - bb);
}
// counts: [0]=fma chain k0..3 from c, [1]=fma chain k3..0, [2]=exact (dd) sum rounded once,
// [3]= c + ((p0+p1)+(p2+p3)) with rounded products, [4] = total elements
// mode 0: c random; mode 1: c = 0
__global__ void k_round(unsigned long long* counts, int mode, uint64_t seed) {
  int lane = threadIdx.x & 31;
  uint64_t base = seed * 0x100000000ull + (uint64_t)(blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32) * 256;
  __shared__ double sA[8][8 * 4], sB[8][4 * 8], sC[8][64];
  int w = threadIdx.x / 32;
  for (int i = lane; i < 32; i += 32) { sA[w][i] = urand(base + i); sB[w][i] = urand(base + 32 + i); }
  for (int i = lane; i < 64; i += 32) sC[w][i] = mode == 0 ? urand(base + 64 + i) : 0.0;
  __syncwarp();
  // fragments: A row=lane>>2, k=lane&3 ; B k=lane&3, n=lane>>2 ; C row=lane>>2, col=2*(lane&3)+{0,1}
  double a = sA[w][(lane >> 2) * 4 + (lane & 3)];
  double b = sB[w][(lane & 3) * 8 + (lane >> 2)];
  int r = lane >> 2, c0 = 2 * (lane & 3);
  double d0, d1;
  dmma(d0, d1, a, b, sC[w][r * 8 + c0], sC[w][r * 8 + c0 + 1]);
  double d[2] = {d0, d1};
  unsigned long long cnt[4] = {0, 0, 0, 0};
  for (int h = 0; h < 2; ++h) {
    int col = c0 + h;
    double c = sC[w][r * 8 + col];
    double p[4];
    for (int k = 0; k < 4; ++k) p[k] = sA[w][r * 4 + k] * sB[w][k * 8 + col];
    double m0 = c; for (int k = 0; k < 4; ++k) m0 = fma(sA[w][r * 4 + k], sB[w][k * 8 + col], m0);
    double m1 = c; for (int k = 3; k >= 0; --k) m1 = fma(sA[w][r * 4 + k], sB[w][k * 8 + col], m1);
    // exact sum via double-double accumulation of exact products
    double hi = c, lo = 0;
    for (int k = 0; k < 4; ++k) {
      double ph = sA[w][r * 4 + k] * sB[w][k * 8 + col];
      double pl = fma(sA[w][r * 4 + k], sB[w][k * 8 + col], -ph);
      double s, e; two_sum(hi, ph, s, e); lo += e + pl; hi = s;
    }
    double m2 = hi + lo;
    double m3 = c + ((p[0] + p[1]) + (p[2] + p[3]));
    cnt[0] += (d[h] == m0); cnt[1] += (d[h] == m1); cnt[2] += (d[h] == m2); cnt[3] += (d[h] == m3);
  }
  for (int i = 0; i < 4; ++i) atomicAdd(&counts[i], cnt[i]);
  atomicAdd(&counts[4], 2ull);
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"device\":\"%s\",\"sms\":%d,\"clock_rate_khz\":%d}\n", prop.name, sms, clk_khz);
  void* out; CK(cudaMalloc(&out, 64));
  const int iters = 20000;
  // DMMA: warps per SM sweep
  for (int wps : {4, 8, 16, 32}) {
    for (int bps : {1, 2}) {
      int block = 32 * wps / bps; if (block > 1024) continue;
      int grid = sms * bps;
      float ms;
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      k_dmma<8><<<grid, block>>>((double*)out, iters, 1.0); CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      k_dmma<8><<<grid, block>>>((double*)out, iters, 1.0);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      double flops = (double)grid * (block / 32) * iters * 8 * 512.0;
      printf("{\"probe\":\"dmma_m8n8k4\",\"warps_per_sm\":%d,\"ctas_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n",
             wps, bps, ms, flops / ms / 1e9);
    }
  }
  for (int wps : {8, 16, 32}) {
    int block = 32 * wps; int grid = sms;
    float ms; cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k_dfma<8><<<grid, block>>>((double*)out, iters, 1.0); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    k_dfma<8><<<grid, block>>>((double*)out, iters, 1.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = (double)grid * block * iters * 8 * 2.0;
    printf("{\"probe\":\"dfma\",\"warps_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n", wps, ms, flops / ms / 1e9);
  }
  for (int wps : {16, 32}) {
    int block = 32 * wps; int grid = sms;
    float ms; cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k_ffma<8><<<grid, block>>>((float*)out, iters * 4, 1.0f); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    k_ffma<8><<<grid, block>>>((float*)out, iters * 4, 1.0f);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = (double)grid * block * iters * 4 * 8 * 2.0;
    printf("{\"probe\":\"ffma\",\"warps_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n", wps, ms, flops / ms / 1e9);
    k_ffma2<8><<<grid, block>>>((float*)out, iters * 4, 1.0f); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    k_ffma2<8><<<grid, block>>>((float*)out, iters * 4, 1.0f);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    flops = (double)grid * block * iters * 4 * 8 * 4.0;
    printf("{\"probe\":\"ffma2\",\"warps_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n", wps, ms, flops / ms / 1e9);
  }
  {  // sustained: ~5 s of DMMA at 16 warps/SM, to see the clock under a long fp64 load
    int block = 512, grid = sms; float ms; cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int it2 = 20000 * 8;
    cudaEventRecord(e0);
    for (int rep = 0; rep < 3; ++rep) k_dmma<8><<<grid, block>>>((double*)out, it2, 1.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 3.0 * grid * (block / 32) * (double)it2 * 8 * 512.0;
    printf("{\"probe\":\"dmma_sustained\",\"ms\":%.3f,\"tflops\":%.3f}\n", ms, flops / ms / 1e9);
  }
  unsigned long long* cnt; CK(cudaMalloc(&cnt, 8 * sizeof(unsigned long long)));
  for (int mode : {0, 1}) {
    CK(cudaMemset(cnt, 0, 8 * sizeof(unsigned long long)));
    k_round<<<4096, 256>>>(cnt, mode, 7 + mode);
    CK(cudaDeviceSynchronize());
    unsigned long long h[8]; CK(cudaMemcpy(h, cnt, sizeof(h), cudaMemcpyDeviceToHost));
    printf("{\"probe\":\"dmma_rounding\",\"c\":\"%s\",\"total\":%llu,\"fma_chain_k0to3\":%llu,"
           "\"fma_chain_k3to0\":%llu,\"exact_sum_rounded_once\":%llu,\"rounded_products_pairwise\":%llu}\n",
           mode == 0 ? "random" : "zero", h[4], h[0], h[1], h[2], h[3]);
  }
  return 0;
}
