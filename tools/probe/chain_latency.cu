// Dependent-chain latency of the two fp64 units on sm_100a (evidence for DESIGN §7,
// "why config0 stays latency-bound"): one warp, `chains` independent accumulators,
// each updated `iters` times in sequence; clock64 around the loop. cycles/step =
// elapsed / iters is the time one chain advances by one instruction (DMMA.8x8x4
// advances 4 k of every element it holds; DFMA advances 1 k). Not part of the library.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o chain_latency chain_latency.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int NACC>
__global__ void k_dmma_chain(long long* cyc, double* out, int iters, double seed) {
  double acc0[NACC], acc1[NACC];
  const double a = seed + threadIdx.x * 1e-3, b = seed * 0.5 + threadIdx.x * 1e-4;
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc0[i] = acc1[i] = 0.0;
  __syncwarp();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma(acc0[i], acc1[i], a, b);
  }
  __syncwarp();
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc0[i] + acc1[i];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (s == 12345.678) out[0] = s;
}

template <int NCH>
__global__ void k_dfma_chain(long long* cyc, double* out, int iters, double seed) {
  double acc[NCH];
  const double a = seed + threadIdx.x * 1e-3, b = seed * 0.5;
#pragma unroll
  for (int i = 0; i < NCH; ++i) acc[i] = i;
  __syncwarp();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) acc[i] = fma(a, acc[i], b);
  }
  __syncwarp();
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < NCH; ++i) s += acc[i];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (s == 12345.678) out[0] = s;
}

template <typename K>
static double run(K kern, int iters) {
  long long* d;
  double* o;
  CK(cudaMalloc(&d, sizeof(long long)));
  CK(cudaMalloc(&o, sizeof(double)));
  kern<<<1, 32>>>(d, o, iters, 1.0);  // warm-up
  CK(cudaDeviceSynchronize());
  kern<<<1, 32>>>(d, o, iters, 1.0);
  CK(cudaDeviceSynchronize());
  long long h = 0;
  CK(cudaMemcpy(&h, d, sizeof h, cudaMemcpyDeviceToHost));
  CK(cudaFree(d));
  CK(cudaFree(o));
  return (double)h / iters;
}

int main() {
  const int iters = 4096;
  int clk = 0;
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  printf("{\"probe\": \"chain_latency\", \"iters\": %d, \"max_clock_khz\": %d, \"rows\": [\n", iters, clk);
  const double d1 = run(k_dmma_chain<1>, iters), d2 = run(k_dmma_chain<2>, iters), d4 = run(k_dmma_chain<4>, iters),
               d8 = run(k_dmma_chain<8>, iters), d16 = run(k_dmma_chain<16>, iters);
  printf(" {\"unit\": \"DMMA.8x8x4 (4 k per step)\", \"cycles_per_step\": {\"1\": %.1f, \"2\": %.1f, \"4\": %.1f, \"8\": %.1f, \"16\": %.1f}},\n",
         d1, d2, d4, d8, d16);
  const double f1 = run(k_dfma_chain<1>, iters), f2 = run(k_dfma_chain<2>, iters), f4 = run(k_dfma_chain<4>, iters),
               f8 = run(k_dfma_chain<8>, iters), f16 = run(k_dfma_chain<16>, iters);
  printf(" {\"unit\": \"DFMA (1 k per step)\", \"cycles_per_step\": {\"1\": %.1f, \"2\": %.1f, \"4\": %.1f, \"8\": %.1f, \"16\": %.1f}}\n",
         f1, f2, f4, f8, f16);
  printf("], \"note\": \"one warp alone on the GPU; cycles_per_step with c chains = time for every chain to advance one instruction\"}\n");
  return 0;
}
