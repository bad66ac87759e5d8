// FFMA / FFMA2 issue-mix probe (sm_100a): throughput of independent fma chains when a
// thread interleaves N2 packed FFMA2 chains with N1 scalar FFMA chains. Tells whether
// the exact-fp32 K3 kernel (FFMA2-only, ~87% of the FFMA pipe in a pure loop) could
// gain from mixing in scalar FFMA. Prints one JSON line per (N2, N1, warps/SM).
#include <cstdio>
#include <cuda_runtime.h>

template <int N2, int N1>
__global__ void k_mix(float* out, int iters, float seed) {
  unsigned long long acc2[N2 > 0 ? N2 : 1];
  float acc1[N1 > 0 ? N1 : 1];
  float a = seed + threadIdx.x * 1e-3f, b = seed * 0.5f;
  float2 a2f = make_float2(a, a), b2f = make_float2(b, b * 0.5f);
  unsigned long long a2 = *reinterpret_cast<unsigned long long*>(&a2f);
  unsigned long long b2 = *reinterpret_cast<unsigned long long*>(&b2f);
#pragma unroll
  for (int i = 0; i < (N2 > 0 ? N2 : 1); ++i) {
    float2 v = make_float2((float)i, (float)-i);
    acc2[i] = *reinterpret_cast<unsigned long long*>(&v);
  }
#pragma unroll
  for (int i = 0; i < (N1 > 0 ? N1 : 1); ++i) acc1[i] = (float)i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < (N2 > N1 ? N2 : N1); ++i) {
      if (i < N2) asm volatile("fma.rn.f32x2 %0, %1, %0, %2;" : "+l"(acc2[i]) : "l"(a2), "l"(b2));
      if (i < N1) asm volatile("fma.rn.f32 %0, %1, %0, %2;" : "+f"(acc1[i]) : "f"(a), "f"(b));
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < N2; ++i) s += __int_as_float((int)acc2[i]);
#pragma unroll
  for (int i = 0; i < N1; ++i) s += acc1[i];
  if (s == 12345.678f) out[0] = s;
}

// Outer-product operand pattern of K3: 16 accumulator pairs c[r][q] (r < 8 rows,
// q < 2 column pairs... here 8 x 2), the A scalar broadcast (.F32 operand) from 8
// row registers and the B pair from 2 pair registers; ORDER 0 = rows outer (A reused
// by consecutive FFMA2), 1 = B pair outer (B reused).
template <int ORDER>
__global__ void k_outer(float* out, int iters, float seed) {
  unsigned long long c[8][2];
  float a[8];
  unsigned long long b[2];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    a[r] = seed + r * 1e-3f + threadIdx.x * 1e-6f;
    for (int q = 0; q < 2; ++q) {
      float2 v = make_float2((float)r, (float)q);
      c[r][q] = *reinterpret_cast<unsigned long long*>(&v);
    }
  }
  for (int q = 0; q < 2; ++q) {
    float2 v = make_float2(seed * 0.5f + q + threadIdx.x * 1e-7f, seed * 0.25f - q - threadIdx.x * 1e-7f);
    b[q] = *reinterpret_cast<unsigned long long*>(&v);
  }
  for (int it = 0; it < iters; ++it) {
    if (ORDER == 0) {
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          unsigned long long aa;
          asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a[r]));
          asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c[r][q]) : "l"(aa), "l"(b[q]));
        }
    } else {
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          unsigned long long aa;
          asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a[r]));
          asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c[r][q]) : "l"(aa), "l"(b[q]));
        }
    }
  }
  float s = 0;
#pragma unroll
  for (int r = 0; r < 8; ++r)
    for (int q = 0; q < 2; ++q) s += __int_as_float((int)c[r][q]);
  if (s == 12345.678f) out[0] = s;
}

template <int ORDER>
void run_outer(float* out, int sms, int wps) {
  const int iters = 20000, block = 32 * wps, grid = sms;
  k_outer<ORDER><<<grid, block>>>(out, iters, 1.0f);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_outer<ORDER><<<grid, block>>>(out, iters, 1.0f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double flops = 2.0 * 2.0 * 16 * iters * (double)block * grid;
  printf("{\"probe\":\"ffma2_outer\",\"order\":\"%s\",\"warps_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n",
         ORDER == 0 ? "rows_outer_A_reused" : "pairs_outer_B_reused", wps, ms, flops / ms / 1e9);
}

template <int N2, int N1>
void run(float* out, int sms, int wps) {
  const int iters = 20000, block = 32 * wps, grid = sms;
  k_mix<N2, N1><<<grid, block>>>(out, iters, 1.0f);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_mix<N2, N1><<<grid, block>>>(out, iters, 1.0f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double flops = 2.0 * (2.0 * N2 + N1) * iters * (double)block * grid;
  printf("{\"probe\":\"ffma_mix\",\"ffma2_chains\":%d,\"ffma_chains\":%d,\"warps_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n",
         N2, N1, wps, ms, flops / ms / 1e9);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, 16);
  for (int wps : {8, 16}) {
    run_outer<0>(out, sms, wps);
    run_outer<1>(out, sms, wps);
  }
  for (int wps : {8, 16, 32}) {
    run<8, 0>(out, sms, wps);
    run<0, 16>(out, sms, wps);
    run<8, 4>(out, sms, wps);
    run<8, 8>(out, sms, wps);
    run<6, 8>(out, sms, wps);
    run<4, 8>(out, sms, wps);
    run<16, 0>(out, sms, wps);
  }
  return 0;
}
