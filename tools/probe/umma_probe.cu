// Minimal single-CTA tcgen05.mma probe: M=128, N=128, one MMA (K = 32 bytes), operands
// hand-written into 128B-swizzled shared memory, result read back via tcgen05.ld.
// Cases: 0 = bf16 A K-major / B K-major; 1 = tf32 K/K; 2 = tf32 A K-major / B MN-major.
// Also reports which of truncation / RN the TF32 datapath applies to fp32 inputs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint64_t layout = 2) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (layout << 61);
}

__global__ void k(int mode, float* out, float* dbg, float tval) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = s;            // 16 KiB
  uint8_t* sB = s + 16384;    // 16 KiB
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  int tid = threadIdx.x, warp = tid >> 5;
  // fill: A(r,k) = ((r + k) % 5) - 2 ; B(k,n) = ((k * 3 + n) % 7) - 3
  for (int i = tid; i < 16384 / 4; i += blockDim.x) { ((uint32_t*)sA)[i] = 0; ((uint32_t*)sB)[i] = 0; }
  __syncthreads();
  const int kel = mode == 0 ? 16 : 8;  // K elements per MMA
  const int es = mode == 0 ? 2 : 4;
  for (int i = tid; i < 128 * kel; i += blockDim.x) {
    int r = i / kel, kk = i % kel;
    float va = (float)(((r + kk) % 5) - 2);
    if (mode == 3 && r == 0 && kk == 0) va = tval;  // rounding probe
    int byte = kk * es;
    uint32_t off = r * 128 + ((((byte >> 4)) ^ (r & 7)) << 4) + (byte & 15);
    if (mode == 0) *(__nv_bfloat16*)(sA + off) = __float2bfloat16(va); else *(float*)(sA + off) = va;
  }
  for (int i = tid; i < 128 * kel; i += blockDim.x) {
    int n = i / kel, kk = i % kel;
    float vb = (float)(((kk * 3 + n) % 7) - 3);
    if (mode == 3) vb = (kk == 0 && n == 0) ? 1.0f : 0.0f;
    if (mode == 2 || mode == 3) {
      // MN-major, SWIZZLE_128B_BASE32B: element (k, n) in box n/32, k-row kk, 128-byte rows of
      // 32 floats, 32-byte chunk index XOR (kk & 3)
      int box = n >> 5, c = n & 31;
      int byte = c * 4;
      uint32_t off = box * 4096 + kk * 128 + ((((byte >> 5)) ^ (kk & 3)) << 5) + (byte & 31);
      *(float*)(sB + off) = vb;
    } else {
      int byte = kk * es;
      uint32_t off = n * 128 + ((((byte >> 4)) ^ (n & 7)) << 4) + (byte & 15);
      if (mode == 0) *(__nv_bfloat16*)(sB + off) = __float2bfloat16(vb); else *(float*)(sB + off) = vb;
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t tmem = tslot;
  if (tid == 0) {
    uint32_t idesc;
    uint64_t da = sdesc(su32(sA), 16, 1024), db;
    if (mode == 0) {
      idesc = (1u << 4) | (1u << 7) | (1u << 10) | (16u << 17) | (8u << 24);  // bf16 x bf16 -> f32, K/K
      db = sdesc(su32(sB), 16, 1024);
    } else if (mode == 1) {
      idesc = (1u << 4) | (2u << 7) | (2u << 10) | (16u << 17) | (8u << 24);  // tf32 K/K
      db = sdesc(su32(sB), 16, 1024);
    } else {
      idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) | (16u << 17) | (8u << 24);  // tf32 K/MN
      db = sdesc(su32(sB), 4096, 512, 1);
    }
    if (mode == 0)
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                   ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(0));
    else
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}"
                   ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  }
  // wait
  {
    uint32_t ok = 0;
    while (!ok) {
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
                   : "=r"(ok) : "r"(su32(&bar)) : "memory");
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // read: warp w (0..3) lanes 32w.. ; 128 columns in x16 chunks
  if (warp < 4) {
    int row = warp * 32 + (tid & 31);
    for (int c = 0; c < 128; c += 16) {
      uint32_t r[16];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                     "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                   : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int q = 0; q < 16; ++q) out[row * 128 + c + q] = __uint_as_float(r[q]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

int main() {
  float *out, *dbg;
  cudaMalloc(&out, 128 * 128 * 4);
  cudaMalloc(&dbg, 4096 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40960);
  static float h[128 * 128];
  for (int mode = 0; mode < 3; ++mode) {
    cudaMemset(out, 0xFF, 128 * 128 * 4);
    k<<<1, 256, 40960>>>(mode, out, dbg, 0.f);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    int kel = mode == 0 ? 16 : 8, bad = 0, nz = 0;
    for (int r = 0; r < 128; ++r)
      for (int n = 0; n < 128; ++n) {
        float ref = 0;
        for (int kk = 0; kk < kel; ++kk) ref += (float)(((r + kk) % 5) - 2) * (float)(((kk * 3 + n) % 7) - 3);
        if (h[r * 128 + n] != ref) ++bad;
        if (h[r * 128 + n] != 0) ++nz;
      }
    printf("mode %d: %s bad=%d nonzero=%d  C[0][0..3]=%g %g %g %g\n", mode, cudaGetErrorString(e), bad, nz, h[0], h[1],
           h[2], h[3]);
  }
  // rounding probe: A(0,0) = 1 + 2^-11 + 2^-13, B = e_00 -> D(0,0) = tf32(A00)
  float t = 1.0f + 0x1.0p-11f + 0x1.0p-13f;
  cudaMemset(out, 0, 128 * 128 * 4);
  k<<<1, 256, 40960>>>(3, out, dbg, t);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  printf("tf32 rounding probe (%s): in=%.10f out=%.10f  (trunc -> 1.0, RN -> %.10f)\n", cudaGetErrorString(e), t, h[0],
         1.0f + 0x1.0p-10f);
  return 0;
}
