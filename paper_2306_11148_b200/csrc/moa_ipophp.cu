// moa_ipophp.cu — the "ipophp" siblings of the MoA GEMM on the same row-major
// skeleton ("Matrix Multiplication (MM), Hadamard
// Product (HP), and the Kronecker Product (KP) using one algorithm/circuit").
//
//   Hadamard  C[(i*n)+j] = A[(i*n)+j] * B[(i*n)+j]                       (pointwise)
//   Kronecker C[((i*p)+k)*(n*q) + (j*q)+l] = A[(i*n)+j] * B[(k*q)+l]     (outer + ravel)
//
// Both are HBM-bound streams (no reuse to tile for): roofline = HBM bandwidth.
//  * Hadamard: 2 reads + 1 write per element, 128-bit vector accesses, streaming
//    cache hints, grid-stride persistent grid of SMs x 8 CTAs, 4 vectors in flight
//    per thread.
//  * Kronecker: write-bound (inputs are tiny and stay in L1/L2). Output row
//    r = i*p + k is the MoA axpy pattern without the sum: for each j, the scalar
//    A[i][j] times the contiguous row B[k][:] (Fig. 1's access order). Each CTA
//    streams whole output rows with 128-bit streaming stores.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "moa_internal.h"

namespace moa {
namespace {

template <typename T>
struct Vec;
template <>
struct Vec<double> {
  using V = double2;
  static constexpr int kN = 2;
};
template <>
struct Vec<float> {
  using V = float4;
  static constexpr int kN = 4;
};

__device__ __forceinline__ double2 pack(const double (&v)[2]) { return make_double2(v[0], v[1]); }
__device__ __forceinline__ float4 pack(const float (&v)[4]) { return make_float4(v[0], v[1], v[2], v[3]); }
__device__ __forceinline__ double2 vmul(double2 a, double2 b) { return make_double2(a.x * b.x, a.y * b.y); }
__device__ __forceinline__ double2 vscale(double a, double2 b) { return make_double2(a * b.x, a * b.y); }
__device__ __forceinline__ float4 vscale(float a, float4 b) { return make_float4(a * b.x, a * b.y, a * b.z, a * b.w); }
__device__ __forceinline__ float4 vmul(float4 a, float4 b) {
  return make_float4(a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w);
}

template <typename T>
__global__ void __launch_bounds__(256) k_hadamard_vec(const T* __restrict__ A, const T* __restrict__ B,
                                                      T* __restrict__ C, int64_t count) {
  using V = typename Vec<T>::V;
  constexpr int kN = Vec<T>::kN;
  constexpr int kU = 4;  // vectors in flight per thread
  const int64_t nvec = count / kN;
  const V* a = reinterpret_cast<const V*>(A);
  const V* b = reinterpret_cast<const V*>(B);
  V* c = reinterpret_cast<V*>(C);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (kU - 1) * stride < nvec; i += kU * stride) {
    V x[kU], y[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      x[u] = __ldcs(a + i + u * stride);
      y[u] = __ldcs(b + i + u * stride);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) __stcs(c + i + u * stride, vmul(x[u], y[u]));
  }
  for (; i < nvec; i += stride) __stcs(c + i, vmul(__ldcs(a + i), __ldcs(b + i)));
  // scalar tail
  const int64_t t0 = nvec * kN;
  for (int64_t t = t0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += stride) C[t] = A[t] * B[t];
}

template <typename T>
__global__ void __launch_bounds__(256) k_hadamard_scalar(const T* __restrict__ A, const T* __restrict__ B,
                                                         T* __restrict__ C, int64_t count) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += stride) C[t] = A[t] * B[t];
}

// One CTA per output row at a time (grid-stride over the m*p rows). Row
// r = i*p + k, column c = j*q + l. Vector path: the row length n*q is a multiple
// of the vector width and C is aligned, so each thread stores kN consecutive
// outputs (which may straddle two j's when q is small — handled per element).
// Fast path (q % kN == 0, 16-B aligned B and C): every output vector lies inside
// one j, so it is the scalar A[i][j] times one vector of the row B[k][:] — one
// broadcast load, one vector load, one streaming store; 4 stores in flight.
template <typename T>
__global__ void __launch_bounds__(256) k_kron_rowvec(const T* __restrict__ A, const T* __restrict__ B,
                                                     T* __restrict__ C, int64_t m, int64_t n, int64_t p, int64_t q) {
  using V = typename Vec<T>::V;
  constexpr int kN = Vec<T>::kN;
  constexpr int kU = 4;
  const int64_t rows = m * p, vcols = n * q / kN, qv = q / kN;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const int64_t i = r / p, k = r - i * p;
    const T* arow = A + i * n;
    const V* brow = reinterpret_cast<const V*>(B + k * q);
    V* crow = reinterpret_cast<V*>(C + r * n * q);
    const int64_t step = blockDim.x;
    const int64_t sj = step / qv, sl = step - sj * qv;
    int64_t c = threadIdx.x, j = c / qv, l = c - j * qv;
    for (; c + (kU - 1) * step < vcols; c += kU * step) {
      V out[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        out[u] = vscale(__ldg(arow + j), __ldg(brow + l));
        j += sj;
        l += sl;
        if (l >= qv) {
          l -= qv;
          ++j;
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) __stcs(crow + c + u * step, out[u]);
    }
    for (; c < vcols; c += step) {
      __stcs(crow + c, vscale(__ldg(arow + j), __ldg(brow + l)));
      j += sj;
      l += sl;
      if (l >= qv) {
        l -= qv;
        ++j;
      }
    }
  }
}

template <typename T, bool kVecStore>
__global__ void __launch_bounds__(256) k_kron(const T* __restrict__ A, const T* __restrict__ B, T* __restrict__ C,
                                              int64_t m, int64_t n, int64_t p, int64_t q) {
  using V = typename Vec<T>::V;
  constexpr int kN = Vec<T>::kN;
  const int64_t rows = m * p, cols = n * q;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const int64_t i = r / p, k = r - i * p;
    const T* arow = A + i * n;
    const T* brow = B + k * q;
    T* crow = C + r * cols;
    if (kVecStore) {
      // (j, l) of column c0 tracked incrementally: one division per row, none in the
      // loop (64-bit division is emulated and was the bottleneck).
      const int64_t step = (int64_t)blockDim.x * kN;
      const int64_t sj = step / q, sl = step - sj * q;
      int64_t c0 = (int64_t)threadIdx.x * kN;
      int64_t j = c0 / q, l = c0 - j * q;
      for (; c0 < cols; c0 += step) {
        T v[kN];
        int64_t jj = j, ll = l;
#pragma unroll
        for (int e = 0; e < kN; ++e) {
          v[e] = __ldg(arow + jj) * __ldg(brow + ll);
          if (++ll == q) {
            ll = 0;
            ++jj;
          }
        }
        __stcs(reinterpret_cast<V*>(crow + c0), pack(v));
        j += sj;
        l += sl;
        if (l >= q) {
          l -= q;
          ++j;
        }
      }
    } else {
      for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
        const int64_t j = c / q, l = c - j * q;
        crow[c] = __ldg(arow + j) * __ldg(brow + l);
      }
    }
  }
}

int grid_for(int64_t work_items, int per_block) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = (work_items + per_block - 1) / per_block;
  const int64_t cap = (int64_t)sms * 8;
  if (blocks > cap) blocks = cap;
  return (int)(blocks < 1 ? 1 : blocks);
}

int after_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return MOA_ERR_CUDA;
  }
  return MOA_OK;
}

template <typename T>
int hadamard_t(int64_t m, int64_t n, const void* A, const void* B, void* C, cudaStream_t s) {
  const int64_t count = m * n;
  const bool al = ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) | reinterpret_cast<uintptr_t>(C)) &
                   15u) == 0;
  if (al) {
    k_hadamard_vec<T><<<grid_for(count / Vec<T>::kN + 1, 256 * 4), 256, 0, s>>>((const T*)A, (const T*)B, (T*)C,
                                                                                 count);
  } else {
    k_hadamard_scalar<T><<<grid_for(count, 256 * 4), 256, 0, s>>>((const T*)A, (const T*)B, (T*)C, count);
  }
  return after_launch("k_hadamard");
}

template <typename T>
int kron_t(int64_t m, int64_t n, int64_t p, int64_t q, const void* A, const void* B, void* C, cudaStream_t s) {
  const int64_t rows = m * p, cols = n * q;
  const bool vec = (cols % Vec<T>::kN == 0) && ((reinterpret_cast<uintptr_t>(C) & 15u) == 0);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = rows < (int64_t)sms * 8 ? rows : (int64_t)sms * 8;
  const bool rowvec = (q % Vec<T>::kN == 0) &&
                      (((reinterpret_cast<uintptr_t>(B) | reinterpret_cast<uintptr_t>(C)) & 15u) == 0);
  if (rowvec)
    k_kron_rowvec<T><<<(unsigned)blocks, 256, 0, s>>>((const T*)A, (const T*)B, (T*)C, m, n, p, q);
  else if (vec)
    k_kron<T, true><<<(unsigned)blocks, 256, 0, s>>>((const T*)A, (const T*)B, (T*)C, m, n, p, q);
  else
    k_kron<T, false><<<(unsigned)blocks, 256, 0, s>>>((const T*)A, (const T*)B, (T*)C, m, n, p, q);
  return after_launch("k_kron");
}

}  // namespace

int launch_hadamard(int64_t m, int64_t n, const void* A, const void* B, void* C, int dtype, cudaStream_t s) {
  return dtype == MOA_F64 ? hadamard_t<double>(m, n, A, B, C, s) : hadamard_t<float>(m, n, A, B, C, s);
}

int launch_kron(int64_t m, int64_t n, int64_t p, int64_t q, const void* A, const void* B, void* C, int dtype,
                cudaStream_t s) {
  return dtype == MOA_F64 ? kron_t<double>(m, n, p, q, A, B, C, s) : kron_t<float>(m, n, p, q, A, B, C, s);
}

}  // namespace moa
