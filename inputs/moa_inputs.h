/* moa_inputs.h — seeded, counter-based synthetic input generator.
 *
 * This module is the ONLY code shared (by specification, not by linking) between
 * the CPU oracle side (tests, cpu_baseline) and the CUDA product side (bench,
 * parity tests). It holds none of the method's arithmetic: it only turns
 * (seed, matrix id, linear element index) into a value. The host
 * implementation (moa_inputs.c) and the device implementation
 * (moa_inputs_cuda.cu) are written separately and cross-checked bit-for-bit by
 * tests/test_inputs.py.
 *
 * Generator (splitmix64 stream, Steele et al.):
 *   key(seed,id)      = mix64(seed * 0x9E3779B97F4A7C15 + (id << 56) + 0x632BE59BD9B4E019)
 *   h(seed,id,idx)    = mix64(key + (idx + 1) * 0x9E3779B97F4A7C15)      (mod 2^64)
 *   mix64(z)          = z ^= z>>30; z *= 0xBF58476D1CE4E5B9; z ^= z>>27;
 *                       z *= 0x94D049BB133111EB; z ^= z>>31
 * Value kinds:
 *   MOA_GEN_UNIFORM : f64 = (h>>11)·2^-53·2 − 1  ∈ [−1,1), exact;  f32 = (h>>40)·2^-24·2 − 1
 *   MOA_GEN_INT     : (h mod 9) − 4 ∈ {−4..4}  (integer-valued: exact in f64/f32/tf32)
 * idx is the GLOBAL row-major linear index of the element (γ_row, PAPER.md
 * Eq. 3 addressing), so a rank that owns rows [r0, r0+rows) of A<m,n>
 * generates exactly the same values as a single process by passing
 * start = r0*n.
 */
#ifndef MOA_INPUTS_H
#define MOA_INPUTS_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { MOA_GEN_UNIFORM = 0, MOA_GEN_INT = 1 };

/* Host: fill dst[0..count) with values for linear indices start..start+count-1. */
void moa_gen_fill_f64_host(double* dst, int64_t count, uint64_t seed, uint64_t id, int kind, int64_t start);
void moa_gen_fill_f32_host(float* dst, int64_t count, uint64_t seed, uint64_t id, int kind, int64_t start);
uint64_t moa_gen_hash_host(uint64_t seed, uint64_t id, int64_t idx);

/* Device (libmoa_inputs_cuda.so): same contract, dst is device memory,
 * asynchronous on `stream` (a cudaStream_t passed as void*). Returns 0 or a
 * cudaError_t value. */
int moa_gen_fill_f64_device(double* dst, int64_t count, uint64_t seed, uint64_t id, int kind, int64_t start, void* stream);
int moa_gen_fill_f32_device(float* dst, int64_t count, uint64_t seed, uint64_t id, int kind, int64_t start, void* stream);

#ifdef __cplusplus
}
#endif
#endif
