/* Host implementation of the counter-based input generator (see moa_inputs.h). */
#include "moa_inputs.h"

static uint64_t mix64(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27; z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

uint64_t moa_gen_hash_host(uint64_t seed, uint64_t id, int64_t idx) {
  uint64_t key = mix64(seed * 0x9E3779B97F4A7C15ull + (id << 56) + 0x632BE59BD9B4E019ull);
  return mix64(key + ((uint64_t)idx + 1ull) * 0x9E3779B97F4A7C15ull);
}

void moa_gen_fill_f64_host(double* dst, int64_t count, uint64_t seed, uint64_t id, int kind, int64_t start) {
  for (int64_t t = 0; t < count; ++t) {
    uint64_t h = moa_gen_hash_host(seed, id, start + t);
    if (kind == MOA_GEN_INT) dst[t] = (double)((int)(h % 9ull) - 4);
    else dst[t] = (double)(h >> 11) * 0x1.0p-53 * 2.0 - 1.0;
  }
}

void moa_gen_fill_f32_host(float* dst, int64_t count, uint64_t seed, uint64_t id, int kind, int64_t start) {
  for (int64_t t = 0; t < count; ++t) {
    uint64_t h = moa_gen_hash_host(seed, id, start + t);
    if (kind == MOA_GEN_INT) dst[t] = (float)((int)(h % 9ull) - 4);
    else dst[t] = (float)(h >> 40) * 0x1.0p-24f * 2.0f - 1.0f;
  }
}
