/*
 * inputs/gen.c — seeded synthetic WEIGHT generator shared by the oracle side and
 * the CUDA side (the only code both sides share; it holds none of the method's
 * arithmetic — no gate GEMV, no top-k, no cache, no FFN).
 *
 * Recipe (SURVEY.md §8(d) "Synthetic inputs"):
 *   value(seed, kind, layer, expert, flat) = (2u - 1) * a,  u = top 24 bits of a
 *   splitmix64 hash of the 5-tuple, a = sqrt(3/fan_in)  (so Var = 1/fan_in),
 *   rounded to bf16 with round-to-nearest-even.
 * `flat` is the flat index into the FULL (un-split) nn.Linear-layout matrix:
 *   W1, W3 : [ff][d]  flat = j*d + i     (fan_in = d)
 *   W2     : [d][ff]  flat = c*ff + j    (fan_in = ff)
 * so any row / column slice (tensor-parallel ranks, a 62 GB dev box) regenerates
 * bit-identically and independently.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

enum { KIND_GATE = 0, KIND_W1 = 1, KIND_W3 = 2, KIND_W2 = 3 };

static inline uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline uint64_t key_of(uint64_t seed, int kind, int layer, int expert) {
  uint64_t k = splitmix64(seed);
  k = splitmix64(k ^ ((uint64_t)(uint32_t)kind << 48));
  k = splitmix64(k ^ ((uint64_t)(uint32_t)layer << 24));
  k = splitmix64(k ^ (uint64_t)(uint32_t)expert);
  return k;
}

static inline uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  uint32_t lsb = (u >> 16) & 1u;
  u += 0x7FFFu + lsb;
  return (uint16_t)(u >> 16);
}

static inline uint16_t gen_one(uint64_t key, uint64_t flat, float scale) {
  uint64_t h = splitmix64(key ^ splitmix64(flat));
  int32_t q = (int32_t)(h >> 40) - (1 << 23); /* uniform integer in [-2^23, 2^23) */
  float v = (float)q * scale;                 /* exact product rounding, no transcendental */
  return f32_to_bf16_rne(v);
}

/* Rows [r0, r1) of a [rows_total][cols] matrix, all columns, into out[(r-r0)*cols + c]. */
void gen_rows(uint64_t seed, int kind, int layer, int expert, int64_t cols, float fan_in,
              int64_t r0, int64_t r1, uint16_t* out) {
  const uint64_t key = key_of(seed, kind, layer, expert);
  const float scale = sqrtf(3.0f / fan_in) / 8388608.0f;
#pragma omp parallel for schedule(static)
  for (int64_t r = r0; r < r1; ++r) {
    uint16_t* dst = out + (r - r0) * cols;
    for (int64_t c = 0; c < cols; ++c) dst[c] = gen_one(key, (uint64_t)(r * cols + c), scale);
  }
}

/* All rows, columns [c0, c1) of a [rows][cols_total] matrix into out[r*(c1-c0) + (c-c0)]. */
void gen_cols(uint64_t seed, int kind, int layer, int expert, int64_t rows, int64_t cols_total,
              float fan_in, int64_t c0, int64_t c1, uint16_t* out) {
  const uint64_t key = key_of(seed, kind, layer, expert);
  const float scale = sqrtf(3.0f / fan_in) / 8388608.0f;
  const int64_t w = c1 - c0;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r) {
    uint16_t* dst = out + r * w;
    for (int64_t c = c0; c < c1; ++c) dst[c - c0] = gen_one(key, (uint64_t)(r * cols_total + c), scale);
  }
}

/* float -> bf16 RNE for arrays (used to round generated hidden states / gate rows). */
void f32_to_bf16_array(const float* in, uint16_t* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = f32_to_bf16_rne(in[i]);
}
