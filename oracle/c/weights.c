/*
 * ORACLE (test infrastructure only) — CPU restatement of the deterministic
 * weight initialiser that the product runs on the GPU (ps_init_uniform_bf16 /
 * ps_init_interleaved_bf16 in paper_2604_26334_b200/csrc/elementwise.cu).
 *
 *   z  = splitmix64 finaliser of (seed XOR ((offset + i) * 0x9E3779B97F4A7C15))
 *   u  = (z >> 40) * 2^-24                    in [0, 1), exact in fp32
 *   w  = fmaf(2u - 1, scale, bias)            single rounding (C99 fmaf)
 *   out = bf16 round-to-nearest-even of w
 *
 * Output head (ps_init_rowscaled_bf16): scale is multiplied by the row's
 *   s_r = min(1 / sqrtf(u_r), 64), u_r = ((z_r >> 40) + 0.5) * 2^-24,
 *   z_r = splitmix64 finaliser of ((seed ^ 0xD1B54A32D192ED03) XOR (row * 0x9E3779B97F4A7C15))
 * (correctly rounded IEEE sqrt / div / min / mul on both sides), bias 0.
 *
 * The reference (`shardplan`) has no weights at all; this
 * file is the only definition of model load the parity tests check against.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <pthread.h>
#include <string.h>

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline uint16_t f32_to_bf16_rne(float f) {
  uint32_t b;
  memcpy(&b, &f, 4);
  if ((b & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((b >> 16) | 0x40); /* NaN */
  b += 0x7fffu + ((b >> 16) & 1u);
  return (uint16_t)(b >> 16);
}

static inline uint16_t value(uint64_t seed, uint64_t idx, float scale, float bias) {
  uint64_t z = mix64(seed ^ (idx * 0x9E3779B97F4A7C15ull));
  float u = (float)(z >> 40) * (1.0f / 16777216.0f);
  return f32_to_bf16_rne(fmaf(2.0f * u - 1.0f, scale, bias));
}

static inline float head_row_scale(uint64_t seed, uint64_t row) {
  uint64_t z = mix64((seed ^ 0xD1B54A32D192ED03ull) ^ (row * 0x9E3779B97F4A7C15ull));
  float u = ((float)(z >> 40) + 0.5f) * (1.0f / 16777216.0f);
  float s = 1.0f / sqrtf(u);
  return s < 64.0f ? s : 64.0f;
}

/* n elements of a [rows x cols] output head from element `offset` (heavy-tailed rows) */
void oracle_init_rowscaled_bf16(uint16_t* dst, size_t n, uint64_t seed, uint64_t offset, long long cols,
                                float scale) {
  for (size_t i = 0; i < n; ++i) {
    uint64_t e = offset + i;
    volatile float sr = scale * head_row_scale(seed, e / (uint64_t)cols);
    dst[i] = value(seed, e, sr, 0.0f);
  }
}

typedef struct { uint16_t* dst; size_t lo, hi; uint64_t seed, offset; float scale, bias; } job_t;

static void* run_job(void* p) {
  job_t* j = (job_t*)p;
  for (size_t i = j->lo; i < j->hi; ++i) j->dst[i] = value(j->seed, j->offset + i, j->scale, j->bias);
  return NULL;
}

/* n elements of one tensor starting at element `offset`, on up to `threads` pthreads */
void oracle_init_uniform_bf16(uint16_t* dst, size_t n, uint64_t seed, uint64_t offset,
                              float scale, float bias, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 64) threads = 64;
  pthread_t tid[64];
  job_t jobs[64];
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (job_t){dst, n * t / threads, n * (t + 1) / threads, seed, offset, scale, bias};
    pthread_create(&tid[t], NULL, run_job, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
}

/* rows [0, 2*rows_each) of the interleaved gate/up matrix */
void oracle_init_interleaved_bf16(uint16_t* dst, long long rows_each, int cols, uint64_t seed_a,
                                  uint64_t seed_b, float scale, float bias) {
  for (long long r = 0; r < 2 * rows_each; ++r) {
    uint64_t seed = (r & 1) ? seed_b : seed_a;
    long long src = r >> 1;
    for (int c = 0; c < cols; ++c)
      dst[r * cols + c] = value(seed, (uint64_t)(src * cols + c), scale, bias);
  }
}

/* bf16 bits -> fp32, for the fp32 model oracle */
void oracle_bf16_to_f32(const uint16_t* src, float* dst, size_t n) {
  for (long long i = 0; i < (long long)n; ++i) {
    uint32_t b = (uint32_t)src[i] << 16;
    memcpy(&dst[i], &b, 4);
  }
}
