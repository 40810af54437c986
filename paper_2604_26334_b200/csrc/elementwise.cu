// K2 / K6: RMSNorm, q/k-norm + RoPE + KV append, embedding gather, greedy
// argmax, casts and the deterministic weight initialiser.
//
// The reference folds all of this into `elementwise_epsilon` of the matmul
// FLOPs (`pkg/src/shardplan/model_graph.py:35,142`) and prices KV traffic
// as an ELEMENT_WISE request (`:164-171`). All of it is latency-bound at
// decode and bandwidth-bound (t x d) at prefill.
#include <string.h>

#include "common.cuh"
#include "../../include/pshard.h"

namespace ps {

// ---- deterministic counter-based initialiser (matches oracle/c/weights.c) ----
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void init_uniform_bf16_kernel(__nv_bfloat16* dst, size_t n, uint64_t seed,
                                         uint64_t offset, float scale, float bias) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    uint64_t z = mix64(seed ^ ((offset + i) * 0x9E3779B97F4A7C15ull));
    float u = (float)(z >> 40) * (1.0f / 16777216.0f);  // [0, 1), exact
    float w = 2.0f * u - 1.0f;                           // [-1, 1), exact
    dst[i] = __float2bfloat16_rn(fmaf(w, scale, bias));
  }
}

// Heavy-tailed row scale of the output head (margin-robust init, SURVEY.md §7 hard part 7):
// s_r = min(u_r^(-1/2), 64), u_r in (0, 1) from the row's own hash — Pareto(alpha = 2)
// row norms, so the top-1 logit of a random-init model usually stands clear of the
// runner-up and greedy ids are robust to bf16 rounding noise. Every step is a correctly
// rounded IEEE op (sqrt, div, min, mul), so the C oracle reproduces it bit for bit.
__device__ __forceinline__ float head_row_scale(uint64_t seed, uint64_t row) {
  uint64_t z = mix64((seed ^ 0xD1B54A32D192ED03ull) ^ (row * 0x9E3779B97F4A7C15ull));
  float u = ((float)(z >> 40) + 0.5f) * (1.0f / 16777216.0f);   // (0, 1), exact
  return fminf(__fdiv_rn(1.0f, __fsqrt_rn(u)), 64.0f);
}

__global__ void init_rowscaled_bf16_kernel(__nv_bfloat16* dst, size_t n, uint64_t seed, uint64_t offset,
                                           long long cols, float scale) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    const uint64_t e = offset + i;
    uint64_t z = mix64(seed ^ (e * 0x9E3779B97F4A7C15ull));
    float u = (float)(z >> 40) * (1.0f / 16777216.0f);
    float w = 2.0f * u - 1.0f;
    const float sr = __fmul_rn(scale, head_row_scale(seed, e / (uint64_t)cols));
    dst[i] = __float2bfloat16_rn(fmaf(w, sr, 0.0f));
  }
}

// ---- RMSNorm: out[r] = x[src_row(r)] * rsqrt(mean(x^2) + eps) * w ----
template <bool OUT_BF16>
__global__ void rmsnorm_kernel(const float* __restrict__ x, int ldx, const int* __restrict__ rows,
                               const __nv_bfloat16* __restrict__ w, int d, float eps,
                               void* __restrict__ out, int ldo) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[32];
  int r = blockIdx.x;
  int src = rows ? rows[r] : r;
  const float* xr = x + (long long)src * ldx;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) ss += xr[i] * xr[i];
  ss = block_sum(ss, red);
  float inv = rsqrtf(ss / (float)d + eps);
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    float v = xr[i] * inv * __bfloat162float(w[i]);
    if (OUT_BF16) static_cast<__nv_bfloat16*>(out)[(long long)r * ldo + i] = __float2bfloat16_rn(v);
    else static_cast<float*>(out)[(long long)r * ldo + i] = v;
  }
}

// GEMM-pass RMSNorm to bf16 (thousands of rows): 256 threads per row, the row held in
// registers as float4 (one read of x), 8-byte bf16x4 stores. The one-row-per-1024-thread
// kernel above re-read x and moved 4-byte words: 1.5 TB/s on a 16384 x 4096 prefill
// (CUPTI, config 4), ~16 ms of its TTFT.
constexpr int RMS_VEC_THREADS = 256, RMS_VEC_MAX = 8;   // d <= 4 * 256 * 8 = 8192
__global__ void __launch_bounds__(RMS_VEC_THREADS)
rmsnorm_bf16_vec_kernel(const float* __restrict__ x, int ldx, const int* __restrict__ rows,
                        const __nv_bfloat16* __restrict__ w, int d, float eps, __nv_bfloat16* __restrict__ out,
                        int ldo) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[32];
  const int r = blockIdx.x;
  const int src = rows ? rows[r] : r;
  const float4* xr = reinterpret_cast<const float4*>(x + (long long)src * ldx);
  const int n4 = d >> 2;
  float4 v[RMS_VEC_MAX];
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < RMS_VEC_MAX; ++j) {
    const int i = threadIdx.x + j * RMS_VEC_THREADS;
    v[j] = i < n4 ? __ldcs(xr + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    ss += v[j].x * v[j].x + v[j].y * v[j].y + v[j].z * v[j].z + v[j].w * v[j].w;
  }
  ss = block_sum(ss, red);
  const float inv = rsqrtf(ss / (float)d + eps);
  const uint2* w4 = reinterpret_cast<const uint2*>(w);
  uint2* o4 = reinterpret_cast<uint2*>(out + (long long)r * ldo);
#pragma unroll
  for (int j = 0; j < RMS_VEC_MAX; ++j) {
    const int i = threadIdx.x + j * RMS_VEC_THREADS;
    if (i < n4) {
      const uint2 wb = w4[i];
      const float2 w01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wb.x));
      const float2 w23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wb.y));
      const __nv_bfloat162 a = __floats2bfloat162_rn(v[j].x * inv * w01.x, v[j].y * inv * w01.y);
      const __nv_bfloat162 b = __floats2bfloat162_rn(v[j].z * inv * w23.x, v[j].w * inv * w23.y);
      uint2 o;
      o.x = *reinterpret_cast<const uint32_t*>(&a);
      o.y = *reinterpret_cast<const uint32_t*>(&b);
      o4[i] = o;
    }
  }
}

// ---- q/k norm + RoPE (rotate-half) + K/V append ----
// qkv row layout per token: [q heads (h*hd) | k heads (kv*hd) | v heads (kv*hd)]
// One warp per head; lane owns dims {lane + 32 j}. Pairs (i, i + hd/2) share a lane.
template <int HD>
__global__ void qkv_post_kernel(float* __restrict__ qkv, int ldq, int n_heads, int n_kv,
                                const int* __restrict__ pos, const int* __restrict__ req, KvPages kv,
                                const float2* __restrict__ rope,  // [ctx][HD/2] (cos, sin)
                                const __nv_bfloat16* __restrict__ q_norm,
                                const __nv_bfloat16* __restrict__ k_norm, float eps) {
  pdl_trigger();
  pdl_wait();
  constexpr int PER = HD / 32;
  constexpr int HALF = HD / 2;
  int tok = blockIdx.x;
  int head = blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int lane = threadIdx.x & 31;
  int total = n_heads + 2 * n_kv;
  if (head >= total) return;
  float* row = qkv + (long long)tok * ldq + (long long)head * HD;
  float v[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) v[j] = row[lane + 32 * j];

  bool is_q = head < n_heads, is_k = !is_q && head < n_heads + n_kv;
  const __nv_bfloat16* nw = is_q ? q_norm : (is_k ? k_norm : nullptr);
  if (nw) {
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < PER; ++j) ss += v[j] * v[j];
    ss = warp_sum(ss);
    float inv = rsqrtf(ss / (float)HD + eps);
#pragma unroll
    for (int j = 0; j < PER; ++j) v[j] = v[j] * inv * __bfloat162float(nw[lane + 32 * j]);
  }
  int p = pos[tok];
  if (is_q || is_k) {
    const float2* cs = rope + (long long)p * HALF;
#pragma unroll
    for (int j = 0; j < PER / 2; ++j) {
      int i = lane + 32 * j;  // i < HALF
      float2 c = cs[i];
      float a = v[j], b = v[j + PER / 2];
      v[j] = a * c.x - b * c.y;
      v[j + PER / 2] = b * c.x + a * c.y;
    }
  }
  if (is_q) {
#pragma unroll
    for (int j = 0; j < PER; ++j) row[lane + 32 * j] = v[j];
  } else {
    int r = req ? req[tok] : 0;
    int kvh = is_k ? head - n_heads : head - n_heads - n_kv;
    __nv_bfloat16* dst = kv.pool + kv.row(r, p) + (is_k ? 0 : (long long)n_kv * HD) + (long long)kvh * HD;
#pragma unroll
    for (int j = 0; j < PER; ++j) dst[lane + 32 * j] = __float2bfloat16_rn(v[j]);
  }
}

// ---- embedding gather (table may be host-mapped: zero-copy) ----
__global__ void embed_kernel(const __nv_bfloat16* __restrict__ table, const int* __restrict__ ids,
                             int d, float* __restrict__ out, int ldo) {
  pdl_trigger();
  pdl_wait();
  int r = blockIdx.x;
  const uint4* src = reinterpret_cast<const uint4*>(table + (long long)ids[r] * d);
  float* o = out + (long long)r * ldo;
  for (int i = threadIdx.x; i < d / 8; i += blockDim.x) {
    uint4 w = src[i];
    o[8 * i + 0] = bf16_lo(w.x); o[8 * i + 1] = bf16_hi(w.x);
    o[8 * i + 2] = bf16_lo(w.y); o[8 * i + 3] = bf16_hi(w.y);
    o[8 * i + 4] = bf16_lo(w.z); o[8 * i + 5] = bf16_hi(w.z);
    o[8 * i + 6] = bf16_lo(w.w); o[8 * i + 7] = bf16_hi(w.w);
  }
}

// ---- greedy argmax per row; ties -> lowest index (torch.argmax semantics) ----
__global__ void argmax_kernel(const float* __restrict__ logits, int V, int ldl, int* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  __shared__ float sv[32];
  __shared__ int si[32];
  const float* row = logits + (long long)blockIdx.x * ldl;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    float v = row[i];
    if (v > best || (v == best && i < bi)) { best = v; bi = i; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float ov = __shfl_xor_sync(0xffffffffu, best, o);
    int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { sv[warp] = best; si[warp] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    int nw = blockDim.x >> 5;
    for (int w = 1; w < nw; ++w)
      if (sv[w] > best || (sv[w] == best && si[w] < bi)) { best = sv[w]; bi = si[w]; }
    // w = 0 already folded in (thread 0 is lane 0 of warp 0)
    out[blockIdx.x] = bi;
  }
}

__global__ void cast_f32_bf16_kernel(const float* __restrict__ src, int lds, __nv_bfloat16* __restrict__ dst,
                                     int ldd, int rows, int cols) {
  long long n = (long long)rows * cols;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    long long r = i / cols, c = i - r * cols;
    dst[r * ldd + c] = __float2bfloat16_rn(src[r * lds + c]);
  }
}

__global__ void add_f32_kernel(float* __restrict__ dst, const float* __restrict__ src, long long n) {
  pdl_trigger();
  pdl_wait();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] += src[i];
}

}  // namespace ps

using namespace ps;

extern "C" {

int ps_init_uniform_bf16(void* dst, size_t n, unsigned long long seed, unsigned long long offset,
                         float scale, float bias, void* stream) {
  if (n == 0) return PS_OK;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 64) blocks = 148 * 64;
  init_uniform_bf16_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
      static_cast<__nv_bfloat16*>(dst), n, seed, offset, scale, bias);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

int ps_init_rowscaled_bf16(void* dst, size_t n, unsigned long long seed, unsigned long long offset,
                           long long cols, float scale, void* stream) {
  if (n == 0) return PS_OK;
  PS_REQUIRE(cols >= 1, "ps_init_rowscaled_bf16: cols=%lld", cols);
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 64) blocks = 148 * 64;
  init_rowscaled_bf16_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
      static_cast<__nv_bfloat16*>(dst), n, seed, offset, cols, scale);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

int ps_rmsnorm(const float* x, int ldx, const int* rows, int n_rows, const void* w, int d,
               float eps, void* out, int ldo, int out_bf16, void* stream) {
  if (n_rows <= 0) return PS_OK;
  int threads = d >= 1024 ? 1024 : ((d + 31) / 32) * 32;
  const bool vec = out_bf16 && n_rows >= 64 && d % 4 == 0 && d <= 4 * RMS_VEC_THREADS * RMS_VEC_MAX &&
                   ldx % 4 == 0 && ldo % 4 == 0 && ((uintptr_t)x & 15) == 0 && ((uintptr_t)out & 7) == 0 &&
                   ((uintptr_t)w & 7) == 0;
  if (vec)
    launch_k(rmsnorm_bf16_vec_kernel, n_rows, RMS_VEC_THREADS, 0, (cudaStream_t)stream, x, ldx, rows,
             static_cast<const __nv_bfloat16*>(w), d, eps, static_cast<__nv_bfloat16*>(out), ldo);
  else if (out_bf16)
    launch_k(rmsnorm_kernel<true>, n_rows, threads, 0, (cudaStream_t)stream,
             x, ldx, rows, static_cast<const __nv_bfloat16*>(w), d, eps, out, ldo);
  else
    launch_k(rmsnorm_kernel<false>, n_rows, threads, 0, (cudaStream_t)stream,
             x, ldx, rows, static_cast<const __nv_bfloat16*>(w), d, eps, out, ldo);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

int ps_qkv_rope_append(float* qkv, int ldq, int t, int n_heads, int n_kv, int head_dim,
                       const int* pos, const int* req, void* kv_pool, int row_elems, const int* block_table,
                       int bt_stride, int page_rows, const void* rope_cs, const void* q_norm,
                       const void* k_norm, float eps, void* stream) {
  if (t <= 0) return PS_OK;
  KvPages kv;
  PS_REQUIRE(kv_pages(kv, kv_pool, row_elems, block_table, bt_stride, page_rows),
             "ps_qkv_rope_append: bad paged cache (page_rows %d, bt_stride %d)", page_rows, bt_stride);
  PS_REQUIRE(row_elems == 2 * n_kv * head_dim, "ps_qkv_rope_append: row_elems %d != 2 * n_kv * head_dim", row_elems);
  int total = n_heads + 2 * n_kv;
  int warps = 8;
  dim3 grid(t, (total + warps - 1) / warps);
  auto cs = static_cast<const float2*>(rope_cs);
  auto qn = static_cast<const __nv_bfloat16*>(q_norm);
  auto kn = static_cast<const __nv_bfloat16*>(k_norm);
  cudaStream_t s = (cudaStream_t)stream;
  switch (head_dim) {
    case 64:
      launch_k(qkv_post_kernel<64>, grid, warps * 32, 0, s, qkv, ldq, n_heads, n_kv, pos, req, kv, cs, qn, kn, eps);
      break;
    case 128:
      launch_k(qkv_post_kernel<128>, grid, warps * 32, 0, s, qkv, ldq, n_heads, n_kv, pos, req, kv, cs, qn, kn, eps);
      break;
    default:
      ps_set_error("ps_qkv_rope_append: head_dim %d unsupported (64, 128)", head_dim);
      return PS_ERR_UNSUPPORTED;
  }
  PS_CHECK_LAUNCH();
  return PS_OK;
}

int ps_embed_gather(const void* table, const int* ids, int n, int d, float* out, int ldo,
                    void* stream) {
  PS_REQUIRE(d % 8 == 0, "ps_embed_gather: d must be a multiple of 8");
  if (n <= 0) return PS_OK;
  launch_k(embed_kernel, n, 128, 0, (cudaStream_t)stream, static_cast<const __nv_bfloat16*>(table), ids, d,
           out, ldo);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

int ps_argmax(const float* logits, int rows, int V, int ldl, int* out, void* stream) {
  if (rows <= 0) return PS_OK;
  launch_k(argmax_kernel, rows, 1024, 0, (cudaStream_t)stream, logits, V, ldl, out);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

int ps_cast_f32_bf16(const float* src, int lds, void* dst, int ldd, int rows, int cols,
                     void* stream) {
  long long n = (long long)rows * cols;
  if (n <= 0) return PS_OK;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  cast_f32_bf16_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
      src, lds, static_cast<__nv_bfloat16*>(dst), ldd, rows, cols);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

int ps_add_f32(float* dst, const float* src, long long n, void* stream) {
  if (n <= 0) return PS_OK;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  launch_k(add_f32_kernel, blocks, 256, 0, (cudaStream_t)stream, dst, src, n);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

}  // extern "C"

// ---- interleaved gate/up initialiser: dst row 2j <- tensor a row j, 2j+1 <- tensor b row j ----
namespace ps {
__global__ void init_interleaved_bf16_kernel(__nv_bfloat16* dst, long long rows_each, long long row_begin,
                                             long long n_rows, int cols, uint64_t seed_a, uint64_t seed_b,
                                             float scale, float bias) {
  long long n = n_rows * cols;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    long long r = row_begin + i / cols, c = i % cols;
    long long src_row = r >> 1;
    uint64_t seed = (r & 1) ? seed_b : seed_a;
    uint64_t idx = (uint64_t)(src_row * cols + c);
    uint64_t z = mix64(seed ^ (idx * 0x9E3779B97F4A7C15ull));
    float u = (float)(z >> 40) * (1.0f / 16777216.0f);
    dst[i] = __float2bfloat16_rn(fmaf(2.0f * u - 1.0f, scale, bias));
  }
}
}  // namespace ps

extern "C" int ps_init_interleaved_bf16(void* dst, long long rows_each, long long row_begin, long long n_rows,
                                        int cols, unsigned long long seed_a, unsigned long long seed_b,
                                        float scale, float bias, void* stream) {
  long long n = n_rows * cols;
  if (n <= 0) return PS_OK;
  PS_REQUIRE(row_begin + n_rows <= 2 * rows_each, "ps_init_interleaved_bf16: rows out of range");
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  ps::init_interleaved_bf16_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(
      static_cast<__nv_bfloat16*>(dst), rows_each, row_begin, n_rows, cols, seed_a, seed_b, scale, bias);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

namespace ps {
struct SmallBlob { unsigned char b[4000]; };
__global__ void upload_small_kernel(unsigned char* dst, SmallBlob blob, int n) {
  pdl_trigger();
  pdl_wait();
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = blob.b[i];
}
}  // namespace ps

// Host -> device copy of <= 4000 bytes carried in the kernel's parameter
// block: no copy engine is involved, so a tiny per-pass upload on the
// compute stream never queues behind multi-MB weight transfers.
extern "C" int ps_upload_small(void* dst, const void* src, int nbytes, void* stream) {
  PS_REQUIRE(nbytes >= 0 && nbytes <= 4000, "ps_upload_small: %d bytes > 4000", nbytes);
  if (nbytes == 0) return PS_OK;
  ps::SmallBlob blob;
  memcpy(blob.b, src, nbytes);
  ps::launch_k(ps::upload_small_kernel, 1, 256, 0, (cudaStream_t)stream, static_cast<unsigned char*>(dst), blob,
               nbytes);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

int ps_preload_elementwise() {
  using namespace ps;
  int n = 0;
  touch_kernel(init_uniform_bf16_kernel, n);
  touch_kernel(rmsnorm_kernel<true>, n);
  touch_kernel(rmsnorm_kernel<false>, n);
  touch_kernel(rmsnorm_bf16_vec_kernel, n);
  touch_kernel(qkv_post_kernel<64>, n);
  touch_kernel(qkv_post_kernel<128>, n);
  touch_kernel(embed_kernel, n);
  touch_kernel(argmax_kernel, n);
  touch_kernel(cast_f32_bf16_kernel, n);
  touch_kernel(add_f32_kernel, n);
  touch_kernel(init_interleaved_bf16_kernel, n);
  touch_kernel(upload_small_kernel, n);
  return n;
}
