// K4: attention over the per-request KV blocks, GQA/MHA.
//
// Prices: GQA (t, ctx, h, kv, hd) / MHA requests, flops 4*t*ctx*h*hd
// (`pkg/src/shardplan/model_graph.py:154-161`). The cache is PAGED (KvPages,
// common.cuh): request slot s's position p lives in physical page
// table[s][p / page_rows], row p % page_rows; a row is bf16 [K heads | V heads].
//
// * decode (t = 1 per request): split-KV. Each CTA owns a contiguous range
//   of positions for one kv head and all of its G query heads; a warp scores
//   32 positions at once (lane = position), keeps an online softmax, and
//   accumulates V with lanes owning contiguous dims. Splits are merged by a
//   second small kernel. HBM-bound on the cache.
// * prefill (t new tokens per request, causal, varlen): flash attention on
//   the legacy mma.sync m16n8k16 bf16 tensor-core path (FA2 register
//   layout: S = Q K^T and O += P V with P kept in registers), 64 queries
//   per CTA, 64-key tiles staged in padded shared memory, V fragments via
//   ldmatrix.trans.
#include <float.h>

#include <type_traits>

#include "common.cuh"
#include "../../include/pshard.h"

namespace ps {

// ------------------------------- decode -------------------------------------
#define PS_DECODE_CHUNK 128  // positions per split (4 warps x 32)
template <int HD, int G>
__global__ void __launch_bounds__(128)
attn_decode_kernel(const float* __restrict__ q, int ldq, KvPages kv, const int* __restrict__ req_slot,
                   const int* __restrict__ lens, int n_kv, int chunk, float scale,
                   float* __restrict__ out, int ldo, float* __restrict__ ws_o, float* __restrict__ ws_ml,
                   int n_splits) {
  pdl_trigger();
  pdl_wait();
  constexpr int PER = HD / 32;
  __shared__ __align__(16) float qs[G][HD];
  __shared__ float red_ml[4][G][2];
  __shared__ __align__(16) float red_o[4][G][HD];

  const int split = blockIdx.x, kvh = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int L = lens[b];
  const int begin = split * chunk;
  const int end = min(L, begin + chunk);
  const int n_heads = n_kv * G;

  for (int i = threadIdx.x; i < G * HD; i += blockDim.x) {
    int g = i / HD, d = i - g * HD;
    qs[g][d] = q[(long long)b * ldq + (long long)(kvh * G + g) * HD + d] * scale;
  }
  __syncthreads();

  const int slot = req_slot ? req_slot[b] : b;
  const __nv_bfloat16* kcol = kv.pool + (long long)kvh * HD;
  const __nv_bfloat16* vcol = kv.pool + (long long)(n_kv + kvh) * HD;
  const long long rs = kv.row_elems;

  float m[G], l[G], acc[G][PER];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m[g] = -INFINITY; l[g] = 0.f;
#pragma unroll
    for (int e = 0; e < PER; ++e) acc[g][e] = 0.f;
  }

  // Each warp takes 32 positions per step: lane = position for the scores, lane =
  // PER contiguous dims for V. Every K and V load of the step is issued before
  // any is used (16 + 32 independent loads per lane), so a step costs one
  // memory round trip instead of one per position.
  using VT = typename std::conditional<PER == 4, uint2, uint32_t>::type;
  for (int t0 = begin + warp * 32; t0 < end; t0 += 4 * 32) {
    const int p = t0 + lane;
    const bool valid = p < end;
    const int cnt = min(32, end - t0);
    // t0 is a multiple of 32 and pages hold >= 64 positions: the step's 32 rows are
    // consecutive rows of one page
    const long long r0 = kv.row(slot, t0);
    uint4 kk[HD / 8];
    const uint4* krow = reinterpret_cast<const uint4*>(kcol + r0 + (long long)(valid ? lane : 0) * rs);
#pragma unroll
    for (int c = 0; c < HD / 8; ++c) kk[c] = valid ? __ldg(krow + c) : make_uint4(0, 0, 0, 0);
    VT vv[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const VT* vrow = reinterpret_cast<const VT*>(vcol + r0 + (long long)(j < cnt ? j : 0) * rs + lane * PER);
      vv[j] = __ldg(vrow);
    }
    float s[G];
#pragma unroll
    for (int g = 0; g < G; ++g) s[g] = 0.f;
#pragma unroll
    for (int c = 0; c < HD / 8; ++c) {
      const uint4 k4 = kk[c];
      const float k8[8] = {bf16_lo(k4.x), bf16_hi(k4.x), bf16_lo(k4.y), bf16_hi(k4.y),
                           bf16_lo(k4.z), bf16_hi(k4.z), bf16_lo(k4.w), bf16_hi(k4.w)};
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float4* qq = reinterpret_cast<const float4*>(&qs[g][8 * c]);
        const float4 a = qq[0], bb = qq[1];
        s[g] += a.x * k8[0] + a.y * k8[1] + a.z * k8[2] + a.w * k8[3] + bb.x * k8[4] + bb.y * k8[5] +
                bb.z * k8[6] + bb.w * k8[7];
      }
    }
    float pr[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float sv = valid ? s[g] : -INFINITY;
      float mt = warp_max(sv);
      float mn = fmaxf(m[g], mt);
      float corr = (m[g] == -INFINITY) ? 0.f : __expf(m[g] - mn);
      pr[g] = valid ? __expf(sv - mn) : 0.f;
      l[g] = l[g] * corr + warp_sum(pr[g]);
#pragma unroll
      for (int e = 0; e < PER; ++e) acc[g][e] *= corr;
      m[g] = mn;
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      float v4[PER];
      if constexpr (PER == 4) {
        const uint2 w = *reinterpret_cast<const uint2*>(&vv[j]);
        v4[0] = bf16_lo(w.x); v4[1] = bf16_hi(w.x); v4[2] = bf16_lo(w.y); v4[3] = bf16_hi(w.y);
      } else {
        const uint32_t w = *reinterpret_cast<const uint32_t*>(&vv[j]);
        v4[0] = bf16_lo(w); v4[1] = bf16_hi(w);
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float pj = __shfl_sync(0xffffffffu, pr[g], j);   // 0 for j >= cnt (invalid lanes)
#pragma unroll
        for (int e = 0; e < PER; ++e) acc[g][e] = fmaf(pj, v4[e], acc[g][e]);
      }
    }
  }

  // merge the 4 warps
  if (lane == 0) {
#pragma unroll
    for (int g = 0; g < G; ++g) { red_ml[warp][g][0] = m[g]; red_ml[warp][g][1] = l[g]; }
  }
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int e = 0; e < PER; ++e) red_o[warp][g][lane * PER + e] = acc[g][e];
  __syncthreads();
  for (int i = threadIdx.x; i < G * HD; i += blockDim.x) {
    int g = i / HD, d = i - g * HD;
    float M = -INFINITY;
    for (int w = 0; w < 4; ++w) M = fmaxf(M, red_ml[w][g][0]);
    float Ls = 0.f, O = 0.f;
    if (M != -INFINITY) {
      for (int w = 0; w < 4; ++w) {
        float mw = red_ml[w][g][0];
        if (mw == -INFINITY) continue;
        float f = __expf(mw - M);
        Ls += red_ml[w][g][1] * f;
        O += red_o[w][g][d] * f;
      }
    }
    int h = kvh * G + g;
    if (n_splits == 1) {
      out[(long long)b * ldo + (long long)h * HD + d] = Ls > 0.f ? O / Ls : 0.f;
    } else {
      long long slot = ((long long)b * n_heads + h) * n_splits + split;
      ws_o[slot * HD + d] = O;
      if (d == 0) { ws_ml[slot * 2] = M; ws_ml[slot * 2 + 1] = Ls; }
    }
  }
}

template <int HD>
__global__ void attn_decode_merge_kernel(const float* __restrict__ ws_o, const float* __restrict__ ws_ml,
                                         int n_heads, int n_splits, float* __restrict__ out, int ldo) {
  pdl_trigger();
  pdl_wait();
  int b = blockIdx.y, h = blockIdx.x, d = threadIdx.x;
  long long base = ((long long)b * n_heads + h) * n_splits;
  float M = -INFINITY;
  for (int s = 0; s < n_splits; ++s) M = fmaxf(M, ws_ml[(base + s) * 2]);
  float Ls = 0.f, O = 0.f;
  if (M != -INFINITY) {
    for (int s = 0; s < n_splits; ++s) {
      float ms = ws_ml[(base + s) * 2];
      if (ms == -INFINITY) continue;
      float f = __expf(ms - M);
      Ls += ws_ml[(base + s) * 2 + 1] * f;
      O += ws_o[(base + s) * HD + d] * f;
    }
  }
  out[(long long)b * ldo + (long long)h * HD + d] = Ls > 0.f ? O / Ls : 0.f;
}

// ------------------------------- prefill ------------------------------------
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
}

constexpr int PF_BQ = 64, PF_BK = 64;

template <int HD>
__global__ void __launch_bounds__(128)
attn_prefill_kernel(const float* __restrict__ q, int ldq, const int* __restrict__ q_start,
                    const int* __restrict__ p0s, KvPages kv, const int* __restrict__ req_slot, int n_heads,
                    int n_kv, float scale_log2, void* __restrict__ out,
                    int ldo, int out_bf16) {
  constexpr int LDS = HD + 8;  // padded smem row (bf16)
  constexpr int KSTEPS = HD / 16;
  constexpr int NT_O = HD / 8;
  __shared__ __align__(16) __nv_bfloat16 Ks[PF_BK][LDS];
  __shared__ __align__(16) __nv_bfloat16 Vs[PF_BK][LDS];

  const int b = blockIdx.z, h = blockIdx.y, qt = blockIdx.x;
  const int qs0 = q_start[b], n_new = q_start[b + 1] - qs0;
  if (qt * PF_BQ >= n_new) return;
  const int p0 = p0s[b];
  const int G = n_heads / n_kv;
  const int kvh = h / G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r_lo = qt * PF_BQ + warp * 16 + (lane >> 2);  // query index (within sequence) of row A
  const int r_hi = r_lo + 8;
  const int qpos_lo = p0 + r_lo, qpos_hi = p0 + r_hi;

  // Q fragments (bf16, pre-scaled by softmax scale * log2 e)
  uint32_t qf[KSTEPS][4];
  {
    const float* qa = q + (long long)(qs0 + min(r_lo, n_new - 1)) * ldq + (long long)h * HD;
    const float* qb = q + (long long)(qs0 + min(r_hi, n_new - 1)) * ldq + (long long)h * HD;
    bool va = r_lo < n_new, vb = r_hi < n_new;
#pragma unroll
    for (int kk = 0; kk < KSTEPS; ++kk) {
      int c = kk * 16 + (lane & 3) * 2;
      float2 a0 = va ? *reinterpret_cast<const float2*>(qa + c) : make_float2(0.f, 0.f);
      float2 a1 = vb ? *reinterpret_cast<const float2*>(qb + c) : make_float2(0.f, 0.f);
      float2 a2 = va ? *reinterpret_cast<const float2*>(qa + c + 8) : make_float2(0.f, 0.f);
      float2 a3 = vb ? *reinterpret_cast<const float2*>(qb + c + 8) : make_float2(0.f, 0.f);
      qf[kk][0] = pack_bf16(a0.x * scale_log2, a0.y * scale_log2);
      qf[kk][1] = pack_bf16(a1.x * scale_log2, a1.y * scale_log2);
      qf[kk][2] = pack_bf16(a2.x * scale_log2, a2.y * scale_log2);
      qf[kk][3] = pack_bf16(a3.x * scale_log2, a3.y * scale_log2);
    }
  }

  float o[NT_O][4];
#pragma unroll
  for (int j = 0; j < NT_O; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m_lo = -INFINITY, m_hi = -INFINITY, l_lo = 0.f, l_hi = 0.f;

  const int last_q = min(qt * PF_BQ + PF_BQ, n_new) - 1;
  const int kv_end = p0 + last_q + 1;  // keys [0, kv_end)
  const int slot = req_slot ? req_slot[b] : b;

  for (int k0 = 0; k0 < kv_end; k0 += PF_BK) {
    __syncthreads();
    // stage K and V tiles (16-byte chunks)
    constexpr int CH = HD / 8;
    for (int i = threadIdx.x; i < PF_BK * CH; i += blockDim.x) {
      int r = i / CH, c = i - r * CH;
      int kp = k0 + r;
      uint4 kv4 = make_uint4(0, 0, 0, 0), vv4 = make_uint4(0, 0, 0, 0);
      if (kp < kv_end) {
        const __nv_bfloat16* row = kv.pool + kv.row(slot, kp);
        kv4 = *reinterpret_cast<const uint4*>(row + (long long)kvh * HD + c * 8);
        vv4 = *reinterpret_cast<const uint4*>(row + (long long)(n_kv + kvh) * HD + c * 8);
      }
      *reinterpret_cast<uint4*>(&Ks[r][c * 8]) = kv4;
      *reinterpret_cast<uint4*>(&Vs[r][c * 8]) = vv4;
    }
    __syncthreads();

    // S = Q K^T for this warp's 16 rows x 64 keys
    float s[PF_BK / 8][4];
#pragma unroll
    for (int j = 0; j < PF_BK / 8; ++j) {
      s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
      const __nv_bfloat16* krow = &Ks[j * 8 + (lane >> 2)][(lane & 3) * 2];
#pragma unroll
      for (int kk = 0; kk < KSTEPS; ++kk) {
        uint32_t b0 = *reinterpret_cast<const uint32_t*>(krow + kk * 16);
        uint32_t b1 = *reinterpret_cast<const uint32_t*>(krow + kk * 16 + 8);
        mma_bf16_16816(s[j], qf[kk], b0, b1);
      }
    }
    // causal / bounds mask and online softmax (base-2)
    float mx_lo = -INFINITY, mx_hi = -INFINITY;
#pragma unroll
    for (int j = 0; j < PF_BK / 8; ++j) {
      int kp = k0 + j * 8 + (lane & 3) * 2;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (kp + e > qpos_lo || kp + e >= kv_end) s[j][e] = -INFINITY;
        if (kp + e > qpos_hi || kp + e >= kv_end) s[j][2 + e] = -INFINITY;
        mx_lo = fmaxf(mx_lo, s[j][e]);
        mx_hi = fmaxf(mx_hi, s[j][2 + e]);
      }
    }
    mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, 1));
    mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, 2));
    mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, 1));
    mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, 2));
    float mn_lo = fmaxf(m_lo, mx_lo), mn_hi = fmaxf(m_hi, mx_hi);
    float base_lo = mn_lo == -INFINITY ? 0.f : mn_lo;
    float base_hi = mn_hi == -INFINITY ? 0.f : mn_hi;
    float c_lo = exp2f(m_lo - base_lo), c_hi = exp2f(m_hi - base_hi);
    m_lo = mn_lo; m_hi = mn_hi;
    l_lo *= c_lo; l_hi *= c_hi;
#pragma unroll
    for (int j = 0; j < NT_O; ++j) { o[j][0] *= c_lo; o[j][1] *= c_lo; o[j][2] *= c_hi; o[j][3] *= c_hi; }
    uint32_t pf[PF_BK / 16][4];
#pragma unroll
    for (int j = 0; j < PF_BK / 8; ++j) {
      float p0v = exp2f(s[j][0] - base_lo), p1v = exp2f(s[j][1] - base_lo);
      float p2v = exp2f(s[j][2] - base_hi), p3v = exp2f(s[j][3] - base_hi);
      l_lo += p0v + p1v; l_hi += p2v + p3v;
      int kk = j >> 1;
      if ((j & 1) == 0) { pf[kk][0] = pack_bf16(p0v, p1v); pf[kk][1] = pack_bf16(p2v, p3v); }
      else { pf[kk][2] = pack_bf16(p0v, p1v); pf[kk][3] = pack_bf16(p2v, p3v); }
    }
    // O += P V
#pragma unroll
    for (int kk = 0; kk < PF_BK / 16; ++kk) {
#pragma unroll
      for (int n = 0; n < NT_O; n += 2) {
        uint32_t r[4];
        int mat = lane >> 3, rr = lane & 7;
        const __nv_bfloat16* p = &Vs[kk * 16 + (mat & 1) * 8 + rr][n * 8 + (mat >> 1) * 8];
        ldmatrix_x4_trans(r, p);
        mma_bf16_16816(o[n], pf[kk], r[0], r[1]);
        mma_bf16_16816(o[n + 1], pf[kk], r[2], r[3]);
      }
    }
  }

  l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 1);
  l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 2);
  l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 1);
  l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 2);
  float inv_lo = l_lo > 0.f ? 1.f / l_lo : 0.f, inv_hi = l_hi > 0.f ? 1.f / l_hi : 0.f;
#pragma unroll
  for (int j = 0; j < NT_O; ++j) {
    int col = h * HD + j * 8 + (lane & 3) * 2;
    if (r_lo < n_new) {
      long long off = (long long)(qs0 + r_lo) * ldo + col;
      if (out_bf16) *reinterpret_cast<uint32_t*>(static_cast<__nv_bfloat16*>(out) + off) = pack_bf16(o[j][0] * inv_lo, o[j][1] * inv_lo);
      else *reinterpret_cast<float2*>(static_cast<float*>(out) + off) = make_float2(o[j][0] * inv_lo, o[j][1] * inv_lo);
    }
    if (r_hi < n_new) {
      long long off = (long long)(qs0 + r_hi) * ldo + col;
      if (out_bf16) *reinterpret_cast<uint32_t*>(static_cast<__nv_bfloat16*>(out) + off) = pack_bf16(o[j][2] * inv_hi, o[j][3] * inv_hi);
      else *reinterpret_cast<float2*>(static_cast<float*>(out) + off) = make_float2(o[j][2] * inv_hi, o[j][3] * inv_hi);
    }
  }
}

}  // namespace ps

using namespace ps;

template <int HD>
static int decode_dispatch(int G, dim3 grid, cudaStream_t s, const float* q, int ldq, const KvPages& kv,
                           const int* req_slot, const int* lens, int n_kv, int chunk, float scale, float* out, int ldo,
                           float* ws_o, float* ws_ml, int n_splits) {
#define PS_DEC(GG)                                                                                       \
  launch_k(attn_decode_kernel<HD, GG>, grid, 128, 0, s, q, ldq, kv, req_slot, lens, n_kv, chunk, scale, out, ldo, \
           ws_o, ws_ml, n_splits)
  switch (G) {
    case 1: PS_DEC(1); break;
    case 2: PS_DEC(2); break;
    case 4: PS_DEC(4); break;
    case 8: PS_DEC(8); break;
    default: ps_set_error("ps_attn_decode: group size %d unsupported", G); return PS_ERR_UNSUPPORTED;
  }
#undef PS_DEC
  PS_CHECK_LAUNCH();
  return PS_OK;
}

extern "C" int ps_attn_decode_workspace(int batch, int n_heads, int head_dim, int max_len, long long* floats) {
  PS_REQUIRE(floats != nullptr, "ps_attn_decode_workspace: floats is null");
  int n_splits = (max_len + PS_DECODE_CHUNK - 1) / PS_DECODE_CHUNK;
  if (n_splits < 1) n_splits = 1;
  *floats = n_splits > 1 ? (long long)batch * n_heads * n_splits * (head_dim + 2) : 0;
  return PS_OK;
}

extern "C" int ps_attn_decode(const float* q, int ldq, int batch, int n_heads, int n_kv, int head_dim,
                              const int* req_slot, const void* kv_pool, int row_elems, const int* block_table,
                              int bt_stride, int page_rows, const int* lens, int max_len,
                              float scale, float* out, int ldo, float* workspace, long long workspace_floats,
                              void* stream) {
  PS_REQUIRE(n_heads % n_kv == 0, "ps_attn_decode: n_heads %% n_kv != 0");
  if (batch <= 0) return PS_OK;
  KvPages kv;
  PS_REQUIRE(kv_pages(kv, kv_pool, row_elems, block_table, bt_stride, page_rows) && row_elems == 2 * n_kv * head_dim,
             "ps_attn_decode: bad paged cache (page_rows %d, bt_stride %d, row_elems %d)", page_rows, bt_stride,
             row_elems);
  int G = n_heads / n_kv;
  int chunk = PS_DECODE_CHUNK;
  int n_splits = (max_len + chunk - 1) / chunk;
  if (n_splits < 1) n_splits = 1;
  long long need = (long long)batch * n_heads * n_splits * (head_dim + 2);
  if (n_splits > 1) PS_REQUIRE(workspace && workspace_floats >= need, "ps_attn_decode: workspace too small (%lld floats needed)", need);
  float* ws_o = workspace;
  float* ws_ml = workspace ? workspace + (long long)batch * n_heads * n_splits * head_dim : nullptr;
  dim3 grid(n_splits, n_kv, batch);
  cudaStream_t s = (cudaStream_t)stream;
  int rc;
  if (head_dim == 128) rc = decode_dispatch<128>(G, grid, s, q, ldq, kv, req_slot, lens, n_kv, chunk, scale, out, ldo, ws_o, ws_ml, n_splits);
  else if (head_dim == 64) rc = decode_dispatch<64>(G, grid, s, q, ldq, kv, req_slot, lens, n_kv, chunk, scale, out, ldo, ws_o, ws_ml, n_splits);
  else { ps_set_error("ps_attn_decode: head_dim %d unsupported", head_dim); return PS_ERR_UNSUPPORTED; }
  if (rc || n_splits == 1) return rc;
  if (head_dim == 128)
    launch_k(attn_decode_merge_kernel<128>, dim3(n_heads, batch), 128, 0, s, ws_o, ws_ml, n_heads, n_splits, out, ldo);
  else
    launch_k(attn_decode_merge_kernel<64>, dim3(n_heads, batch), 64, 0, s, ws_o, ws_ml, n_heads, n_splits, out, ldo);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

extern "C" int ps_attn_prefill(const float* q, int ldq, int batch, const int* q_start, const int* p0,
                               const int* req_slot, int max_new, int n_heads, int n_kv, int head_dim,
                               const void* kv_pool, int row_elems, const int* block_table, int bt_stride,
                               int page_rows, float scale, void* out, int ldo, int out_bf16, void* stream) {
  PS_REQUIRE(n_heads % n_kv == 0, "ps_attn_prefill: n_heads %% n_kv != 0");
  if (batch <= 0 || max_new <= 0) return PS_OK;
  KvPages kv;
  PS_REQUIRE(kv_pages(kv, kv_pool, row_elems, block_table, bt_stride, page_rows) && row_elems == 2 * n_kv * head_dim,
             "ps_attn_prefill: bad paged cache (page_rows %d, bt_stride %d, row_elems %d)", page_rows, bt_stride,
             row_elems);
  dim3 grid((max_new + PF_BQ - 1) / PF_BQ, n_heads, batch);
  float sl2 = scale * 1.4426950408889634f;
  cudaStream_t s = (cudaStream_t)stream;
  if (head_dim == 128)
    attn_prefill_kernel<128><<<grid, 128, 0, s>>>(q, ldq, q_start, p0, kv, req_slot, n_heads, n_kv, sl2, out, ldo, out_bf16);
  else if (head_dim == 64)
    attn_prefill_kernel<64><<<grid, 128, 0, s>>>(q, ldq, q_start, p0, kv, req_slot, n_heads, n_kv, sl2, out, ldo, out_bf16);
  else { ps_set_error("ps_attn_prefill: head_dim %d unsupported", head_dim); return PS_ERR_UNSUPPORTED; }
  PS_CHECK_LAUNCH();
  return PS_OK;
}

int ps_preload_attention() {
  int n = 0;
#define PS_G(HD) \
  touch_kernel(attn_decode_kernel<HD, 1>, n); touch_kernel(attn_decode_kernel<HD, 2>, n); \
  touch_kernel(attn_decode_kernel<HD, 4>, n); touch_kernel(attn_decode_kernel<HD, 8>, n); \
  touch_kernel(attn_decode_merge_kernel<HD>, n); touch_kernel(attn_prefill_kernel<HD>, n);
  PS_G(64) PS_G(128)
#undef PS_G
  return n;
}
