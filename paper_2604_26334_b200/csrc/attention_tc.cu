// K4 prefill on the 5th-generation tensor cores: causal varlen flash attention
// with tcgen05.mma, TMEM accumulators and TMA-fed K/V tiles.
//
// Prices the GQA/MHA requests of a prefill pass (`pkg/src/shardplan/model_graph.py:154-161`,
// flops 4*t*ctx*h*hd, causal half executed). Replaces the mma.sync (HMMA) kernel of
// attention.cu on sm_100a.
//
// One CTA = one (request, query head, block of 128 queries); 6 warps:
//   warps 0-3  softmax: thread i owns query row i (= TMEM lane i). Loads its Q row
//              (fp32 -> scaled bf16) into smem once; per key block reads its S row
//              from TMEM (tcgen05.ld), masks (causal / length), runs the base-2
//              online softmax, rescales its O row in TMEM when the max moves
//              (tcgen05.ld/st), writes its P row (bf16) to smem; epilogue O / l.
//   warp 4     TMA producer: K and V tiles of 128 positions x 64 dims straight from the
//              paged KV cache: one 3-D tensor map over the page pool [pool rows][K heads |
//              V heads][hd], a 128-key tile = two 64-row boxes, each at the row its page's
//              block-table entry names (keys past the request's end: an out-of-range box,
//              zero-filled by TMA); 2-stage ring, 128-byte swizzle.
//   warp 5     MMA issuer (one lane): S = Q K^T (M=128, N=128 keys, K=hd; both K-major)
//              into TMEM columns [0,128); O += P V (M=128, N=hd, K=128 keys; A=P
//              K-major, B=V MN-major) into columns [128, 128+hd).
// Barriers: k/v full (TMA -> MMA), kv empty (MMA -> TMA), s full (MMA -> softmax),
// p full (softmax -> MMA), o done (MMA -> softmax).
#include <cuda.h>
#include <float.h>
#include <stdlib.h>

#include "common.cuh"
#include "mbarrier.cuh"
#include "../../include/pshard.h"

namespace ps {

constexpr int TC_BQ = 128, TC_BK = 128;

// Watchdog for the pipeline barriers: a wait that spins for more than 1 s records
// where it was stuck (role, barrier, block) and lets the kernel finish (wrong
// output, never a hung GPU) and raises FAULT_ATTN in the host-mapped fault words
// (common.cuh), which the executor checks after every pass. Read with
// ps_attn_tc_watchdog() / ps_fault_status().
__device__ unsigned g_attn_tc_stuck = 0;
__device__ unsigned* g_attn_tc_fault = nullptr;

__device__ __forceinline__ void wait_wd(uint64_t* bar, uint32_t parity, unsigned code) {
  uint32_t done = 0;
  unsigned long long t0 = 0;
  for (int it = 0;; ++it) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    if (done) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (it == 0) t0 = t;
    else if (t - t0 > 1000000000ull) {
      atomicCAS(&g_attn_tc_stuck, 0u, code);
      if (g_attn_tc_fault) raise_fault(g_attn_tc_fault, FAULT_ATTN, code);
      return;
    }
  }
}
constexpr int TC_SUB = 128 * 64 * 2;   // one [128 rows x 64 cols] bf16 swizzled sub-tile = 16 KB

__device__ __forceinline__ uint64_t desc_k_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= 1ull << 16;                        // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;       // SBO: 8-row groups
  d |= 1ull << 46;                        // sm100 descriptor version
  d |= 2ull << 61;                        // 128B swizzle
  return d;
}

// MN-major, 128B swizzle: 64 MN-elements x 8 K-rows per 1 KB atom; next 8 K-rows at
// SBO, next 64 MN-elements at LBO.
__device__ __forceinline__ uint64_t desc_mn_sw128(uint32_t saddr, uint32_t lbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= 1ull << 46;
  d |= 2ull << 61;
  return d;
}

constexpr uint32_t idesc_f16(int m, int n, bool b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (b_mn_major ? (1u << 16) : 0u) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void commit_to(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tm_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tm_st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
      "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])),
      "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])),
      "r"(__float_as_uint(v[17])), "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])),
      "r"(__float_as_uint(v[20])), "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])),
      "r"(__float_as_uint(v[23])), "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])),
      "r"(__float_as_uint(v[26])), "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])),
      "r"(__float_as_uint(v[29])), "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// 2^x on the SFU (ex2.approx: ~2 ulp, exact 0 for -inf); P is rounded to bf16 anyway
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t pack2_bf16(float a, float b) {
  __nv_bfloat162 p = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&p);
}

// Write row `r` (64 bf16 = 8 x 16-byte chunks, values v[0..63]) of a 128B-swizzled
// [128 x 64] sub-tile: chunk c lands at chunk c ^ (r % 8).
__device__ __forceinline__ void st_row_sw128(uint8_t* sub, int r, const float* v) {
  uint8_t* row = sub + r * 128;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    uint4 o;
    o.x = pack2_bf16(v[8 * c + 0], v[8 * c + 1]);
    o.y = pack2_bf16(v[8 * c + 2], v[8 * c + 3]);
    o.z = pack2_bf16(v[8 * c + 4], v[8 * c + 5]);
    o.w = pack2_bf16(v[8 * c + 6], v[8 * c + 7]);
    *reinterpret_cast<uint4*>(row + ((c ^ (r & 7)) << 4)) = o;
  }
}

template <int HD>
__global__ void __launch_bounds__(192, 1)
attn_prefill_tc_kernel(const __grid_constant__ CUtensorMap kv_map, const float* __restrict__ q, int ldq,
                       const int* __restrict__ q_start, const int* __restrict__ p0s, const int* __restrict__ req_slot,
                       const int* __restrict__ table, int bt_stride, int page_shift, int pool_rows,
                       int n_heads, int n_kv, float scale_log2, void* __restrict__ out, int ldo, int out_bf16,
                       int dbg) {
  constexpr int DH = HD / 64;                 // 64-wide dim sub-tiles
  constexpr int TILE = DH * TC_SUB;           // Q, K or V tile bytes
  constexpr uint32_t IDS = idesc_f16(TC_BQ, TC_BK, false);
  constexpr uint32_t IDO = idesc_f16(TC_BQ, HD, true);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm;
  uint8_t* sK = sQ + TILE;             // [2][TILE]
  uint8_t* sV = sK + 2 * TILE;         // [2][TILE]
  uint8_t* sP = sV + 2 * TILE;         // [2 key halves][TC_SUB]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + 2 * TC_SUB);
  uint64_t* k_full = bars;             // [2]
  uint64_t* v_full = bars + 2;         // [2]
  uint64_t* kv_empty = bars + 4;       // [2]
  uint64_t* s_full = bars + 6;
  uint64_t* p_full = bars + 7;
  uint64_t* o_done = bars + 8;
  uint64_t* q_ready = bars + 9;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);

  const int b = blockIdx.z, h = blockIdx.y, qt = blockIdx.x;
  const int qs0 = q_start[b], n_new = q_start[b + 1] - qs0;
  if (qt * TC_BQ >= n_new) return;     // whole CTA, before any barrier
  const int p0 = p0s[b];
  const int kvh = h / (n_heads / n_kv);
  const int slot = req_slot ? req_slot[b] : b;
  const int last_q = min(qt * TC_BQ + TC_BQ, n_new) - 1;
  const int kv_end = p0 + last_q + 1;                    // keys [0, kv_end)
  const int nkb = (kv_end + TC_BK - 1) / TC_BK;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 160) {
    for (int s = 0; s < 2; ++s) { mbar_init(&k_full[s], 1); mbar_init(&v_full[s], 1); mbar_init(&kv_empty[s], 1); }
    mbar_init(s_full, 1);
    mbar_init(p_full, 128);
    mbar_init(o_done, 1);
    mbar_init(q_ready, 128);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tO = tmem + 128;

  if (warp == 4) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&kv_map)) : "memory");
      const int* bt = table + (long long)slot * bt_stride;
      const int pmask = (1 << page_shift) - 1;
      for (int j = 0; j < nkb; ++j) {
        const int s = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        int rows[2];                       // pool row of each 64-key half (pool_rows: past the end)
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          const int key = j * TC_BK + hf * 64;
          rows[hf] = key < kv_end ? (__ldg(bt + (key >> page_shift)) << page_shift) + (key & pmask) : pool_rows;
        }
        wait_wd(&kv_empty[s], ph ^ 1, 0x01010000u | (j & 0xffff));
        mbar_expect_tx(&k_full[s], TILE);
#pragma unroll
        for (int dh = 0; dh < DH; ++dh)
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            if (dbg & 8) asm volatile("mbarrier.complete_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&k_full[s])), "r"(TC_SUB / 2) : "memory");
            else tma_load_3d(sK + s * TILE + dh * TC_SUB + hf * (TC_SUB / 2), &kv_map, &k_full[s], dh * 64, kvh, rows[hf]);
          }
        mbar_expect_tx(&v_full[s], TILE);
#pragma unroll
        for (int dh = 0; dh < DH; ++dh)
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            if (dbg & 8) asm volatile("mbarrier.complete_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&v_full[s])), "r"(TC_SUB / 2) : "memory");
            else tma_load_3d(sV + s * TILE + dh * TC_SUB + hf * (TC_SUB / 2), &kv_map, &v_full[s], dh * 64, n_kv + kvh,
                             rows[hf]);
          }
      }
    }
  } else if (warp == 5) {
    // ---------------- MMA issuer (lane 0; the warp zeroes stale V rows) ----------------
    if (lane == 0) {
      wait_wd(q_ready, 0, 0x02010000u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    const uint32_t aQ = smem_u32(sQ), aP = smem_u32(sP);
    for (int j = 0; j < nkb; ++j) {
      const int s = j & 1;
      const uint32_t ph = (j >> 1) & 1;
      if (lane == 0) {
        wait_wd(&k_full[s], ph, 0x02020000u | (j & 0xffff));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t aK = smem_u32(sK + s * TILE);
        if (!(dbg & 1)) {
#pragma unroll
          for (int k = 0; k < HD / 16; ++k) {
            const uint32_t off = (k >> 2) * TC_SUB + (k & 3) * 32;
            mma_f16(tS, desc_k_sw128(aQ + off), desc_k_sw128(aK + off), IDS, k > 0);
          }
        }
        commit_to(s_full);
        wait_wd(p_full, j & 1, 0x02030000u | (j & 0xffff));
        wait_wd(&v_full[s], ph, 0x02040000u | (j & 0xffff));
      }
      __syncwarp();
      const int valid = kv_end - j * TC_BK;     // keys of this block that exist
      if (valid < TC_BK) {
        // rows past the request's end inside its last page hold stale bytes (maybe NaN):
        // P is 0 there but 0 * NaN is not, so zero them before O += P V. A 128-B row of a
        // 128B-swizzled sub-tile stays in its own 128-B line, whatever the swizzle.
        for (int i = lane; i < (TC_BK - valid) * DH * 8; i += 32) {
          const int r = valid + i / (DH * 8), c = i % (DH * 8);
          *reinterpret_cast<uint4*>(sV + s * TILE + (c >> 3) * TC_SUB + r * 128 + (c & 7) * 16) =
              make_uint4(0, 0, 0, 0);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
      }
      if (lane == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t aV = smem_u32(sV + s * TILE);
        if (!(dbg & 2)) {
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k) {
            const uint32_t offp = (k >> 2) * TC_SUB + (k & 3) * 32;  // P: K-major, 64-key halves
            const uint32_t offv = k * 16 * 128;                      // V: 16 key rows of 128 B
            mma_f16(tO, desc_k_sw128(aP + offp), desc_mn_sw128(aV + offv, TC_SUB), IDO, (j > 0 || k > 0));
          }
        }
        commit_to(&kv_empty[s]);
        commit_to(o_done);
      }
      __syncwarp();
    }
  } else {
    // ---------------- softmax warps: thread i owns query row i ----------------
    const int i = threadIdx.x;
    const int qi = qt * TC_BQ + i;
    const bool valid = qi < n_new;
    const int qpos = p0 + qi;
    {
      float v[64];
      const float* qrow = q + (long long)(qs0 + (valid ? qi : 0)) * ldq + (long long)h * HD;
#pragma unroll
      for (int dh = 0; dh < DH; ++dh) {
#pragma unroll
        for (int c = 0; c < 64; c += 4) {
          float4 a = valid ? *reinterpret_cast<const float4*>(qrow + dh * 64 + c) : make_float4(0.f, 0.f, 0.f, 0.f);
          v[c] = a.x * scale_log2; v[c + 1] = a.y * scale_log2; v[c + 2] = a.z * scale_log2; v[c + 3] = a.w * scale_log2;
        }
        st_row_sw128(sQ + dh * TC_SUB, i, v);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(q_ready);
    }
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < nkb; ++j) {
      wait_wd(s_full, j & 1, 0x03010000u | (j & 0xffff));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      float sv[TC_BK];
#pragma unroll
      for (int c = 0; c < TC_BK; c += 32) {
        float t[32];
        tm_ld32(tS + lane_base + c, t);
#pragma unroll
        for (int e = 0; e < 32; ++e) sv[c + e] = t[e];
      }
      const int k0 = j * TC_BK;
      // the causal / length mask only touches blocks that reach past this row's position
      if (k0 + TC_BK - 1 > qpos || k0 + TC_BK > kv_end) {
#pragma unroll
        for (int c = 0; c < TC_BK; ++c)
          if (k0 + c > qpos || k0 + c >= kv_end) sv[c] = -INFINITY;
      }
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int c = 0; c < TC_BK; c += 2) { mx0 = fmaxf(mx0, sv[c]); mx1 = fmaxf(mx1, sv[c + 1]); }
      const float m_new = fmaxf(m, fmaxf(mx0, mx1));
      const float base = m_new == -INFINITY ? 0.f : m_new;
      const float corr = fast_exp2(m - base);      // 0 when m = -inf (first block)
      float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
      for (int c = 0; c < TC_BK; c += 2) {
        sv[c] = fast_exp2(sv[c] - base);
        sv[c + 1] = fast_exp2(sv[c + 1] - base);
        rs0 += sv[c];
        rs1 += sv[c + 1];
      }
      const float rs = rs0 + rs1;
      l = l * corr + rs;
      if (j > 0) {
        wait_wd(o_done, (j - 1) & 1, 0x03020000u | (j & 0xffff));   // O(j-1) complete, P buffer free
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // tcgen05.ld/st are warp-collective: rescale when any row of the warp moved
        if (__any_sync(0xffffffffu, corr != 1.f) && !(dbg & 4)) {
#pragma unroll 1
          for (int c = 0; c < HD; c += 32) {
            float t[32];
            tm_ld32(tO + lane_base + c, t);
#pragma unroll
            for (int e = 0; e < 32; ++e) t[e] *= corr;
            tm_st32(tO + lane_base + c, t);
          }
        }
      }
      st_row_sw128(sP, i, sv);
      st_row_sw128(sP + TC_SUB, i, sv + 64);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(p_full);
      m = m_new;
    }
    wait_wd(o_done, (nkb - 1) & 1, 0x03030000u);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll 1
    for (int c = 0; c < HD; c += 32) {
      float t[32];
      tm_ld32(tO + lane_base + c, t);
      if (valid) {
        const long long off = (long long)(qs0 + qi) * ldo + (long long)h * HD + c;
        if (out_bf16) {
          __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(out) + off;
#pragma unroll
          for (int e = 0; e < 32; e += 8) {
            uint4 o;
            o.x = pack2_bf16(t[e] * inv, t[e + 1] * inv);
            o.y = pack2_bf16(t[e + 2] * inv, t[e + 3] * inv);
            o.z = pack2_bf16(t[e + 4] * inv, t[e + 5] * inv);
            o.w = pack2_bf16(t[e + 6] * inv, t[e + 7] * inv);
            *reinterpret_cast<uint4*>(dst + e) = o;
          }
        } else {
          float* dst = static_cast<float*>(out) + off;
#pragma unroll
          for (int e = 0; e < 32; e += 4)
            *reinterpret_cast<float4*>(dst + e) = make_float4(t[e] * inv, t[e + 1] * inv, t[e + 2] * inv, t[e + 3] * inv);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 4) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
  }
}

typedef CUresult (*EncodeTiledFn4)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int HD>
static int launch_tc(const CUtensorMap& map, const float* q, int ldq, int batch, const int* q_start, const int* p0,
                     const int* req_slot, const int* table, int bt_stride, int page_shift, int pool_rows, int max_new,
                     int n_heads, int n_kv, float scale_log2, void* out, int ldo, int out_bf16, cudaStream_t s) {
  constexpr int TILE = (HD / 64) * TC_SUB;
  constexpr int SMEM = 5 * TILE + 2 * TC_SUB + 1024 + 128;
  static bool attr = false;
  if (!attr) {
    PS_CHECK_CUDA(cudaFuncSetAttribute(attn_prefill_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
    attr = true;
  }
  dim3 grid((max_new + TC_BQ - 1) / TC_BQ, n_heads, batch);
  static int dbg = -1;
  if (dbg < 0) {
    const char* e = getenv("PS_ATTN_TC_DBG");
    dbg = e ? atoi(e) : 0;
  }
  attn_prefill_tc_kernel<HD><<<grid, 192, SMEM, s>>>(map, q, ldq, q_start, p0, req_slot, table, bt_stride, page_shift,
                                                     pool_rows, n_heads, n_kv, scale_log2, out, ldo, out_bf16, dbg);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

}  // namespace ps

int ps_preload_attention_tc() {
  using namespace ps;
  int n = 0;
  touch_kernel(attn_prefill_tc_kernel<64>, n);
  touch_kernel(attn_prefill_tc_kernel<128>, n);
  unsigned* f = fault_dev();
  if (cudaMemcpyToSymbol(g_attn_tc_fault, &f, sizeof(f)) != cudaSuccess) cudaGetLastError();
  return n;
}

extern "C" int ps_attn_tc_watchdog(unsigned* code, int reset) {
  PS_CHECK_CUDA(cudaMemcpyFromSymbol(code, ps::g_attn_tc_stuck, sizeof(unsigned)));
  if (reset) {
    unsigned z = 0;
    PS_CHECK_CUDA(cudaMemcpyToSymbol(ps::g_attn_tc_stuck, &z, sizeof(unsigned)));
  }
  return PS_OK;
}

extern "C" int ps_attn_prefill_tc(const float* q, int ldq, int batch, const int* q_start, const int* p0,
                                  const int* req_slot, int max_new, int n_heads, int n_kv, int head_dim,
                                  const void* kv_pool, int row_elems, const int* block_table, int bt_stride,
                                  int page_rows, int pool_pages, float scale, void* out, int ldo, int out_bf16,
                                  void* stream) {
  using namespace ps;
  PS_REQUIRE(head_dim == 64 || head_dim == 128, "ps_attn_prefill_tc: head_dim %d unsupported", head_dim);
  PS_REQUIRE(n_heads % n_kv == 0, "ps_attn_prefill_tc: n_heads %% n_kv != 0");
  KvPages kv;
  PS_REQUIRE(kv_pages(kv, kv_pool, row_elems, block_table, bt_stride, page_rows) && row_elems == 2 * n_kv * head_dim,
             "ps_attn_prefill_tc: bad paged cache (page_rows %d, bt_stride %d, row_elems %d)", page_rows, bt_stride,
             row_elems);
  PS_REQUIRE(pool_pages >= 1, "ps_attn_prefill_tc: pool_pages %d", pool_pages);
  PS_REQUIRE(((uintptr_t)kv_pool & 15) == 0 && ldq % 4 == 0, "ps_attn_prefill_tc: alignment");
  if (batch <= 0 || max_new <= 0) return PS_OK;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  PS_CHECK_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr));
  PS_REQUIRE(fn && qr == cudaDriverEntryPointSuccess, "cuTensorMapEncodeTiled unavailable");
  const long long pool_rows = (long long)pool_pages * page_rows;
  PS_REQUIRE(pool_rows < (1LL << 31), "ps_attn_prefill_tc: pool of %lld rows", pool_rows);
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)head_dim, (cuuint64_t)(2 * n_kv), (cuuint64_t)pool_rows};
  cuuint64_t strides[2] = {(cuuint64_t)head_dim * 2, (cuuint64_t)row_elems * 2};
  cuuint32_t box[3] = {64, 1, 64};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = reinterpret_cast<EncodeTiledFn4>(fn)(
      &map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(kv_pool), dims, strides, box, estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  PS_REQUIRE(r == CUDA_SUCCESS, "ps_attn_prefill_tc: cuTensorMapEncodeTiled failed (%d)", (int)r);
  const float sl2 = scale * 1.4426950408889634f;
  cudaStream_t s = (cudaStream_t)stream;
  if (head_dim == 128)
    return launch_tc<128>(map, q, ldq, batch, q_start, p0, req_slot, block_table, bt_stride, kv.page_shift,
                          (int)pool_rows, max_new, n_heads, n_kv, sl2, out, ldo, out_bf16, s);
  return launch_tc<64>(map, q, ldq, batch, q_start, p0, req_slot, block_table, bt_stride, kv.page_shift,
                       (int)pool_rows, max_new, n_heads, n_kv, sl2, out, ldo, out_bf16, s);
}
