// K3: tcgen05 / TMEM / TMA GEMM for prefill and batched projections.
//
// Prices: MATMUL requests with t >= 64 new tokens
// (`pkg/src/shardplan/model_graph.py:147-153,173-179`).
// C[M x N] (op)= A[M x K] * B[N x K]^T; A = activations (bf16, row-major),
// B = weights (bf16, row-major [N x K]) — both K-major, the native UMMA
// operand layout. fp32 accumulation in TMEM.
//
// Two kernels, one epilogue:
//
// * gemm_2cta (M > 128, the prefill shapes): a persistent CTA-pair kernel.
//   A cluster of 2 CTAs on one TPC owns 256 x 256 output tiles and walks
//   them in grouped-raster order (74 pairs on 148 SMs). Each CTA TMA-loads
//   its 128-row half of A and its 128-row half of B into a 6-stage ring
//   (32 KB / stage, 128-byte swizzle); both halves signal the leader's
//   mbarrier. The leader's elected lane issues tcgen05.mma.cta_group::2
//   (M = 256, N = 256, K = 16), so each SM streams half the B tile it
//   would need alone. The fp32 accumulator is double-buffered in TMEM
//   (2 x 256 columns = all 512): the epilogue warps of both CTAs drain tile
//   i (tcgen05.ld -> fused epilogue -> global) while the MMA runs tile i+1.
// * gemm_1cta (M <= 128): one 128 x 256 tile per CTA, 4-stage ring.
//
// Warp roles (256 threads): warp 0 TMA producer, warp 1 MMA issuer
// (leader CTA), warp 2 TMEM allocator, warps 4..7 epilogue (TMEM lane
// quarter = warp % 4).
// Epilogues: fp32 store / fp32 accumulate (fused residual add) / bf16 store /
// SwiGLU on interleaved gate-up columns -> bf16.
#include <cuda.h>

#include "common.cuh"
#include "mbarrier.cuh"
#include "../../include/pshard.h"

namespace ps {

constexpr int GBK = 64;                                  // K per stage (128 B of bf16 = one swizzle row)
// 1-CTA kernel
constexpr int GBM = 128, GBN = 256, GSTAGES = 4;
constexpr int A_STAGE_BYTES = GBM * GBK * 2;            // 16 KB
constexpr int B_STAGE_BYTES = GBN * GBK * 2;            // 32 KB
constexpr int STAGE_BYTES = A_STAGE_BYTES + B_STAGE_BYTES;
constexpr int GEMM_SMEM = GSTAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr int TMEM_COLS = 256;
// 2-CTA persistent kernel: pair tile 256 x 256, per-CTA halves 128 x 64 of A and of B
constexpr int PBM = 256, PBN = 256, PSTAGES = 6, PGROUP_M = 16;
constexpr int P_HALF_BYTES = 128 * GBK * 2;             // 16 KB
constexpr int P_STAGE_BYTES = 2 * P_HALF_BYTES;         // A half + B half = 32 KB per CTA
constexpr int P_SMEM = PSTAGES * P_STAGE_BYTES + 1024 + 256;
constexpr int P_TMEM_COLS = 512;                        // two 256-column fp32 accumulators

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// CTA-pair TMA: data lands in this CTA's smem, the byte count is credited to the
// mbarrier at `cluster_bar` (the leader CTA's).
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t cluster_bar, int c0,
                                                 int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(cluster_bar), "r"(c0), "r"(c1)
      : "memory");
}

// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t umma_desc_sw128(const void* smem) {
  uint64_t addr = smem_u32(smem);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;          // start address
  d |= 1ull << 16;                        // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;       // SBO
  d |= 1ull << 46;                        // descriptor version (sm100)
  d |= 2ull << 61;                        // SWIZZLE_128B
  return d;
}

// Instruction descriptor: BF16 x BF16 -> F32, both K-major.
constexpr uint32_t make_idesc(int m, int n) {
  return (1u << 4)                      // D = f32
       | (1u << 7)                      // A = bf16
       | (1u << 10)                     // B = bf16
       | ((uint32_t)(n >> 3) << 17)
       | ((uint32_t)(m >> 4) << 24);
}
constexpr uint32_t IDESC = make_idesc(GBM, GBN);
constexpr uint32_t IDESC_PAIR = make_idesc(PBM, PBN);

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(IDESC), "r"(accumulate));
}

__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(IDESC_PAIR), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// Arrive on the barrier at the same smem offset in both CTAs of the pair once
// every previously issued tcgen05.mma of this thread has completed.
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\t"
      "mov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}"
      ::"r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 p = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&p);
}

// One thread's 32 accumulator columns [col, col + 32) of output row `row`.
template <int EPI>
__device__ __forceinline__ void epilogue_store(const uint32_t (&v)[32], int row, int col, int M, int N, void* C,
                                               int ldc) {
  if (row >= M || col >= N) return;
  const int ncols = N - col < 32 ? N - col : 32;
  if (EPI == PS_EPI_STORE || EPI == PS_EPI_ACCUM) {
    float* dst = static_cast<float*>(C) + (long long)row * ldc + col;
    if (ncols == 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        float4 o = make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]), __uint_as_float(v[i + 2]),
                               __uint_as_float(v[i + 3]));
        if (EPI == PS_EPI_ACCUM) {
          float4 p = *reinterpret_cast<float4*>(dst + i);
          o.x += p.x; o.y += p.y; o.z += p.z; o.w += p.w;
        }
        *reinterpret_cast<float4*>(dst + i) = o;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        if (i < ncols) {
          float o = __uint_as_float(v[i]);
          if (EPI == PS_EPI_ACCUM) o += dst[i];
          dst[i] = o;
        }
      }
    }
  } else if (EPI == PS_EPI_STORE_BF16) {
    __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(C) + (long long)row * ldc + col;
    if (ncols == 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
      for (int i = 0; i < 32; i += 8) {
        uint4 o;
        o.x = pack_bf16(__uint_as_float(v[i]), __uint_as_float(v[i + 1]));
        o.y = pack_bf16(__uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
        o.z = pack_bf16(__uint_as_float(v[i + 4]), __uint_as_float(v[i + 5]));
        o.w = pack_bf16(__uint_as_float(v[i + 6]), __uint_as_float(v[i + 7]));
        *reinterpret_cast<uint4*>(dst + i) = o;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i < ncols) dst[i] = __float2bfloat16_rn(__uint_as_float(v[i]));
    }
  } else {  // PS_EPI_SWIGLU: columns (2j, 2j+1) = (gate_j, up_j) -> out[j] (bf16)
    __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(C) + (long long)row * ldc + col / 2;
    if (ncols == 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
      for (int i = 0; i < 16; i += 8) {
        float h[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) h[j] = silu(__uint_as_float(v[2 * (i + j)])) * __uint_as_float(v[2 * (i + j) + 1]);
        uint4 o;
        o.x = pack_bf16(h[0], h[1]);
        o.y = pack_bf16(h[2], h[3]);
        o.z = pack_bf16(h[4], h[5]);
        o.w = pack_bf16(h[6], h[7]);
        *reinterpret_cast<uint4*>(dst + i) = o;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (2 * i + 1 < ncols)
          dst[i] = __float2bfloat16_rn(silu(__uint_as_float(v[2 * i])) * __uint_as_float(v[2 * i + 1]));
    }
  }
}

// ------------------------------------------------------------------------------------------
// 1-CTA kernel: one 128 x 256 tile per CTA.
template <int EPI>
__global__ void __launch_bounds__(256, 1)
gemm_bf16_tcgen05_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                         int M, int N, int K, void* __restrict__ C, int ldc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + GSTAGES * STAGE_BYTES);
  uint64_t* empty = full + GSTAGES;
  uint64_t* tmem_full = empty + GSTAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * GBN;
  const int m0 = blockIdx.y * GBM;
  const int num_kb = K / GBK;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < GSTAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < num_kb; ++kb) {
        int s = kb % GSTAGES;
        uint32_t ph = (kb / GSTAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* sa = smem + s * STAGE_BYTES;
        uint8_t* sb = sa + A_STAGE_BYTES;
        mbar_expect_tx(&full[s], STAGE_BYTES);
        tma_load_2d(sa, &map_a, &full[s], kb * GBK, m0);
        tma_load_2d(sb, &map_b, &full[s], kb * GBK, n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      for (int kb = 0; kb < num_kb; ++kb) {
        int s = kb % GSTAGES;
        uint32_t ph = (kb / GSTAGES) & 1;
        mbar_wait(&full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint8_t* sa = smem + s * STAGE_BYTES;
        const uint8_t* sb = sa + A_STAGE_BYTES;
        uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sb);
#pragma unroll
        for (int k = 0; k < GBK / 16; ++k) {
          // advance the start address by 16 bf16 = 32 bytes (>> 4 = 2) inside the swizzle atom
          umma_bf16(tmem_base, da + 2 * k, db + 2 * k, (kb | k) != 0);
        }
        umma_commit(&empty[s]);
      }
      umma_commit(tmem_full);
    }
  } else if (warp >= 4) {
    mbar_wait(tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int q = warp - 4;  // TMEM lane quarter
    const int row = m0 + q * 32 + lane;
    const uint32_t t_row = tmem_base + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
    for (int c = 0; c < GBN; c += 32) {
      uint32_t v[32];
      tmem_ld32(t_row + c, v);
      epilogue_store<EPI>(v, row, n0 + c, M, N, C, ldc);
    }
  }

  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                 : "memory");
  }
}

// ------------------------------------------------------------------------------------------
// 2-CTA persistent kernel.
__device__ __forceinline__ void pair_tile_coords(int t, int num_m, int num_n, int& tm, int& tn) {
  // grouped raster: PGROUP_M pair-rows of A stay hot in L2 while every B column tile passes
  const int per_group = PGROUP_M * num_n;
  const int g = t / per_group;
  const int first_m = g * PGROUP_M;
  const int gm = min(PGROUP_M, num_m - first_m);
  const int r = t - g * per_group;
  tm = first_m + r % gm;
  tn = r / gm;
}

template <int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
gemm_bf16_pair_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                      int M, int N, int K, void* __restrict__ C, int ldc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + PSTAGES * P_STAGE_BYTES);
  uint64_t* empty = full + PSTAGES;
  uint64_t* tmem_full = empty + PSTAGES;       // [2]
  uint64_t* tmem_empty = tmem_full + 2;        // [2] (leader's are the live ones)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int num_m = (M + PBM - 1) / PBM;
  const int num_n = (N + PBN - 1) / PBN;
  const int num_tiles = num_m * num_n;
  const int pair = blockIdx.x >> 1;
  const int num_pairs = gridDim.x >> 1;
  const int num_kb = K / GBK;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < PSTAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tmem_full[a], 1); mbar_init(&tmem_empty[a], 8); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(P_TMEM_COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t leader_full0 = cluster_addr(&full[0], 0);
      int it = 0;  // global k-block counter (ring position)
      for (int t = pair; t < num_tiles; t += num_pairs) {
        int tm, tn;
        pair_tile_coords(t, num_m, num_n, tm, tn);
        const int arow = tm * PBM + (int)rank * 128;
        const int brow = tn * PBN + (int)rank * 128;
        for (int kb = 0; kb < num_kb; ++kb, ++it) {
          const int s = it % PSTAGES;
          const uint32_t ph = (it / PSTAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* sa = smem + s * P_STAGE_BYTES;
          uint8_t* sb = sa + P_HALF_BYTES;
          if (rank == 0) mbar_expect_tx(&full[s], 2 * P_STAGE_BYTES);  // both CTAs' halves
          const uint32_t fb = leader_full0 + s * 8;
          tma_load_2d_pair(sa, &map_a, fb, kb * GBK, arow);
          tma_load_2d_pair(sb, &map_b, fb, kb * GBK, brow);
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && lane == 0) {
      int it = 0, local = 0;
      for (int t = pair; t < num_tiles; t += num_pairs, ++local) {
        const int acc = local & 1;
        const uint32_t acc_ph = (local >> 1) & 1;
        mbar_wait(&tmem_empty[acc], acc_ph ^ 1);  // both CTAs' epilogues drained this accumulator
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem_base + (uint32_t)(acc * PBN);
        for (int kb = 0; kb < num_kb; ++kb, ++it) {
          const int s = it % PSTAGES;
          const uint32_t ph = (it / PSTAGES) & 1;
          mbar_wait(&full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint8_t* sa = smem + s * P_STAGE_BYTES;
          uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sa + P_HALF_BYTES);
#pragma unroll
          for (int k = 0; k < GBK / 16; ++k) umma_bf16_pair(d, da + 2 * k, db + 2 * k, (kb | k) != 0);
          umma_commit_pair(&empty[s]);        // frees the stage in both CTAs
        }
        umma_commit_pair(&tmem_full[acc]);    // accumulator ready in both CTAs
      }
    }
  } else if (warp >= 4) {
    const int q = warp - 4;  // TMEM lane quarter
    const uint32_t leader_empty0 = cluster_addr(&tmem_empty[0], 0);
    int local = 0;
    for (int t = pair; t < num_tiles; t += num_pairs, ++local) {
      int tm, tn;
      pair_tile_coords(t, num_m, num_n, tm, tn);
      const int acc = local & 1;
      const uint32_t acc_ph = (local >> 1) & 1;
      mbar_wait(&tmem_full[acc], acc_ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int row = tm * PBM + (int)rank * 128 + q * 32 + lane;
      const uint32_t t_row = tmem_base + (uint32_t)(acc * PBN) + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int c = 0; c < PBN; c += 32) {
        uint32_t v[32];
        tmem_ld32(t_row + c, v);
        epilogue_store<EPI>(v, row, tn * PBN + c, M, N, C, ldc);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_empty0 + acc * 8);
    }
  }

  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(P_TMEM_COLS)
                 : "memory");
  }
}

// ---- host side: TMA descriptors through the driver entry point (no -lcuda) ----
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

static int make_map(CUtensorMap* map, const void* base, int rows, int cols, long long ld, int box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) {
    ps_set_error("cuTensorMapEncodeTiled unavailable");
    return PS_ERR_CUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)GBK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    ps_set_error("cuTensorMapEncodeTiled failed (%d) rows=%d cols=%d ld=%lld", (int)r, rows, cols, ld);
    return PS_ERR_CUDA;
  }
  return PS_OK;
}

static int g_gemm_sms = 0;

template <int EPI>
static int launch_gemm(const void* A, int M, int K, long long lda, const void* B, int N, long long ldb, void* C,
                       int ldc, cudaStream_t s, int variant) {
  CUtensorMap ma, mb;
  const bool pair = variant == 2 || (variant == 0 && M > GBM);
  int rc = make_map(&ma, A, M, K, lda, pair ? 128 : GBM);
  if (rc) return rc;
  rc = make_map(&mb, B, N, K, ldb, pair ? 128 : GBN);
  if (rc) return rc;
  if (pair) {
    static bool attr = false;
    if (!attr) {
      PS_CHECK_CUDA(cudaFuncSetAttribute(gemm_bf16_pair_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         P_SMEM));
      attr = true;
    }
    if (!g_gemm_sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&g_gemm_sms, cudaDevAttrMultiProcessorCount, dev);
      if (g_gemm_sms < 2) g_gemm_sms = 148;
    }
    const int tiles = ((M + PBM - 1) / PBM) * ((N + PBN - 1) / PBN);
    const int pairs = tiles < g_gemm_sms / 2 ? tiles : g_gemm_sms / 2;
    gemm_bf16_pair_kernel<EPI><<<2 * pairs, 256, P_SMEM, s>>>(ma, mb, M, N, K, C, ldc);
  } else {
    static bool attr = false;
    if (!attr) {
      PS_CHECK_CUDA(cudaFuncSetAttribute(gemm_bf16_tcgen05_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         GEMM_SMEM));
      attr = true;
    }
    dim3 grid((N + GBN - 1) / GBN, (M + GBM - 1) / GBM);
    gemm_bf16_tcgen05_kernel<EPI><<<grid, 256, GEMM_SMEM, s>>>(ma, mb, M, N, K, C, ldc);
  }
  PS_CHECK_LAUNCH();
  return PS_OK;
}

static int gemm_checked(const void* A, int M, int K, long long lda, const void* B, int N, long long ldb, void* C,
                        int ldc, int epilogue, void* stream, int variant) {
  PS_REQUIRE(K % GBK == 0 && K > 0, "ps_gemm_bf16: K=%d must be a positive multiple of %d", K, GBK);
  PS_REQUIRE(lda % 8 == 0 && ldb % 8 == 0, "ps_gemm_bf16: lda/ldb must be multiples of 8 elements");
  PS_REQUIRE(((uintptr_t)A & 15) == 0 && ((uintptr_t)B & 15) == 0, "ps_gemm_bf16: A/B must be 16-byte aligned");
  PS_REQUIRE(epilogue != PS_EPI_SWIGLU || N % 2 == 0, "ps_gemm_bf16: SWIGLU needs an even N");
  PS_REQUIRE(variant >= 0 && variant <= 2, "ps_gemm_bf16: variant %d not in {0, 1, 2}", variant);
  if (M <= 0 || N <= 0) return PS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  switch (epilogue) {
    case PS_EPI_STORE: return launch_gemm<PS_EPI_STORE>(A, M, K, lda, B, N, ldb, C, ldc, s, variant);
    case PS_EPI_ACCUM: return launch_gemm<PS_EPI_ACCUM>(A, M, K, lda, B, N, ldb, C, ldc, s, variant);
    case PS_EPI_STORE_BF16: return launch_gemm<PS_EPI_STORE_BF16>(A, M, K, lda, B, N, ldb, C, ldc, s, variant);
    case PS_EPI_SWIGLU: return launch_gemm<PS_EPI_SWIGLU>(A, M, K, lda, B, N, ldb, C, ldc, s, variant);
    default: ps_set_error("ps_gemm_bf16: unsupported epilogue %d", epilogue); return PS_ERR_ARG;
  }
}

}  // namespace ps

extern "C" int ps_gemm_bf16(const void* A, int M, int K, long long lda, const void* B, int N, long long ldb,
                            void* C, int ldc, int epilogue, void* stream) {
  return ps::gemm_checked(A, M, K, lda, B, N, ldb, C, ldc, epilogue, stream, 0);
}

extern "C" int ps_gemm_bf16_cfg(const void* A, int M, int K, long long lda, const void* B, int N, long long ldb,
                                void* C, int ldc, int epilogue, void* stream, int variant) {
  return ps::gemm_checked(A, M, K, lda, B, N, ldb, C, ldc, epilogue, stream, variant);
}

int ps_preload_gemm() {
  using namespace ps;
  int n = 0;
  touch_kernel(gemm_bf16_tcgen05_kernel<PS_EPI_STORE>, n);
  touch_kernel(gemm_bf16_tcgen05_kernel<PS_EPI_ACCUM>, n);
  touch_kernel(gemm_bf16_tcgen05_kernel<PS_EPI_STORE_BF16>, n);
  touch_kernel(gemm_bf16_tcgen05_kernel<PS_EPI_SWIGLU>, n);
  touch_kernel(gemm_bf16_pair_kernel<PS_EPI_STORE>, n);
  touch_kernel(gemm_bf16_pair_kernel<PS_EPI_ACCUM>, n);
  touch_kernel(gemm_bf16_pair_kernel<PS_EPI_STORE_BF16>, n);
  touch_kernel(gemm_bf16_pair_kernel<PS_EPI_SWIGLU>, n);
  return n;
}
