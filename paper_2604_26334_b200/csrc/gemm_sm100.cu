// K3: tcgen05 / TMEM / TMA GEMM for prefill and batched projections.
//
// Prices: MATMUL requests with t >= 64 new tokens
// (`pkg/src/shardplan/model_graph.py:147-153,173-179`).
// C[M x N] (op)= A[M x K] * B[N x K]^T; A = activations (bf16, row-major),
// B = weights (bf16, row-major [N x K]) — both K-major, the native UMMA
// operand layout. fp32 accumulation in TMEM.
//
// Structure (one 128 x 256 output tile per CTA, 8 warps):
//   warp 0      TMA producer: 4-stage ring of {A 128x64, B 256x64} tiles,
//               128-byte swizzle, mbarrier full/empty pipeline
//   warp 1      MMA issuer: one elected lane issues tcgen05.mma
//               (kind::f16, M=128, N=256, K=16) into a 256-column TMEM
//               accumulator; tcgen05.commit releases smem stages
//   warp 2      TMEM allocator
//   warps 4..7  epilogue: tcgen05.ld 32x32b.x32 -> registers -> fused
//               epilogue (fp32 store / fp32 accumulate / bf16 store /
//               SwiGLU on interleaved gate-up rows -> bf16) -> global
#include <cuda.h>

#include "common.cuh"
#include "../../include/pshard.h"

namespace ps {

constexpr int GBM = 128, GBN = 256, GBK = 64, GSTAGES = 4;
constexpr int A_STAGE_BYTES = GBM * GBK * 2;            // 16 KB
constexpr int B_STAGE_BYTES = GBN * GBK * 2;            // 32 KB
constexpr int STAGE_BYTES = A_STAGE_BYTES + B_STAGE_BYTES;
constexpr int GEMM_SMEM = GSTAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr int TMEM_COLS = 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
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

// Instruction descriptor: BF16 x BF16 -> F32, both K-major, M = 128, N = 256.
constexpr uint32_t IDESC = (1u << 4)            // D = f32
                         | (1u << 7)            // A = bf16
                         | (1u << 10)           // B = bf16
                         | ((uint32_t)(GBN >> 3) << 17)
                         | ((uint32_t)(GBM >> 4) << 24);

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(IDESC), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
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
      if (row >= M || n0 + c >= N) continue;
      int ncols = N - (n0 + c) < 32 ? N - (n0 + c) : 32;
      if (EPI == PS_EPI_STORE || EPI == PS_EPI_ACCUM) {
        float* dst = static_cast<float*>(C) + (long long)row * ldc + n0 + c;
        if (ncols == 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            float4 o = make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]),
                                   __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
            if (EPI == PS_EPI_ACCUM) {
              float4 p = *reinterpret_cast<float4*>(dst + i);
              o.x += p.x; o.y += p.y; o.z += p.z; o.w += p.w;
            }
            *reinterpret_cast<float4*>(dst + i) = o;
          }
        } else {
          for (int i = 0; i < ncols; ++i) {
            float o = __uint_as_float(v[i]);
            if (EPI == PS_EPI_ACCUM) o += dst[i];
            dst[i] = o;
          }
        }
      } else if (EPI == PS_EPI_STORE_BF16) {
        __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(C) + (long long)row * ldc + n0 + c;
        if (ncols == 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            uint4 o;
            __nv_bfloat162 p0 = __floats2bfloat162_rn(__uint_as_float(v[i]), __uint_as_float(v[i + 1]));
            __nv_bfloat162 p1 = __floats2bfloat162_rn(__uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
            __nv_bfloat162 p2 = __floats2bfloat162_rn(__uint_as_float(v[i + 4]), __uint_as_float(v[i + 5]));
            __nv_bfloat162 p3 = __floats2bfloat162_rn(__uint_as_float(v[i + 6]), __uint_as_float(v[i + 7]));
            o.x = *reinterpret_cast<uint32_t*>(&p0); o.y = *reinterpret_cast<uint32_t*>(&p1);
            o.z = *reinterpret_cast<uint32_t*>(&p2); o.w = *reinterpret_cast<uint32_t*>(&p3);
            *reinterpret_cast<uint4*>(dst + i) = o;
          }
        } else {
          for (int i = 0; i < ncols; ++i) dst[i] = __float2bfloat16_rn(__uint_as_float(v[i]));
        }
      } else {  // PS_EPI_SWIGLU: columns (2j, 2j+1) = (gate_j, up_j) -> out[j] (bf16)
        __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(C) + (long long)row * ldc + (n0 + c) / 2;
        if (ncols == 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
          for (int i = 0; i < 16; i += 8) {
            float h[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
              h[j] = silu(__uint_as_float(v[2 * (i + j)])) * __uint_as_float(v[2 * (i + j) + 1]);
            uint4 o;
            __nv_bfloat162 p0 = __floats2bfloat162_rn(h[0], h[1]);
            __nv_bfloat162 p1 = __floats2bfloat162_rn(h[2], h[3]);
            __nv_bfloat162 p2 = __floats2bfloat162_rn(h[4], h[5]);
            __nv_bfloat162 p3 = __floats2bfloat162_rn(h[6], h[7]);
            o.x = *reinterpret_cast<uint32_t*>(&p0); o.y = *reinterpret_cast<uint32_t*>(&p1);
            o.z = *reinterpret_cast<uint32_t*>(&p2); o.w = *reinterpret_cast<uint32_t*>(&p3);
            *reinterpret_cast<uint4*>(dst + i) = o;
          }
        } else {
          for (int i = 0; 2 * i + 1 < ncols; ++i)
            dst[i] = __float2bfloat16_rn(silu(__uint_as_float(v[2 * i])) * __uint_as_float(v[2 * i + 1]));
        }
      }
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

template <int EPI>
static int launch_gemm(const CUtensorMap& ma, const CUtensorMap& mb, int M, int N, int K, void* C, int ldc,
                       cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    PS_CHECK_CUDA(cudaFuncSetAttribute(gemm_bf16_tcgen05_kernel<EPI>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM));
    attr_set = true;
  }
  dim3 grid((N + GBN - 1) / GBN, (M + GBM - 1) / GBM);
  gemm_bf16_tcgen05_kernel<EPI><<<grid, 256, GEMM_SMEM, s>>>(ma, mb, M, N, K, C, ldc);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

}  // namespace ps

extern "C" int ps_gemm_bf16(const void* A, int M, int K, long long lda, const void* B, int N, long long ldb,
                            void* C, int ldc, int epilogue, void* stream) {
  using namespace ps;
  PS_REQUIRE(K % GBK == 0, "ps_gemm_bf16: K=%d must be a multiple of %d", K, GBK);
  PS_REQUIRE(lda % 8 == 0 && ldb % 8 == 0, "ps_gemm_bf16: lda/ldb must be multiples of 8 elements");
  PS_REQUIRE(((uintptr_t)A & 15) == 0 && ((uintptr_t)B & 15) == 0, "ps_gemm_bf16: A/B must be 16-byte aligned");
  PS_REQUIRE(epilogue != PS_EPI_SWIGLU || N % 2 == 0, "ps_gemm_bf16: SWIGLU needs an even N");
  if (M <= 0 || N <= 0) return PS_OK;
  CUtensorMap ma, mb;
  int rc = make_map(&ma, A, M, K, lda, GBM);
  if (rc) return rc;
  rc = make_map(&mb, B, N, K, ldb, GBN);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  switch (epilogue) {
    case PS_EPI_STORE: return launch_gemm<PS_EPI_STORE>(ma, mb, M, N, K, C, ldc, s);
    case PS_EPI_ACCUM: return launch_gemm<PS_EPI_ACCUM>(ma, mb, M, N, K, C, ldc, s);
    case PS_EPI_STORE_BF16: return launch_gemm<PS_EPI_STORE_BF16>(ma, mb, M, N, K, C, ldc, s);
    case PS_EPI_SWIGLU: return launch_gemm<PS_EPI_SWIGLU>(ma, mb, M, N, K, C, ldc, s);
    default: ps_set_error("ps_gemm_bf16: unsupported epilogue %d", epilogue); return PS_ERR_ARG;
  }
}
