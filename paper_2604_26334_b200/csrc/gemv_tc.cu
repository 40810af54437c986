// K1 for decode passes of 9..32 tokens on the 5th-generation tensor cores: one pass over
// the weights whatever the batch.
//
// Prices the MATMUL requests of a batched decode pass (`pkg/src/shardplan/model_graph.py:
// 147-153,173-179,202-209`, t = batch): y[t, n] (epi)= x[t, :] . W[n, :], W bf16 [N x K]
// (or exponent-coded rows, runtime/wcomp.py), x / y fp32. The CUDA-core GEMV (gemv_tma.cu)
// keeps x in registers and so takes 8 tokens per launch: at t = 32 it reads W four times.
// Here the weights are the stationary operand:
//
//   D[128 rows x 32 tokens] += W_tile[128 x 64] . X_tile[32 x 64]^T   (tcgen05.mma, M=128 N=32)
//
// with the fp32 activations split into three bf16 planes x = x1 + x2 + x3 (8 + 8 + 8
// mantissa bits; the products with bf16 weights are exact in fp32), three MMAs per K step,
// each plane into its OWN fp32 TMEM tile (the tensor core's accumulator keeps ~fp32 bits
// relative to its own magnitude: added into x1's sum, the 2^-16-sized x3 products would
// be truncated away), summed x1 + (x2 + x3) in the epilogue: the decode numerics stay
// fp32-faithful (bf16 activations would make batched decode tokens chaotic).
//
// CTA = 128 weight rows x one K range (split-K when N / 128 is small: partials reduced in a
// fixed order by a second kernel, deterministic). Warp roles:
//   warp 0       TMA producer: W tile (bf16: one 128B-swizzled box; coded: the rows' sign|
//                mantissa bytes and codes as two plain boxes) + the three x planes
//   warp 1       MMA issuer (one lane), 4 K steps x 3 planes per stage
//   warp 2       TMEM allocator (128 columns: three 32-column plane accumulators)
//   warps 4..11  (coded) decode the staged rows into the swizzled bf16 W tile; warps 4..7
//                drain TMEM in the epilogue (store / residual add / SwiGLU, or partials)
#include <cuda.h>

#include "common.cuh"
#include "mbarrier.cuh"
#include "wcodec.cuh"
#include "../../include/pshard.h"

namespace ps {

constexpr int TG_M = 128, TG_N = 32, TG_K = 64, TG_STAGES = 4;
constexpr int TG_A = TG_M * TG_K * 2;           // 16 KB bf16 W tile (128B swizzle)
constexpr int TG_B = 3 * TG_N * TG_K * 2;       // 12 KB: three x planes
constexpr int TG_CS = TG_M * TG_K;              // 8 KB coded sign|mantissa bytes
constexpr int TG_CN = TG_M * TG_K / 2;          // 4 KB coded exponent codes
constexpr int TG_TRAILER_MAX = 256;
constexpr int TG_THREADS = 384;                 // 12 warps
constexpr int TG_CONV_THREADS = 256;            // warps 4..11

template <bool COMP>
constexpr int tg_stage_bytes() { return TG_A + TG_B + (COMP ? TG_CS + TG_CN : 0); }
template <bool COMP>
constexpr int tg_smem_bytes() {
  return TG_STAGES * tg_stage_bytes<COMP>() + (COMP ? TG_M * TG_TRAILER_MAX : 0) + 1024 + 256;
}

__device__ __forceinline__ void tg_tma_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ uint64_t tg_desc(const void* smem) {   // K-major, 128B swizzle
  uint64_t addr = smem_u32(smem);
  return ((addr >> 4) & 0x3FFFull) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

constexpr uint32_t TG_IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TG_N >> 3) << 17) |
                              ((uint32_t)(TG_M >> 4) << 24);

__device__ __forceinline__ void tg_mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d), "l"(da), "l"(db),
      "r"(TG_IDESC), "r"(acc));
}

__device__ __forceinline__ void tg_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tg_ld32(uint32_t taddr, float (&v)[32]) {
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

// y row `row` for tokens [0, t): the fused epilogue (store / residual add / SwiGLU on
// interleaved gate-up rows — the gate row's thread writes silu(gate) * up).
template <int EPI>
__device__ __forceinline__ void tg_epilogue(const float (&v)[32], int row, int N, int t, float* y, int ldy) {
  if (EPI == PS_EPI_SWIGLU) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float up = __shfl_xor_sync(0xffffffffu, v[i], 1);
      if ((row & 1) == 0 && row + 1 < N && i < t) y[(long long)i * ldy + (row >> 1)] = silu(v[i]) * up;
    }
    return;
  }
  if (row >= N) return;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    if (i < t) {
      float* p = y + (long long)i * ldy + row;
      *p = EPI == PS_EPI_ACCUM ? *p + v[i] : v[i];
    }
  }
}

// Decode this converter thread's quarter row (32 of the stage's 64 columns: 4 groups of
// 8) into the 128B-swizzled bf16 tile: row r's 16-byte chunk c lives at chunk c ^ (r & 7).
__device__ __forceinline__ void tg_convert(const uint8_t* cs, const uint8_t* cn, const uint8_t* trailers, int tb,
                                           uint8_t* a_tile, int conv, int k0) {
  const int r = conv & (TG_M - 1), half = conv >> 7;       // 256 threads: 128 rows x 2 halves
  const uint32_t* trailer = reinterpret_cast<const uint32_t*>(trailers + r * tb);
  const uint32_t base7 = ((trailer[0] & 0xFFu) * 0x10001u) << 7;
#pragma unroll
  for (int gi = 0; gi < 4; ++gi) {
    const int g = (gi + r) & 3;                             // staggered: fewer bank conflicts
    const int col = half * 32 + g * 8;                      // column within the stage
    const uint2 sm = *reinterpret_cast<const uint2*>(cs + r * TG_K + col);
    const uint32_t nb = *reinterpret_cast<const uint32_t*>(cn + r * (TG_K / 2) + col / 2);
    uint4 w = gt_decode8(sm, nb, base7);
    if (gt_escapes(nb)) w = gt_patch_escapes(w, sm, nb, trailer, k0 + col);
    const int chunk = (col >> 3) ^ (r & 7);
    *reinterpret_cast<uint4*>(a_tile + r * 128 + chunk * 16) = w;
  }
}

template <int EPI, bool COMP>
__global__ void __launch_bounds__(TG_THREADS, 1)
gemv_tc_kernel(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_codes,
               const __grid_constant__ CUtensorMap map_trailer, const __grid_constant__ CUtensorMap map_x,
               int N, int K, int t, int tb, int k_per_split, float* __restrict__ y, int ldy,
               float* __restrict__ partial) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int STG = tg_stage_bytes<COMP>();
  uint8_t* trailers = sm + TG_STAGES * STG;
  uint64_t* bars = reinterpret_cast<uint64_t*>(trailers + (COMP ? TG_M * TG_TRAILER_MAX : 0));
  uint64_t* full = bars;                       // [stages] TMA bytes landed
  uint64_t* conv = bars + TG_STAGES;           // [stages] coded rows decoded into the W tile
  uint64_t* empty = bars + 2 * TG_STAGES;      // [stages] MMAs done with the stage
  uint64_t* tr_full = bars + 3 * TG_STAGES;    // trailers landed
  uint64_t* acc_full = tr_full + 1;            // accumulator complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * TG_M;
  const int split = blockIdx.y;
  const int kb0 = split * k_per_split / TG_K;
  const int kb1 = min(K, (split + 1) * k_per_split) / TG_K;
  const int nkb = kb1 - kb0;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_x)) : "memory");
    if (COMP) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_codes)) : "memory");
    else asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_w)) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < TG_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], TG_CONV_THREADS / 32);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tr_full, 1);
    mbar_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      if (COMP) {
        mbar_expect_tx(tr_full, (uint32_t)(TG_M * tb));
        tg_tma_2d(trailers, &map_trailer, tr_full, K * 3 / 2, m0);
      }
      for (int i = 0; i < nkb; ++i) {
        const int s = i % TG_STAGES;
        const uint32_t ph = (i / TG_STAGES) & 1;
        const int k0 = (kb0 + i) * TG_K;
        mbar_wait(&empty[s], ph ^ 1);
        fence_proxy_async_smem();   // consumers' generic reads -> the next bulk copy
        uint8_t* st = sm + s * STG;
        mbar_expect_tx(&full[s], (uint32_t)(TG_B + (COMP ? TG_CS + TG_CN : TG_A)));
        if (COMP) {
          tg_tma_2d(st + TG_A + TG_B, &map_w, &full[s], k0, m0);                     // sign|mantissa bytes
          tg_tma_2d(st + TG_A + TG_B + TG_CS, &map_codes, &full[s], K + k0 / 2, m0); // exponent codes
        } else {
          tg_tma_2d(st, &map_w, &full[s], k0, m0);
        }
#pragma unroll
        for (int p = 0; p < 3; ++p) tg_tma_2d(st + TG_A + p * (TG_B / 3), &map_x, &full[s], k0, p * TG_N);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % TG_STAGES;
        const uint32_t ph = (i / TG_STAGES) & 1;
        mbar_wait(COMP ? &conv[s] : &full[s], ph);
        if (COMP) mbar_wait(&full[s], ph);    // the x planes (already landed: conv waited on full)
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint8_t* st = sm + s * STG;
        const uint64_t da = tg_desc(st);
#pragma unroll
        for (int k = 0; k < TG_K / 16; ++k)
#pragma unroll
          for (int p = 0; p < 3; ++p)
            tg_mma(tmem + p * TG_N, da + 2 * k, tg_desc(st + TG_A + p * (TG_B / 3)) + 2 * k, (i | k) != 0);
        tg_commit(&empty[s]);
      }
      tg_commit(acc_full);
    }
  } else if (warp >= 4) {
    if (COMP) {
      const int c = threadIdx.x - 128;                      // converter 0..255
      mbar_wait(tr_full, 0);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % TG_STAGES;
        const uint32_t ph = (i / TG_STAGES) & 1;
        mbar_wait(&full[s], ph);
        uint8_t* st = sm + s * STG;
        tg_convert(st + TG_A + TG_B, st + TG_A + TG_B + TG_CS, trailers, tb, st, c, (kb0 + i) * TG_K);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> MMA reads
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[s]);
      }
    }
    if (warp < 8) {
      mbar_wait(acc_full, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int q = warp - 4;
      const int row = m0 + q * 32 + lane;
      float v[32], v1[32], v2[32];
      const uint32_t lanes = (uint32_t)(q * 32) << 16;
      tg_ld32(tmem + lanes, v);
      tg_ld32(tmem + lanes + TG_N, v1);
      tg_ld32(tmem + lanes + 2 * TG_N, v2);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] += v1[i] + v2[i];
      if (partial == nullptr) {
        tg_epilogue<EPI>(v, row, N, t, y, ldy);
      } else if (row < N) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (i < t) partial[((long long)split * TG_N + i) * N + row] = v[i];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem) : "memory");
  }
}

// Split-K partials [splits][32][N] -> y, summed in split order (deterministic), fused epilogue.
template <int EPI>
__global__ void gemv_tc_reduce_kernel(const float* __restrict__ partial, int splits, int N, int t, float* y,
                                      int ldy) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  const int tok = blockIdx.y;
  if (EPI == PS_EPI_SWIGLU) {
    const int j = row;                                      // output column = gate/up pair j
    if (2 * j + 1 >= N) return;
    float g = 0.f, u = 0.f;
    for (int s = 0; s < splits; ++s) {
      g += partial[((long long)s * TG_N + tok) * N + 2 * j];
      u += partial[((long long)s * TG_N + tok) * N + 2 * j + 1];
    }
    y[(long long)tok * ldy + j] = silu(g) * u;
    return;
  }
  if (row >= N) return;
  float a = 0.f;
  for (int s = 0; s < splits; ++s) a += partial[((long long)s * TG_N + tok) * N + row];
  float* p = y + (long long)tok * ldy + row;
  *p = EPI == PS_EPI_ACCUM ? *p + a : a;
}

// fp32 x [t x K] -> bf16 planes [3][32][K]: x1 = rn(x), x2 = rn(x - x1), x3 = rn(x - x1 - x2);
// rows t..31 are zero.
__global__ void split_x3_kernel(const float* __restrict__ x, int ldx, int t, int K, __nv_bfloat16* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int tok = blockIdx.y;
  if (k >= K) return;
  const float v = tok < t ? x[(long long)tok * ldx + k] : 0.f;
  const __nv_bfloat16 a = __float2bfloat16_rn(v);
  const float r1 = v - __bfloat162float(a);
  const __nv_bfloat16 b = __float2bfloat16_rn(r1);
  const __nv_bfloat16 c = __float2bfloat16_rn(r1 - __bfloat162float(b));
  out[(0LL * TG_N + tok) * K + k] = a;
  out[(1LL * TG_N + tok) * K + k] = b;
  out[(2LL * TG_N + tok) * K + k] = c;
}

typedef CUresult (*TgEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static TgEncodeFn tg_encode() {
  static TgEncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<TgEncodeFn>(p);
  }
  return fn;
}

static int tg_map(CUtensorMap* m, CUtensorMapDataType dt, int esize, const void* base, long long cols, int rows,
                  long long ld_bytes, int box_cols, int box_rows, CUtensorMapSwizzle sw) {
  TgEncodeFn enc = tg_encode();
  PS_REQUIRE(enc != nullptr, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld_bytes};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  PS_REQUIRE(r == CUDA_SUCCESS, "gemv_tc: cuTensorMapEncodeTiled failed (%d): cols %lld rows %d ld %lld box %dx%d",
             (int)r, cols, rows, ld_bytes, box_cols, box_rows);
  (void)esize;
  return PS_OK;
}

static int g_tg_sms = 0;

static long long tg_planes_bytes(int K) { return ((3LL * TG_N * K * 2 + 255) / 256) * 256; }

// K split so that the grid covers the SMs at least twice over (split-K only when the
// row tiles alone do not), and so that the partials fit `workspace` bytes after the x
// planes (< 0: no limit); every split a multiple of TG_K columns.
static void tg_split(int N, int K, int* splits, int* k_per_split, long long workspace = -1) {
  if (!g_tg_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_tg_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_tg_sms <= 0) g_tg_sms = 148;
  }
  const int tiles = (N + TG_M - 1) / TG_M;
  const int kb = K / TG_K;
  int s = 1;
  while (tiles * s < g_tg_sms && s < 8 && kb / (2 * s) >= 8 &&
         (workspace < 0 || tg_planes_bytes(K) + 2LL * s * TG_N * N * 4 <= workspace))
    s *= 2;
  const int per = (kb + s - 1) / s;
  *splits = (kb + per - 1) / per;
  *k_per_split = per * TG_K;
}

static long long tg_workspace(int N, int K) {
  int splits, kps;
  tg_split(N, K, &splits, &kps);
  const long long part = splits > 1 ? (long long)splits * TG_N * N * 4 : 0;
  return tg_planes_bytes(K) + part;
}

template <int EPI, bool COMP>
static int tg_launch(const CUtensorMap& mw, const CUtensorMap& mc, const CUtensorMap& mt, const CUtensorMap& mx,
                     int N, int K, int t, int tb, float* y, int ldy, float* partial, int splits, int kps,
                     cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    PS_CHECK_CUDA(cudaFuncSetAttribute(gemv_tc_kernel<EPI, COMP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       tg_smem_bytes<COMP>()));
    attr = true;
  }
  dim3 grid((N + TG_M - 1) / TG_M, splits);
  gemv_tc_kernel<EPI, COMP><<<grid, TG_THREADS, tg_smem_bytes<COMP>(), s>>>(
      mw, mc, mt, mx, N, K, t, tb, kps, y, ldy, splits > 1 ? partial : nullptr);
  PS_CHECK_LAUNCH();
  if (splits > 1) {
    const int cols = EPI == PS_EPI_SWIGLU ? N / 2 : N;
    gemv_tc_reduce_kernel<EPI><<<dim3((cols + 255) / 256, t), 256, 0, s>>>(partial, splits, N, t, y, ldy);
    PS_CHECK_LAUNCH();
  }
  return PS_OK;
}

}  // namespace ps

extern "C" int ps_gemv_tc_workspace(int N, int K, long long* bytes) {
  PS_REQUIRE(bytes != nullptr && N > 0 && K > 0, "ps_gemv_tc_workspace: bad arguments");
  *bytes = ps::tg_workspace(N, K);
  return PS_OK;
}

extern "C" int ps_gemv_tc(const float* x, int ldx, int t, const void* W, int N, int K, long long ldw, int coded,
                          float* y, int ldy, int epilogue, void* workspace, long long workspace_bytes, void* stream) {
  using namespace ps;
  PS_REQUIRE(t >= 1 && t <= TG_N, "ps_gemv_tc: t=%d outside [1, 32]", t);
  PS_REQUIRE(K % TG_K == 0 && K > 0, "ps_gemv_tc: K=%d must be a multiple of %d", K, TG_K);
  PS_REQUIRE(epilogue == PS_EPI_STORE || epilogue == PS_EPI_ACCUM || epilogue == PS_EPI_SWIGLU,
             "ps_gemv_tc: unsupported epilogue %d", epilogue);
  PS_REQUIRE(epilogue != PS_EPI_SWIGLU || N % 2 == 0, "ps_gemv_tc: SWIGLU needs an even N");
  PS_REQUIRE(((uintptr_t)W & 15) == 0 && ((uintptr_t)workspace & 255) == 0, "ps_gemv_tc: alignment");
  if (N <= 0) return PS_OK;
  // the workspace must hold the x planes; split-K partials use what is left (fewer splits
  // in a small workspace: same result, fewer CTAs)
  PS_REQUIRE(workspace != nullptr && workspace_bytes >= tg_planes_bytes(K),
             "ps_gemv_tc: workspace %lld < %lld bytes (x planes)", workspace_bytes, tg_planes_bytes(K));
  int splits, kps;
  tg_split(N, K, &splits, &kps, workspace_bytes);
  cudaStream_t s = (cudaStream_t)stream;
  auto planes = static_cast<__nv_bfloat16*>(workspace);
  float* partial = reinterpret_cast<float*>(static_cast<char*>(workspace) + tg_planes_bytes(K));
  split_x3_kernel<<<dim3((K + 255) / 256, TG_N), 256, 0, s>>>(x, ldx, t, K, planes);
  PS_CHECK_LAUNCH();
  CUtensorMap mw, mc, mt, mx;
  int rc = tg_map(&mx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, planes, K, 3 * TG_N, (long long)K * 2, TG_K, TG_N,
                  CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  int tb = 0;
  if (coded) {
    tb = (int)(ldw - (long long)K * 3 / 2);
    PS_REQUIRE(tb >= 16 && tb <= TG_TRAILER_MAX && tb % 16 == 0, "ps_gemv_tc: coded row stride %lld (trailer %d)",
               ldw, tb);
    rc = tg_map(&mw, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, W, ldw, N, ldw, TG_K, TG_M, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (!rc) rc = tg_map(&mc, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, W, ldw, N, ldw, TG_K / 2, TG_M, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (!rc) rc = tg_map(&mt, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, W, ldw, N, ldw, tb, TG_M, CU_TENSOR_MAP_SWIZZLE_NONE);
  } else {
    PS_REQUIRE(ldw % 8 == 0, "ps_gemv_tc: ldw %lld must be a multiple of 8", ldw);
    rc = tg_map(&mw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, W, K, N, ldw * 2, TG_K, TG_M, CU_TENSOR_MAP_SWIZZLE_128B);
    mc = mw;
    mt = mw;
  }
  if (rc) return rc;
#define PS_TG(E)                                                                                           \
  return coded ? tg_launch<E, true>(mw, mc, mt, mx, N, K, t, tb, y, ldy, partial, splits, kps, s)          \
               : tg_launch<E, false>(mw, mc, mt, mx, N, K, t, tb, y, ldy, partial, splits, kps, s)
  if (epilogue == PS_EPI_STORE) PS_TG(PS_EPI_STORE);
  if (epilogue == PS_EPI_ACCUM) PS_TG(PS_EPI_ACCUM);
  PS_TG(PS_EPI_SWIGLU);
#undef PS_TG
}

int ps_preload_gemv_tc() {
  using namespace ps;
  int n = 0;
#define PS_P(E)                                        \
  touch_kernel(gemv_tc_kernel<E, false>, n);           \
  touch_kernel(gemv_tc_kernel<E, true>, n);            \
  touch_kernel(gemv_tc_reduce_kernel<E>, n);
  PS_P(PS_EPI_STORE) PS_P(PS_EPI_ACCUM) PS_P(PS_EPI_SWIGLU)
#undef PS_P
  touch_kernel(split_x3_kernel, n);
  return n;
}
