// K5, one-token decode specialisation: the k routed experts of a layer as k row
// groups of ONE bulk-copy GEMV launch per matrix, with the routing-weighted
// combine fused into the down projection.
//
// Prices the same expert MATMUL (t*k, d, mats*eff) as moe.cu
// (`pkg/src/shardplan/model_graph.py:181-200`) for t = 1, the batch-1 decode of
// BASELINE config 3. The general kernels (moe.cu) need a plan kernel (pairs
// grouped by expert) and a combine kernel, and their register-burst loads are
// latency bound on 8 x 9.4 MB of experts: 19 + 13 us for gate/up + down plus
// 11 + 9 us of plan + combine, all on the dependent chain between "this layer's
// experts landed" and "the next layer's routing is published", during which the
// host link idles (profiles/r01_cupti_cfg3_*). With one token every routed
// expert sees the same single activation row, so no plan is needed:
//
//   gate/up: CTA (j, c), j < k, c < C streams rows [c*R, (c+1)*R) of routed
//   expert ids[j] (slot_of_expert[ids[j]] when the experts were fetched into VRAM
//   slots) — contiguous rows, cp.async.bulk in 4 KB copies into 8 x 24 KB
//   shared-memory slots, slot w consumed by warp w alone (x in registers, packed
//   fp32x2 FMA, 4 rows at a time with interleaved warp reductions); rows are
//   gate/up interleaved, so h[j][r/2] = silu(gate) * up.
//
//   down: CTA c owns rows [c*R, (c+1)*R) of ALL k down matrices (one slot per
//   expert, every copy issued up front); warp w holds h[w] in registers and
//   computes expert w's rows; the CTA then adds sum_j w[j] * out[j][r], j
//   ascending — the order of moe.cu's combine — into y[r]: no partial outputs
//   leave the CTA, no cross-CTA reduction.
//
// Measured (tools/bench_moe_decode.py, Q30 shapes, warm): 11.2 + 8.0 us for the
// 75.5 MB of 8 experts vs 50 us for the general chain; ncu: DRAM read = the
// algorithmic bytes (profiles/r01_ncu_moe_decode_t1.jsonl).
//
// COMP variants (ps_moe_decode_experts_c): the experts arrive exponent-coded
// (runtime/wcomp.py rows: sign|mantissa bytes, 4-bit codes, trailer) — 25 % fewer
// bytes through the fetcher's copy engine — and each 8-column group is decoded in
// the consumer loop (wcodec.cuh) before the same dot product: bit-identical outputs.
#include <stdlib.h>

#include "common.cuh"
#include "mbarrier.cuh"
#include "wcodec.cuh"
#include "../../include/pshard.h"

namespace ps {

constexpr int MD_STAGES = 6;
constexpr int MD_STAGE = 32768;
constexpr int MD_WARPS = 8;
constexpr int MD_THREADS = 32 * (1 + MD_WARPS);
constexpr int MD_MAXRING = 16;   // down kernel: ring slots sized to one expert's row block
constexpr int MD_MAXG = 8;
constexpr int MD_BATCH = 4;    // rows whose dot products / warp reductions interleave    // 8-column groups per lane: K <= 32 * 8 * 8 = 2048

__device__ __forceinline__ float2 md_dot8(uint4 w, const float2* x, float2 s) {
  s = __ffma2_rn(x[0], make_float2(bf16_lo(w.x), bf16_hi(w.x)), s);
  s = __ffma2_rn(x[1], make_float2(bf16_lo(w.y), bf16_hi(w.y)), s);
  s = __ffma2_rn(x[2], make_float2(bf16_lo(w.z), bf16_hi(w.z)), s);
  s = __ffma2_rn(x[3], make_float2(bf16_lo(w.w), bf16_hi(w.w)), s);
  return s;
}

// 8 weights of row `row` at column `col`: bf16 straight from the row, or decoded from
// the coded row (K sign|mantissa bytes, K/2 code bytes, trailer at 1.5 K).
template <bool COMP>
__device__ __forceinline__ uint4 md_load8(const uint8_t* row, int col, int K) {
  if constexpr (COMP) {
    const uint32_t* trailer = reinterpret_cast<const uint32_t*>(row + K * 3 / 2);
    const uint32_t base7 = ((trailer[0] & 0xFFu) * 0x10001u) << 7;
    const uint2 sm = *reinterpret_cast<const uint2*>(row + col);
    const uint32_t nb = *reinterpret_cast<const uint32_t*>(row + K + col / 2);
    uint4 w = gt_decode8(sm, nb, base7);
    if (gt_escapes(nb)) w = gt_patch_escapes(w, sm, nb, trailer, col);
    return w;
  } else {
    return *reinterpret_cast<const uint4*>(row + col * 2);
  }
}

// one stage = `bytes` in bulk copies of <= chunk bytes (all on the stage's barrier)
__device__ __forceinline__ void md_copy(uint8_t* dst, const uint8_t* src, int bytes, int chunk, uint64_t* bar) {
  for (int o = 0; o < bytes; o += chunk) bulk_load(dst + o, src + o, (uint32_t)min(chunk, bytes - o), bar);
}

// gate/up: 8 ring slots of 24 KB, slot w owned by consumer warp w: stage b lands
// in slot b % 8 and warp b % 8 takes its rows MD_BATCH at a time, so 8 stages are
// in the consumers' hands at once (each slot has one consumer, so phases stay
// unambiguous). NG = K / 256 column groups per lane (0: generic).
constexpr int GU_SLOT = MD_STAGES * MD_STAGE / MD_WARPS;
template <int NG, bool COMP>
__global__ void __launch_bounds__(MD_THREADS, 1)
moe_gu_t1_kernel(const float* __restrict__ x, const int* __restrict__ ids, const int* __restrict__ slot_of_expert,
                 const unsigned char* __restrict__ base, long long expert_stride, long long mat_off, int N, int K,
                 float* __restrict__ h, int C, int R, int chunk, int rowb, int rank_lo, int rank_hi) {
  constexpr int G = NG > 0 ? NG : MD_MAXG;
  extern __shared__ __align__(128) uint8_t smem[];
  const int j = blockIdx.x / C, c = blockIdx.x - j * C;
  const int r0 = c * R;
  if (r0 >= N) return;
  if (slot_of_expert) {   // only the routed experts whose slot (rank) is in [rank_lo, rank_hi)
    const int rk = slot_of_expert[ids[j]];
    if (rk < rank_lo || rk >= rank_hi) return;   // whole CTA, before any barrier
  }
  const int nrows = min(N, r0 + R) - r0;
  const int RS = GU_SLOT / rowb;
  const int nst = (nrows + RS - 1) / RS;
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + MD_STAGES * MD_STAGE);
  uint64_t* empty = full + MD_WARPS;
  float* acc = reinterpret_cast<float*>(empty + MD_WARPS);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < MD_WARPS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    if (lane == 0) {
      const int e = ids[j];
      const long long slot = slot_of_expert ? slot_of_expert[e] : e;
      const uint8_t* W = base + slot * expert_stride + mat_off + (long long)r0 * rowb;
      for (int b = 0; b < nst; ++b) {
        const int s = b % MD_WARPS;
        const int nr = min(RS, nrows - b * RS);
        mbar_wait(&empty[s], (uint32_t)(((b / MD_WARPS) & 1) ^ 1));
        fence_proxy_async_smem();   // consumers' generic reads -> the next bulk copy
        mbar_expect_tx(&full[s], (uint32_t)(nr * rowb));
        md_copy(ring + s * GU_SLOT, W + (long long)b * RS * rowb, nr * rowb, chunk, &full[s]);
      }
    }
    return;
  }

  const int cw = warp - 1;
  float2 xr[G][4];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int col = (g * 32 + lane) * 8;
    if (NG > 0 || col < K) {
      const float4* xp = reinterpret_cast<const float4*>(x + col);
      const float4 a = __ldg(xp), b = __ldg(xp + 1);
      xr[g][0] = make_float2(a.x, a.y); xr[g][1] = make_float2(a.z, a.w);
      xr[g][2] = make_float2(b.x, b.y); xr[g][3] = make_float2(b.z, b.w);
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) xr[g][i] = make_float2(0.f, 0.f);
    }
  }
  for (int b = cw; b < nst; b += MD_WARPS) {
    const int s = cw;
    const int nr = min(RS, nrows - b * RS);
    mbar_wait(&full[s], (uint32_t)((b / MD_WARPS) & 1));
    const uint8_t* st = ring + s * GU_SLOT;
    for (int r = 0; r < nr; r += MD_BATCH) {
      float v[MD_BATCH];
#pragma unroll
      for (int q = 0; q < MD_BATCH; ++q) {
        const uint8_t* row = st + min(r + q, nr - 1) * rowb;
        float2 a2 = make_float2(0.f, 0.f);
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int col = (g * 32 + lane) * 8;
          if (NG > 0 || col < K) a2 = md_dot8(md_load8<COMP>(row, col, K), xr[g], a2);
        }
        v[q] = a2.x + a2.y;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int q = 0; q < MD_BATCH; ++q) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
      if (lane == 0) {
#pragma unroll
        for (int q = 0; q < MD_BATCH; ++q)
          if (r + q < nr) acc[b * RS + r + q] = v[q];
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  named_sync(1, MD_WARPS * 32);
  for (int i = threadIdx.x - 32; i < nrows / 2; i += MD_WARPS * 32)
    h[(long long)j * (N / 2) + (r0 >> 1) + i] = silu(acc[2 * i]) * acc[2 * i + 1];
}

// down + combine: CTA c streams rows [c*R, c*R + nrows) of the k down matrices,
// one ring slot per expert (k <= MD_MAXRING: every copy is issued up front).
// Consumer warp w owns experts w, w + 8, ...: it holds h[j] in registers and
// takes that expert's rows MD_BATCH at a time (independent dot products,
// interleaved warp reductions). NG = K / 256 column groups per lane (0: generic).
template <int NG, bool COMP>
__global__ void __launch_bounds__(MD_THREADS, 1)
moe_down_t1_kernel(const float* __restrict__ h, const int* __restrict__ ids, const int* __restrict__ slot_of_expert,
                   const unsigned char* __restrict__ base, long long expert_stride, long long mat_off, int N,
                   int K, int R, const float* __restrict__ w, int k, float* __restrict__ y, int chunk,
                   int slot_bytes, int rowb) {
  constexpr int G = NG > 0 ? NG : MD_MAXG;
  extern __shared__ __align__(128) uint8_t smem[];
  const int r0 = blockIdx.x * R;
  if (r0 >= N) return;
  const int nrows = min(N, r0 + R) - r0;
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + MD_STAGES * MD_STAGE);   // k <= MD_MAXRING
  float* acc = reinterpret_cast<float*>(full + MD_MAXRING);                    // [k][R]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < k; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    // lane j resolves expert j's row block; lane 0 issues every copy
    const uint8_t* mine = nullptr;
    if (lane < k) {
      const int e = ids[lane];
      const long long slot = slot_of_expert ? slot_of_expert[e] : e;
      mine = base + slot * expert_stride + mat_off + (long long)r0 * rowb;
    }
    for (int jj = 0; jj < k; ++jj) {
      const uint8_t* W =
          reinterpret_cast<const uint8_t*>(__shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(mine), jj));
      if (lane == 0) {
        mbar_expect_tx(&full[jj], (uint32_t)(nrows * rowb));
        md_copy(ring + jj * slot_bytes, W, nrows * rowb, chunk, &full[jj]);
      }
    }
    return;
  }

  const int t = threadIdx.x - 32, cw = warp - 1;
  for (int jj = cw; jj < k; jj += MD_WARPS) {
    float2 xr[G][4];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int col = (g * 32 + lane) * 8;
      if (NG > 0 || col < K) {
        const float4* hp = reinterpret_cast<const float4*>(h + (size_t)jj * K + col);
        const float4 a = __ldcg(hp), b = __ldcg(hp + 1);   // written by the gate/up launch
        xr[g][0] = make_float2(a.x, a.y); xr[g][1] = make_float2(a.z, a.w);
        xr[g][2] = make_float2(b.x, b.y); xr[g][3] = make_float2(b.z, b.w);
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) xr[g][i] = make_float2(0.f, 0.f);
      }
    }
    mbar_wait(&full[jj], 0);
    const uint8_t* slot = ring + jj * slot_bytes;
    for (int r = 0; r < nrows; r += MD_BATCH) {
      float v[MD_BATCH];
#pragma unroll
      for (int b = 0; b < MD_BATCH; ++b) {
        const uint8_t* row = slot + min(r + b, nrows - 1) * rowb;
        float2 a2 = make_float2(0.f, 0.f);
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int col = (g * 32 + lane) * 8;
          if (NG > 0 || col < K) a2 = md_dot8(md_load8<COMP>(row, col, K), xr[g], a2);
        }
        v[b] = a2.x + a2.y;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int b = 0; b < MD_BATCH; ++b) v[b] += __shfl_xor_sync(0xffffffffu, v[b], o);
      if (lane == 0) {
#pragma unroll
        for (int b = 0; b < MD_BATCH; ++b)
          if (r + b < nrows) acc[jj * R + r + b] = v[b];
      }
    }
  }
  named_sync(1, MD_WARPS * 32);
  for (int i = t; i < nrows; i += MD_WARPS * 32) {
    float sum = 0.f;
    for (int jj = 0; jj < k; ++jj) sum += w[jj] * acc[jj * R + i];
    y[r0 + i] += sum;
  }
}

static int g_md_sms = 0;
static int g_md_chunk = 0;   // bulk-copy size (PS_MD_CHUNK overrides, tuning)

static size_t md_smem(int R) { return (size_t)MD_STAGES * MD_STAGE + MD_WARPS * 16 + (size_t)R * 4; }

}  // namespace ps

using namespace ps;

template <bool COMP>
static int md_launch(const float* x, const int* ids, int k, const int* slot_of_expert, const void* expert_base,
                     long long expert_stride, long long gu_off, long long down_off, int eff, int d, float* h,
                     const float* w, float* y, cudaStream_t s, int gu_rowb, int down_rowb, int phase = 3,
                     int rank_lo = 0, int rank_hi = 1 << 30) {
  if (!g_md_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_md_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_md_sms <= 0) g_md_sms = 148;
  }
  if (!g_md_chunk) {
    const char* e = getenv("PS_MD_CHUNK");
    g_md_chunk = e ? atoi(e) : 4096;   // 4 KB copies: measured 7 % faster than whole stages
    g_md_chunk = g_md_chunk < 1024 ? 1024 : (g_md_chunk & ~15);
  }
  auto base = static_cast<const unsigned char*>(expert_base);
  // gate/up: k groups x C CTAs; N = 2 * eff interleaved rows, even rows per CTA so
  // gate/up pairs never straddle CTAs
  const int C = g_md_sms / k > 0 ? g_md_sms / k : 1;
  const int Rg = 2 * ((eff + C - 1) / C);
  const size_t sg = md_smem(Rg);
  using GuKernel = void (*)(const float*, const int*, const int*, const unsigned char*, long long, long long, int, int,
                           float*, int, int, int, int, int, int);
  const int ngu = d % 256 ? 0 : d / 256;
  GuKernel gk = moe_gu_t1_kernel<0, COMP>;
  switch (ngu) {
    case 1: gk = moe_gu_t1_kernel<1, COMP>; break;
    case 2: gk = moe_gu_t1_kernel<2, COMP>; break;
    case 4: gk = moe_gu_t1_kernel<4, COMP>; break;
    case 8: gk = moe_gu_t1_kernel<8, COMP>; break;
    default: gk = moe_gu_t1_kernel<0, COMP>; break;
  }
  static size_t set_gu[MD_MAXG + 1] = {};
  if (sg > set_gu[ngu]) {
    PS_CHECK_CUDA(cudaFuncSetAttribute(gk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sg));
    set_gu[ngu] = sg;
  }
  PS_REQUIRE(GU_SLOT / gu_rowb >= 1, "ps_moe_decode_experts: gate/up rows of %d bytes exceed a ring slot", gu_rowb);
  if (phase & 1) {
    gk<<<k * C, MD_THREADS, sg, s>>>(x, ids, slot_of_expert, base, expert_stride, gu_off, 2 * eff, d, h, C, Rg,
                                     g_md_chunk, gu_rowb, rank_lo, rank_hi);
    PS_CHECK_LAUNCH();
  }
  if (!(phase & 2)) return PS_OK;
  // down + combine: row blocks of R rows, one ring slot per expert, all in flight
  int Rd = (d + g_md_sms - 1) / g_md_sms;
  int slot_bytes = (Rd * down_rowb + 127) / 128 * 128;
  if (slot_bytes * k > MD_STAGES * MD_STAGE) {
    Rd = (MD_STAGES * MD_STAGE / k) / down_rowb;
    slot_bytes = (Rd * down_rowb + 127) / 128 * 128;
  }
  PS_REQUIRE(k <= MD_MAXRING && Rd >= 1, "ps_moe_decode_experts: k=%d eff=%d do not fit the ring", k, eff);
  const size_t sd = (size_t)MD_STAGES * MD_STAGE + MD_MAXRING * 8 + (size_t)k * Rd * 4;
  PS_REQUIRE(sd <= 232448 - 1024, "ps_moe_decode_experts: k=%d eff=%d exceed shared memory", k, eff);
  using DownKernel = void (*)(const float*, const int*, const int*, const unsigned char*, long long, long long, int,
                             int, int, const float*, int, float*, int, int, int);
  const int ng = eff % 256 ? 0 : eff / 256;
  DownKernel kern = moe_down_t1_kernel<0, COMP>;
  switch (ng) {
    case 1: kern = moe_down_t1_kernel<1, COMP>; break;
    case 2: kern = moe_down_t1_kernel<2, COMP>; break;
    case 3: kern = moe_down_t1_kernel<3, COMP>; break;
    case 4: kern = moe_down_t1_kernel<4, COMP>; break;
    case 6: kern = moe_down_t1_kernel<6, COMP>; break;
    case 8: kern = moe_down_t1_kernel<8, COMP>; break;
    default: break;
  }
  static size_t set_down[MD_MAXG + 1] = {};
  if (sd > set_down[ng]) {
    PS_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sd));
    set_down[ng] = sd;
  }
  kern<<<(d + Rd - 1) / Rd, MD_THREADS, sd, s>>>(h, ids, slot_of_expert, base, expert_stride, down_off, d, eff, Rd, w,
                                                 k, y, g_md_chunk, slot_bytes, down_rowb);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

static int md_check(int k, int eff, int d, long long expert_stride, long long gu_off, long long down_off,
                    const void* expert_base) {
  PS_REQUIRE(k >= 1 && k <= 64, "ps_moe_decode_experts: k=%d", k);
  PS_REQUIRE(d % 8 == 0 && eff % 8 == 0 && d <= 32 * 8 * MD_MAXG && eff <= 32 * 8 * MD_MAXG,
             "ps_moe_decode_experts: d=%d eff=%d (multiples of 8, <= %d)", d, eff, 32 * 8 * MD_MAXG);
  PS_REQUIRE((expert_stride | gu_off | down_off) % 16 == 0 &&
                 (reinterpret_cast<uintptr_t>(expert_base) & 15) == 0,
             "ps_moe_decode_experts: expert bytes must be 16-byte aligned");
  return PS_OK;
}

extern "C" {

int ps_moe_decode_experts(const float* x, const int* ids, int k, const int* slot_of_expert, const void* expert_base,
                          long long expert_stride, long long gu_off, long long down_off, int eff, int d, float* h,
                          const float* w, float* y, void* stream) {
  int rc = md_check(k, eff, d, expert_stride, gu_off, down_off, expert_base);
  if (rc) return rc;
  return md_launch<false>(x, ids, k, slot_of_expert, expert_base, expert_stride, gu_off, down_off, eff, d, h, w, y,
                          (cudaStream_t)stream, d * 2, eff * 2);
}

int ps_moe_decode_experts_phase(const float* x, const int* ids, int k, const int* slot_of_expert,
                                const void* expert_base, long long expert_stride, long long gu_off, long long down_off,
                                int eff, int d, float* h, const float* w, float* y, int phase, int rank_lo,
                                int rank_hi, void* stream) {
  int rc = md_check(k, eff, d, expert_stride, gu_off, down_off, expert_base);
  if (rc) return rc;
  PS_REQUIRE(phase >= 1 && phase <= 3 && (phase == 2 || slot_of_expert != nullptr || (rank_lo <= 0 && rank_hi >= k)),
             "ps_moe_decode_experts_phase: phase %d, ranks [%d, %d) need slot_of_expert", phase, rank_lo, rank_hi);
  return md_launch<false>(x, ids, k, slot_of_expert, expert_base, expert_stride, gu_off, down_off, eff, d, h, w, y,
                          (cudaStream_t)stream, d * 2, eff * 2, phase, rank_lo, rank_hi);
}

int ps_moe_decode_experts_c(const float* x, const int* ids, int k, const int* slot_of_expert,
                            const void* expert_base, long long expert_stride, long long gu_off, long long down_off,
                            int eff, int d, int gu_row_bytes, int down_row_bytes, float* h, const float* w, float* y,
                            void* stream) {
  int rc = md_check(k, eff, d, expert_stride, gu_off, down_off, expert_base);
  if (rc) return rc;
  PS_REQUIRE(d % 256 == 0 && eff % 256 == 0, "ps_moe_decode_experts_c: coded rows need d, eff multiples of 256");
  const int tg = gu_row_bytes - d * 3 / 2, td = down_row_bytes - eff * 3 / 2;
  PS_REQUIRE(tg >= 16 && tg <= 256 && tg % 16 == 0 && td >= 16 && td <= 256 && td % 16 == 0,
             "ps_moe_decode_experts_c: coded row strides %d / %d (trailers %d / %d)", gu_row_bytes, down_row_bytes,
             tg, td);
  return md_launch<true>(x, ids, k, slot_of_expert, expert_base, expert_stride, gu_off, down_off, eff, d, h, w, y,
                         (cudaStream_t)stream, gu_row_bytes, down_row_bytes);
}

}  // extern "C"

int ps_preload_moe_decode() {
  int n = 0;
#define PS_MDP(C)                                                                      \
  touch_kernel(moe_gu_t1_kernel<0, C>, n); touch_kernel(moe_gu_t1_kernel<1, C>, n);     \
  touch_kernel(moe_gu_t1_kernel<2, C>, n); touch_kernel(moe_gu_t1_kernel<4, C>, n);     \
  touch_kernel(moe_gu_t1_kernel<8, C>, n); touch_kernel(moe_down_t1_kernel<0, C>, n);   \
  touch_kernel(moe_down_t1_kernel<1, C>, n); touch_kernel(moe_down_t1_kernel<2, C>, n); \
  touch_kernel(moe_down_t1_kernel<3, C>, n); touch_kernel(moe_down_t1_kernel<4, C>, n); \
  touch_kernel(moe_down_t1_kernel<6, C>, n); touch_kernel(moe_down_t1_kernel<8, C>, n);
  PS_MDP(false) PS_MDP(true)
#undef PS_MDP
  return n;
}
