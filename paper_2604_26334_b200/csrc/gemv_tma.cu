// K1: decode GEMV streamed through shared memory by the bulk-copy (TMA) engine.
//
// Prices the same MATMUL requests as gemv.cu (`pkg/src/shardplan/model_graph.py:147-153,
// 173-179,202-209`) at t <= 8 tokens per launch: y[t, n] (epi)= sum_k x[t, k] W[n, k],
// W bf16 row-major [N x ldw], x / y fp32, fp32 accumulation.
//
// Why a second GEMV: the register-burst kernel (gemv.cu) keeps its bytes in
// flight in registers, so occupancy caps it near 65-78 % of HBM. Here one
// producer lane per CTA keeps a 5-stage x 32 KB ring of cp.async.bulk copies
// in flight (160 KB per SM, no register cost) and 8 consumer warps read the
// weights from shared memory.
//
// Decomposition (persistent, one CTA per SM): CTA b owns the contiguous row
// range [b*R, (b+1)*R) (R even, so SwiGLU gate/up pairs never straddle CTAs)
// and walks it K-chunk-outer: for each chunk of KC <= 2048 columns every
// consumer thread holds its 8 columns of x (x t tokens) in registers and the
// ring streams the range's rows in blocks of RS rows (RS*KC*2 = 32 KB, one
// bulk copy per row segment). Per stage each thread forms RS x t partial dot
// products, reduce-scattered across its warp with shuffles, and the warp adds
// them into its own per-row fp32 accumulators in shared memory — warps never
// synchronise with each other inside the K loop. The epilogue sums the 8
// warps' partials (fixed order: deterministic) and stores / accumulates /
// applies SwiGLU once per row.
#include <stdlib.h>

#include "common.cuh"
#include "mbarrier.cuh"
#include "wcodec.cuh"
#include "../../include/pshard.h"

namespace ps {

constexpr int GT_STAGES = 5;
constexpr int GT_STAGE_BYTES = 32768;
#ifndef PS_GT_CONSUMERS_LO
#define PS_GT_CONSUMERS_LO 8
#endif
#ifndef PS_GT_CONSUMERS_HI
#define PS_GT_CONSUMERS_HI 8
#endif
// Consumer warps per token count, the same for bf16 and coded rows (identical
// decomposition = bit-identical outputs). 8: an A/B with 16 at t <= 4 (tools/
// bench_gemv_nc.py, r02) gained the coded kernel 3 % on the 235 MB matrix and cost the
// bf16 kernel 5-12 % on 25-64 MB pieces; 16 regressed t = 8 outright.
constexpr int gt_consumers(int T) { return T <= 4 ? PS_GT_CONSUMERS_LO : PS_GT_CONSUMERS_HI; }
constexpr int gt_threads(int T) { return 32 * (1 + gt_consumers(T)); }  // + producer warp

// Per token count: columns per consumer thread (x kept in registers: CPT * T floats)
// and rows per stage (RS * KC * 2 = 32 KB, KC = 256 * CPT columns per chunk).
// COMP: rows in the exponent-coded format (`ps_gemv_bf16c`, runtime/wcomp.py): a
// row segment of KC columns is staged as KC sign|mantissa bytes, KC/2 bytes of 4-bit
// exponent codes, then the row's trailer (base exponent, escape list; <= 256 bytes).
constexpr int gt_pow2_floor(int v) { return v >= 16 ? 16 : v >= 8 ? 8 : v >= 4 ? 4 : v >= 2 ? 2 : 1; }
constexpr int GT_TRAILER_MAX = 256;

template <int T, bool COMP = false> struct GtShape {
  static constexpr int NC = gt_consumers(T);
  // 16 consumer warps: 8 columns per thread at every T (KC = 4096); 8 warps: 16 / 8
  static constexpr int CPT = NC >= 16 ? 8 : (T <= 4 ? 16 : 8);
  static constexpr int KC = NC * 32 * CPT;
  static constexpr int ROWB = COMP ? KC * 3 / 2 + GT_TRAILER_MAX : KC * 2;   // stage bytes per row segment
  static constexpr int RS = COMP ? gt_pow2_floor(GT_STAGE_BYTES / ROWB) : GT_STAGE_BYTES / (KC * 2);
  static constexpr int V = RS * T;  // partial sums reduced per stage
  // warp_reduce_scatter halves V each step: a non-power-of-two V would drop values
  static_assert(RS >= 1 && (V & (V - 1)) == 0, "rows x tokens per stage must be a power of two");
};

__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds_v2(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ uint4 lds_v4(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}

// 8 bf16 weights x 8 fp32 activations, packed fp32x2 FMA (two partial sums).
__device__ __forceinline__ float2 dot8x2(uint4 w, const float2* x, float2 s) {
  s = __ffma2_rn(x[0], make_float2(bf16_lo(w.x), bf16_hi(w.x)), s);
  s = __ffma2_rn(x[1], make_float2(bf16_lo(w.y), bf16_hi(w.y)), s);
  s = __ffma2_rn(x[2], make_float2(bf16_lo(w.z), bf16_hi(w.z)), s);
  s = __ffma2_rn(x[3], make_float2(bf16_lo(w.w), bf16_hi(w.w)), s);
  return s;
}

// Reduce-scatter N values over the lanes that differ in bit O and below: after the
// call lane l holds the warp sum of one value (index fixed by l's high bits).
template <int N, int O, int V>
__device__ __forceinline__ void warp_reduce_scatter(float (&v)[V], int lane) {
  if constexpr (O >= 1) {
    if constexpr (N > 1) {
      const bool upper = (lane & O) != 0;
#pragma unroll
      for (int i = 0; i < N / 2; ++i) {
        const float send = upper ? v[i] : v[i + N / 2];
        const float keep = upper ? v[i + N / 2] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, O);
      }
      warp_reduce_scatter<N / 2, O / 2, V>(v, lane);
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], O);
      warp_reduce_scatter<1, O / 2, V>(v, lane);
    }
  }
}

// XF: the "early head" variant (executor: one-token passes reading a CPU-placed output
// head zero-copy). Launched on a side stream at the start of the pass, its producers
// stream the head rows from host memory while the layers compute on the other SMs; the
// consumers wait for *xflag >= xseq (set on the compute stream once x is final) instead of
// griddepcontrol.wait, and read x through L2 (a previous pass left stale L1 lines).
template <int T, int EPI, bool COMP = false, bool XF = false>
__global__ void __launch_bounds__(gt_threads(T), 1)
gemv_tma_kernel(const float* __restrict__ x, int ldx, int tt, const __nv_bfloat16* __restrict__ W, int N, int K,
                long long ldw, float* __restrict__ y, int ldy, int rows_per_cta, int stages,
                const unsigned* __restrict__ xflag, unsigned xseq, unsigned* fault) {
  using S = GtShape<T, COMP>;
  constexpr int CPT = S::CPT, KC = S::KC, RS = S::RS, V = S::V, ROWB = S::ROWB;
  constexpr int GT_CONSUMERS = S::NC, GT_THREADS = gt_threads(T);
  const uint8_t* Wb = reinterpret_cast<const uint8_t*>(W);   // COMP: ldw is in bytes
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * GT_STAGE_BYTES);
  uint64_t* empty = full + stages;
  // per-warp row accumulators [GT_CONSUMERS][rows_per_cta][T]: warps never wait for
  // each other inside the K loop; the 8 partials are summed once, in the epilogue
  float* acc = reinterpret_cast<float*>(empty + stages);

  pdl_trigger();
  const int r0 = blockIdx.x * rows_per_cta;
  if (r0 >= N) return;  // whole CTA, before any barrier
  const int r1 = min(N, r0 + rows_per_cta);
  const int nrows = r1 - r0;
  const int nchunks = (K + KC - 1) / KC;
  const int nblocks = (nrows + RS - 1) / RS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], GT_CONSUMERS); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < GT_CONSUMERS * rows_per_cta * T; i += GT_THREADS) acc[i] = 0.f;
  __syncthreads();

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int c = 0; c < nchunks; ++c) {
        const int kc = min(KC, K - c * KC);
        for (int b = 0; b < nblocks; ++b) {
          const int rb = r0 + b * RS;
          const int nr = min(RS, r1 - rb);
          mbar_wait(&empty[s], ph ^ 1);
          fence_proxy_async_smem();   // consumers' generic reads -> the next bulk copy
          uint8_t* dst = ring + s * GT_STAGE_BYTES;
          if constexpr (COMP) {
            const uint32_t tb = (uint32_t)(ldw - (long long)K * 3 / 2);   // the row's trailer
            mbar_expect_tx(&full[s], (uint32_t)(nr * (kc + kc / 2 + tb)));
            for (int r = 0; r < nr; ++r) {
              const uint8_t* row = Wb + (long long)(rb + r) * ldw;
              bulk_load(dst + r * ROWB, row + (long long)c * KC, (uint32_t)kc, &full[s]);
              bulk_load(dst + r * ROWB + KC, row + K + (long long)c * (KC / 2), (uint32_t)(kc / 2), &full[s]);
              bulk_load(dst + r * ROWB + KC * 3 / 2, row + (long long)K * 3 / 2, tb, &full[s]);
            }
          } else {
            mbar_expect_tx(&full[s], (uint32_t)(nr * kc * 2));
            for (int r = 0; r < nr; ++r)
              bulk_load(dst + r * KC * 2, W + (long long)(rb + r) * ldw + (long long)c * KC, (uint32_t)(kc * 2),
                        &full[s]);
          }
          if (++s == stages) { s = 0; ph ^= 1; }
        }
      }
    }
    return;
  }

  // weights are never written inside a pass (the producer may stream them before
  // the previous kernel finished); x and y are: consumers wait for it (PDL), or (XF) for
  // the flag that says x is final
  if constexpr (XF) {
    if ((threadIdx.x & 31) == 0) {
      unsigned long long t0, t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      while ((int)(*reinterpret_cast<const volatile unsigned*>(xflag) - xseq) < 0) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 2000000000ull) {   // 2 s: record the fault (the host raises) instead of hanging
          if (fault) raise_fault(fault, FAULT_HEAD, xseq);
          break;
        }
        __nanosleep(256);
      }
      __threadfence();
    }
    __syncwarp();
  } else {
    pdl_wait();
  }
  const int j = threadIdx.x - 32;  // consumer thread 0..255
  const int cw = warp - 1;
  // value index this lane holds after the reduce-scatter, and whether it writes it
  int my_idx = 0;
  {
    int n = V;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1)
      if (n > 1) { if (lane & o) my_idx += n / 2; n >>= 1; }
  }
  constexpr int PER_LANE = V > 32 ? V / 32 : 1;   // values a lane holds after the reduce-scatter
  const bool writer = V >= 32 || (lane & ((32 / V) - 1)) == 0;
  int it = 0, s = 0;
  uint32_t ph = 0;
  const uint32_t ring_s = smem_u32(ring);
  int colb[CPT / 8];   // this thread's 8-column groups within a chunk
#pragma unroll
  for (int h = 0; h < CPT / 8; ++h) colb[h] = (h * GT_CONSUMERS * 32 + j) * 8;
  for (int c = 0; c < nchunks; ++c) {
    const int kc = min(KC, K - c * KC);
    float2 xr[T][CPT / 2];
#pragma unroll
    for (int t = 0; t < T; ++t) {
#pragma unroll
      for (int h = 0; h < CPT / 8; ++h) {
        const int col = (h * GT_CONSUMERS * 32 + j) * 8;   // 8-column groups, consecutive threads adjacent
        if (col < kc && t < tt) {
          const float4* xp = reinterpret_cast<const float4*>(x + (long long)t * ldx + (long long)c * KC + col);
          float4 a, b;
          if constexpr (XF) {
            a = __ldcg(xp);
            b = __ldcg(xp + 1);
          } else {
            a = __ldg(xp);
            b = __ldg(xp + 1);
          }
          xr[t][h * 4 + 0] = make_float2(a.x, a.y); xr[t][h * 4 + 1] = make_float2(a.z, a.w);
          xr[t][h * 4 + 2] = make_float2(b.x, b.y); xr[t][h * 4 + 3] = make_float2(b.z, b.w);
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i) xr[t][h * 4 + i] = make_float2(0.f, 0.f);
        }
      }
    }
    for (int b = 0; b < nblocks; ++b, ++it) {
      const int rb = r0 + b * RS;
      const int nr = min(RS, r1 - rb);
      mbar_wait(&full[s], ph);
      const uint8_t* stage = ring + s * GT_STAGE_BYTES;
      float v[V];
      // (coded rows at 64 values per stage: the second copy of the loop spills; general path)
      if (!(COMP && V > 32) && nr == RS && kc == KC) {
        // full block (all but a CTA's last one): no bounds tests, shared loads by 32-bit
        // address; the same values and accumulation order as the general path below
        const uint32_t sa = ring_s + s * GT_STAGE_BYTES;
#pragma unroll
        for (int r = 0; r < RS; ++r) {
          uint4 w[CPT / 8];
          if constexpr (COMP) {
            const uint32_t ra = sa + r * ROWB;
            const uint32_t hdr = lds_u32(ra + KC * 3 / 2);       // base | n_escapes << 8
            const uint32_t base7 = ((hdr & 0xFFu) * 0x10001u) << 7;
            uint2 sm[CPT / 8];
            uint32_t nb[CPT / 8];
#pragma unroll
            for (int h = 0; h < CPT / 8; ++h) {
              sm[h] = lds_v2(ra + colb[h]);
              nb[h] = lds_u32(ra + KC + colb[h] / 2);
              w[h] = gt_decode8(sm[h], nb[h], base7);
            }
            if (hdr >> 8) {   // the row has escapes (warp-uniform): patch the groups holding one
              const uint32_t* trailer = reinterpret_cast<const uint32_t*>(stage + r * ROWB + KC * 3 / 2);
#pragma unroll
              for (int h = 0; h < CPT / 8; ++h)
                if (gt_escapes(nb[h])) w[h] = gt_patch_escapes(w[h], sm[h], nb[h], trailer, c * KC + colb[h]);
            }
          } else {
#pragma unroll
            for (int h = 0; h < CPT / 8; ++h) w[h] = lds_v4(sa + r * KC * 2 + colb[h] * 2);
          }
#pragma unroll
          for (int t = 0; t < T; ++t) {
            float2 p = make_float2(0.f, 0.f);
#pragma unroll
            for (int h = 0; h < CPT / 8; ++h) p = dot8x2(w[h], &xr[t][h * 4], p);
            v[r * T + t] = p.x + p.y;
          }
        }
      } else {
#pragma unroll
      for (int r = 0; r < RS; ++r) {
        uint4 w[CPT / 8];
        if constexpr (COMP) {
          const uint8_t* rowp = stage + r * ROWB;
          const uint32_t* trailer = reinterpret_cast<const uint32_t*>(rowp + KC * 3 / 2);
          const bool live = r < nr;
          const uint32_t base7 = live ? ((trailer[0] & 0xFFu) * 0x10001u) << 7 : 0u;
          uint2 sm[CPT / 8];
          uint32_t nb[CPT / 8], esc = 0;
#pragma unroll
          for (int h = 0; h < CPT / 8; ++h) {
            const int col = (h * GT_CONSUMERS * 32 + j) * 8;
            const bool ok = live && col < kc;
            sm[h] = ok ? *reinterpret_cast<const uint2*>(rowp + col) : make_uint2(0, 0);
            nb[h] = ok ? *reinterpret_cast<const uint32_t*>(rowp + KC + col / 2) : 0u;
            w[h] = ok ? gt_decode8(sm[h], nb[h], base7) : make_uint4(0, 0, 0, 0);
            esc |= gt_escapes(nb[h]);
          }
          if (esc) {   // rare: one branch per row for all of this thread's groups
#pragma unroll
            for (int h = 0; h < CPT / 8; ++h)
              if (gt_escapes(nb[h]))
                w[h] = gt_patch_escapes(w[h], sm[h], nb[h], trailer, c * KC + (h * GT_CONSUMERS * 32 + j) * 8);
          }
        } else {
#pragma unroll
          for (int h = 0; h < CPT / 8; ++h) {
            const int col = (h * GT_CONSUMERS * 32 + j) * 8;
            w[h] = (r < nr && col < kc) ? *reinterpret_cast<const uint4*>(stage + (r * KC + col) * 2)
                                        : make_uint4(0, 0, 0, 0);
          }
        }
#pragma unroll
        for (int t = 0; t < T; ++t) {
          float2 p = make_float2(0.f, 0.f);
#pragma unroll
          for (int h = 0; h < CPT / 8; ++h) p = dot8x2(w[h], &xr[t][h * 4], p);
          v[r * T + t] = p.x + p.y;
        }
      }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);  // this warp is done reading the stage
      if (++s == stages) { s = 0; ph ^= 1; }
      // reduce-scatter V values over the warp, then butterfly the rest: lane l ends
      // with the warp sum of value my_idx
      warp_reduce_scatter<V, 16, V>(v, lane);
      if (writer) {
#pragma unroll
        for (int i = 0; i < PER_LANE; ++i) {
          const int idx = my_idx + i;
          const int r = idx / T, t = idx - (idx / T) * T;
          if (r < nr) acc[(cw * rows_per_cta + rb - r0 + r) * T + t] += v[i];
        }
      }
    }
  }
  named_sync(1, GT_CONSUMERS * 32);
  const int stride_w = rows_per_cta * T;
  for (int idx = j; idx < nrows * T; idx += GT_CONSUMERS * 32) {
    const int r = idx / T, t = idx - (idx / T) * T;
    if (t >= tt) continue;
    const int row = r0 + r;
    float a = 0.f, b = 0.f;
#pragma unroll
    for (int w = 0; w < GT_CONSUMERS; ++w) a += acc[w * stride_w + idx];   // fixed order: deterministic
    if (EPI == PS_EPI_SWIGLU) {
      if ((r & 1) == 0 && row + 1 < N) {
#pragma unroll
        for (int w = 0; w < GT_CONSUMERS; ++w) b += acc[w * stride_w + idx + T];
        y[(long long)t * ldy + (row >> 1)] = silu(a) * b;
      }
    } else if (EPI == PS_EPI_ACCUM) {
      y[(long long)t * ldy + row] += a;
    } else {
      y[(long long)t * ldy + row] = a;
    }
  }
}

static int g_tma_sms = 0;
static int g_tma_stages = 0;

template <int T, int EPI, bool COMP = false, bool XF = false>
static int launch_tma(const float* x, int ldx, int tt, const __nv_bfloat16* W, int N, int K, long long ldw, float* y,
                      int ldy, cudaStream_t s, int grid_cap, const unsigned* xflag = nullptr, unsigned xseq = 0) {
  if (!g_tma_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_tma_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_tma_sms <= 0) g_tma_sms = 148;
  }
  const int pairs = (N + 1) / 2;
  int grid = grid_cap > 0 ? grid_cap : g_tma_sms;
  if (grid > pairs) grid = pairs;
  if (g_tma_stages == 0) {  // PS_GEMV_STAGES: ring depth override for tuning sweeps
    const char* e = getenv("PS_GEMV_STAGES");
    int v = e ? atoi(e) : GT_STAGES;
    g_tma_stages = v < 2 ? 2 : (v > 12 ? 12 : v);
  }
  const int stages = g_tma_stages;
  constexpr int GT_CONSUMERS = gt_consumers(T), GT_THREADS = gt_threads(T);
  // the per-row accumulators share shared memory with the ring
  const int max_rows = ((232448 - stages * (GT_STAGE_BYTES + 16)) / (GT_CONSUMERS * T * 4)) & ~1;
  int rows_per_cta = 2 * ((pairs + grid - 1) / grid);
  if (rows_per_cta > max_rows) rows_per_cta = max_rows;
  grid = (N + rows_per_cta - 1) / rows_per_cta;
  const size_t smem = (size_t)stages * (GT_STAGE_BYTES + 16) + (size_t)GT_CONSUMERS * rows_per_cta * T * 4;
  static size_t smem_set = 0;
  if (smem > smem_set) {
    PS_CHECK_CUDA(cudaFuncSetAttribute(gemv_tma_kernel<T, EPI, COMP, XF>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    smem_set = smem;
  }
  if constexpr (XF) {   // side stream, plain launch: no programmatic dependency on anything
    gemv_tma_kernel<T, EPI, COMP, XF><<<grid, GT_THREADS, smem, s>>>(x, ldx, tt, W, N, K, ldw, y, ldy, rows_per_cta,
                                                                     stages, xflag, xseq, fault_dev());
  } else {
    launch_k(gemv_tma_kernel<T, EPI, COMP, XF>, grid, GT_THREADS, smem, s, x, ldx, tt, W, N, K, ldw, y, ldy,
             rows_per_cta, stages, (const unsigned*)nullptr, 0u, (unsigned*)nullptr);
  }
  PS_CHECK_LAUNCH();
  return PS_OK;
}

template <int T>
static int launch_tma_epi(int epi, const float* x, int ldx, int tt, const __nv_bfloat16* W, int N, int K,
                          long long ldw, float* y, int ldy, cudaStream_t s, int grid_cap) {
  if (epi == PS_EPI_STORE) return launch_tma<T, PS_EPI_STORE>(x, ldx, tt, W, N, K, ldw, y, ldy, s, grid_cap);
  if (epi == PS_EPI_ACCUM) return launch_tma<T, PS_EPI_ACCUM>(x, ldx, tt, W, N, K, ldw, y, ldy, s, grid_cap);
  return launch_tma<T, PS_EPI_SWIGLU>(x, ldx, tt, W, N, K, ldw, y, ldy, s, grid_cap);
}

// Entry used by gemv.cu's dispatcher (tt <= 8 tokens of one launch).
int gemv_tma_launch(const float* x, int ldx, int tt, const __nv_bfloat16* W, int N, int K, long long ldw, float* y,
                    int ldy, int epi, cudaStream_t s, int grid_cap) {
  if (tt == 1) return launch_tma_epi<1>(epi, x, ldx, tt, W, N, K, ldw, y, ldy, s, grid_cap);
  if (tt == 2) return launch_tma_epi<2>(epi, x, ldx, tt, W, N, K, ldw, y, ldy, s, grid_cap);
  if (tt <= 4) return launch_tma_epi<4>(epi, x, ldx, tt, W, N, K, ldw, y, ldy, s, grid_cap);
  return launch_tma_epi<8>(epi, x, ldx, tt, W, N, K, ldw, y, ldy, s, grid_cap);
}

template <int T>
static int launch_tmac_epi(int epi, const float* x, int ldx, int tt, const void* Wc, int N, int K, long long ldw,
                           float* y, int ldy, cudaStream_t s) {
  auto W = static_cast<const __nv_bfloat16*>(Wc);
  if (epi == PS_EPI_STORE) return launch_tma<T, PS_EPI_STORE, true>(x, ldx, tt, W, N, K, ldw, y, ldy, s, 0);
  if (epi == PS_EPI_ACCUM) return launch_tma<T, PS_EPI_ACCUM, true>(x, ldx, tt, W, N, K, ldw, y, ldy, s, 0);
  return launch_tma<T, PS_EPI_SWIGLU, true>(x, ldx, tt, W, N, K, ldw, y, ldy, s, 0);
}

}  // namespace ps

extern "C" int ps_gemv_bf16c(const float* x, int ldx, int t, const void* Wc, int N, int K, long long ldw,
                             float* y, int ldy, int epilogue, void* stream) {
  using namespace ps;
  PS_REQUIRE(t >= 1 && t <= 8, "ps_gemv_bf16c: t=%d outside [1, 8]", t);
  PS_REQUIRE(K % 256 == 0 && ldx % 4 == 0, "ps_gemv_bf16c: K must be a multiple of 256");
  const long long tb = ldw - (long long)K * 3 / 2;
  PS_REQUIRE(tb >= 16 && tb <= GT_TRAILER_MAX && tb % 16 == 0,
             "ps_gemv_bf16c: row stride %lld leaves a %lld-byte trailer (16..%d, multiple of 16)", ldw, tb,
             GT_TRAILER_MAX);
  PS_REQUIRE(((uintptr_t)Wc & 15) == 0 && ((uintptr_t)x & 15) == 0, "ps_gemv_bf16c: Wc and x must be 16-byte aligned");
  PS_REQUIRE(epilogue != PS_EPI_SWIGLU || N % 2 == 0, "ps_gemv_bf16c: SWIGLU needs an even N");
  if (N <= 0) return PS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (t == 1) return launch_tmac_epi<1>(epilogue, x, ldx, t, Wc, N, K, ldw, y, ldy, s);
  if (t == 2) return launch_tmac_epi<2>(epilogue, x, ldx, t, Wc, N, K, ldw, y, ldy, s);
  if (t <= 4) return launch_tmac_epi<4>(epilogue, x, ldx, t, Wc, N, K, ldw, y, ldy, s);
  return launch_tmac_epi<8>(epilogue, x, ldx, t, Wc, N, K, ldw, y, ldy, s);
}

extern "C" int ps_gemv_head_early(const float* x, int K, const void* W, int N, long long ldw, int coded, float* y,
                                  int grid_cap, const unsigned* xflag, unsigned xseq, void* stream) {
  using namespace ps;
  PS_REQUIRE(K % 256 == 0 && ((uintptr_t)W & 15) == 0 && ((uintptr_t)x & 15) == 0 && xflag != nullptr,
             "ps_gemv_head_early: K %d, alignment, flag", K);
  if (N <= 0) return PS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  auto Wb = static_cast<const __nv_bfloat16*>(W);
  if (coded) {
    const long long tb = ldw - (long long)K * 3 / 2;
    PS_REQUIRE(tb >= 16 && tb <= GT_TRAILER_MAX && tb % 16 == 0, "ps_gemv_head_early: coded row stride %lld", ldw);
    return launch_tma<1, PS_EPI_STORE, true, true>(x, K, 1, Wb, N, K, ldw, y, N, s, grid_cap, xflag, xseq);
  }
  return launch_tma<1, PS_EPI_STORE, false, true>(x, K, 1, Wb, N, K, ldw, y, N, s, grid_cap, xflag, xseq);
}

namespace ps {
__global__ void set_flag_kernel(unsigned* flag, unsigned v) {
  __threadfence();   // this stream's earlier writes (x) before the flag
  *reinterpret_cast<volatile unsigned*>(flag) = v;
  __threadfence();
}
}  // namespace ps

extern "C" int ps_set_flag(unsigned* flag, unsigned value, void* stream) {
  using namespace ps;
  set_flag_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(flag, value);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

namespace ps {
// Coded rows -> bf16 rows (GEMM passes that stream coded pieces: the tcgen05 GEMM reads
// bf16 operands). One thread per 8 weights; rows of ld_in bytes in, K bf16 out.
__global__ void expand_coded_kernel(const uint8_t* __restrict__ in, long long ld_in, int rows, int K,
                                    __nv_bfloat16* __restrict__ out, long long ld_out) {
  const long long groups = (long long)rows * (K / 8);
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < groups;
       g += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(g / (K / 8)), col = (int)(g % (K / 8)) * 8;
    const uint8_t* row = in + r * ld_in;
    const uint32_t* trailer = reinterpret_cast<const uint32_t*>(row + (long long)K * 3 / 2);
    const uint32_t base7 = ((trailer[0] & 0xFFu) * 0x10001u) << 7;
    const uint2 sm = *reinterpret_cast<const uint2*>(row + col);
    const uint32_t nb = *reinterpret_cast<const uint32_t*>(row + K + col / 2);
    uint4 w = gt_decode8(sm, nb, base7);
    if (gt_escapes(nb)) w = gt_patch_escapes(w, sm, nb, trailer, col);
    *reinterpret_cast<uint4*>(out + r * ld_out + col) = w;
  }
}
}  // namespace ps

extern "C" int ps_expand_coded(const void* coded, long long ld_in, int rows, int K, void* out, long long ld_out,
                               void* stream) {
  using namespace ps;
  PS_REQUIRE(K % 256 == 0 && ld_out % 8 == 0 && ld_in >= (long long)K * 3 / 2 + 16,
             "ps_expand_coded: K %d, ld_in %lld, ld_out %lld", K, ld_in, ld_out);
  PS_REQUIRE(((uintptr_t)coded & 15) == 0 && ((uintptr_t)out & 15) == 0, "ps_expand_coded: alignment");
  if (rows <= 0) return PS_OK;
  const long long groups = (long long)rows * (K / 8);
  const int blocks = (int)((groups + 255) / 256 < 148 * 16 ? (groups + 255) / 256 : 148 * 16);
  expand_coded_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(static_cast<const uint8_t*>(coded), ld_in, rows, K,
                                                                static_cast<__nv_bfloat16*>(out), ld_out);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

int ps_preload_gemv_tma() {
  using namespace ps;
  int n = 0;
#define PS_T(T)                                                \
  touch_kernel(gemv_tma_kernel<T, PS_EPI_STORE>, n);           \
  touch_kernel(gemv_tma_kernel<T, PS_EPI_ACCUM>, n);           \
  touch_kernel(gemv_tma_kernel<T, PS_EPI_SWIGLU>, n);          \
  touch_kernel(gemv_tma_kernel<T, PS_EPI_STORE, true>, n);     \
  touch_kernel(gemv_tma_kernel<T, PS_EPI_ACCUM, true>, n);     \
  touch_kernel(gemv_tma_kernel<T, PS_EPI_SWIGLU, true>, n);
  PS_T(1) PS_T(2) PS_T(4) PS_T(8)
#undef PS_T
  touch_kernel(expand_coded_kernel, n);
  touch_kernel(gemv_tma_kernel<1, PS_EPI_STORE, false, true>, n);
  touch_kernel(gemv_tma_kernel<1, PS_EPI_STORE, true, true>, n);
  touch_kernel(set_flag_kernel, n);
  return n;
}
