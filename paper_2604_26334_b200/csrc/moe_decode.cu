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
//   CTA (j, c), j < k, c < C: expert e = ids[j] (slot_of_expert[e] when the
//   experts were fetched into VRAM slots), rows [c*R, (c+1)*R) of its matrix.
//   A producer lane streams those rows (contiguous: row-major, K columns) into
//   a 6 x 32 KB shared-memory ring with cp.async.bulk; 8 consumer warps take
//   whole rows (x held in registers, packed fp32x2 FMA, one warp reduction per
//   row) and leave one fp32 sum per row in shared memory.
//   gate/up (rows interleaved gate, up): h[j][r/2] = silu(gate) * up.
//   down: out[j][r], then the last of the k CTAs of row block c (ticket counter)
//   adds sum_j w[j] * out[j][r], j ascending, into y[r] — the order moe.cu's
//   combine uses, so the result does not depend on CTA scheduling.
#include "common.cuh"
#include "mbarrier.cuh"
#include "../../include/pshard.h"

namespace ps {

constexpr int MD_STAGES = 6;
constexpr int MD_STAGE = 32768;
constexpr int MD_WARPS = 8;
constexpr int MD_THREADS = 32 * (1 + MD_WARPS);
constexpr int MD_MAXG = 8;    // 8-column groups per lane: K <= 32 * 8 * 8 = 2048

__device__ __forceinline__ float2 md_dot8(uint4 w, const float2* x, float2 s) {
  s = __ffma2_rn(x[0], make_float2(bf16_lo(w.x), bf16_hi(w.x)), s);
  s = __ffma2_rn(x[1], make_float2(bf16_lo(w.y), bf16_hi(w.y)), s);
  s = __ffma2_rn(x[2], make_float2(bf16_lo(w.z), bf16_hi(w.z)), s);
  s = __ffma2_rn(x[3], make_float2(bf16_lo(w.w), bf16_hi(w.w)), s);
  return s;
}

template <int DOWN>
__global__ void __launch_bounds__(MD_THREADS, 1)
moe_decode_kernel(const float* __restrict__ x, long long x_gs, const int* __restrict__ ids,
                  const int* __restrict__ slot_of_expert, const unsigned char* __restrict__ base,
                  long long expert_stride, long long mat_off, int N, int K, float* __restrict__ out,
                  long long out_gs, int C, int R, const float* __restrict__ w, int k, float* __restrict__ y,
                  unsigned* __restrict__ tickets) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ int s_last;
  const int j = blockIdx.x / C, c = blockIdx.x - j * C;
  const int r0 = c * R;
  if (r0 >= N) return;   // the same for every j: no ticket is ever waited for
  const int nrows = min(N, r0 + R) - r0;
  const int rowb = K * 2;
  const int RS = MD_STAGE / rowb;
  const int nst = (nrows + RS - 1) / RS;
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + MD_STAGES * MD_STAGE);
  uint64_t* empty = full + MD_STAGES;
  float* acc = reinterpret_cast<float*>(empty + MD_STAGES);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < MD_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], MD_WARPS); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    if (lane == 0) {
      const int e = ids[j];
      const long long slot = slot_of_expert ? slot_of_expert[e] : e;
      const uint8_t* W = base + slot * expert_stride + mat_off + (long long)r0 * rowb;
      int s = 0;
      uint32_t ph = 0;
      for (int b = 0; b < nst; ++b) {
        const int nr = min(RS, nrows - b * RS);
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], (uint32_t)(nr * rowb));
        bulk_load(ring + s * MD_STAGE, W + (long long)b * RS * rowb, (uint32_t)(nr * rowb), &full[s]);
        if (++s == MD_STAGES) { s = 0; ph ^= 1; }
      }
    }
    return;
  }

  const int cw = warp - 1;
  const float* xj = x + j * x_gs;
  float2 xr[MD_MAXG][4];
#pragma unroll
  for (int g = 0; g < MD_MAXG; ++g) {
    const int col = (g * 32 + lane) * 8;
    if (col < K) {
      const float4* xp = reinterpret_cast<const float4*>(xj + col);
      const float4 a = __ldg(xp), b = __ldg(xp + 1);
      xr[g][0] = make_float2(a.x, a.y); xr[g][1] = make_float2(a.z, a.w);
      xr[g][2] = make_float2(b.x, b.y); xr[g][3] = make_float2(b.z, b.w);
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) xr[g][i] = make_float2(0.f, 0.f);
    }
  }
  int s = 0;
  uint32_t ph = 0;
  for (int b = 0; b < nst; ++b) {
    const int nr = min(RS, nrows - b * RS);
    mbar_wait(&full[s], ph);
    const uint8_t* st = ring + s * MD_STAGE;
    for (int r = cw; r < nr; r += MD_WARPS) {
      float2 p = make_float2(0.f, 0.f);
#pragma unroll
      for (int g = 0; g < MD_MAXG; ++g) {
        const int col = (g * 32 + lane) * 8;
        if (col < K) p = md_dot8(*reinterpret_cast<const uint4*>(st + r * rowb + col * 2), xr[g], p);
      }
      const float v = warp_sum(p.x + p.y);
      if (lane == 0) acc[b * RS + r] = v;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == MD_STAGES) { s = 0; ph ^= 1; }
  }
  named_sync(1, MD_WARPS * 32);
  const int t = threadIdx.x - 32;
  if constexpr (!DOWN) {
    for (int i = t; i < nrows / 2; i += MD_WARPS * 32)
      out[j * out_gs + (r0 >> 1) + i] = silu(acc[2 * i]) * acc[2 * i + 1];
  } else {
    for (int i = t; i < nrows; i += MD_WARPS * 32) out[j * out_gs + r0 + i] = acc[i];
    __threadfence();
    named_sync(1, MD_WARPS * 32);
    if (t == 0) s_last = atomicAdd(&tickets[c], 1u) == (unsigned)(k - 1);
    named_sync(1, MD_WARPS * 32);
    if (!s_last) return;
    __threadfence();
    for (int i = t; i < nrows; i += MD_WARPS * 32) {
      float sum = 0.f;
      for (int jj = 0; jj < k; ++jj) sum += w[jj] * __ldcg(out + jj * out_gs + r0 + i);
      y[r0 + i] += sum;
    }
    if (t == 0) tickets[c] = 0u;   // ready for the next launch (stream order)
  }
}

static int g_md_sms = 0;

static size_t md_smem(int R) { return (size_t)MD_STAGES * (MD_STAGE + 16) + (size_t)R * 4; }

}  // namespace ps

using namespace ps;

extern "C" {

int ps_moe_decode_experts(const float* x, const int* ids, int k, const int* slot_of_expert, const void* expert_base,
                          long long expert_stride, long long gu_off, long long down_off, int eff, int d, float* h,
                          float* out, const float* w, float* y, unsigned* tickets, void* stream) {
  PS_REQUIRE(k >= 1 && k <= 64, "ps_moe_decode_experts: k=%d", k);
  PS_REQUIRE(d % 8 == 0 && eff % 8 == 0 && d <= 32 * 8 * MD_MAXG && eff <= 32 * 8 * MD_MAXG,
             "ps_moe_decode_experts: d=%d eff=%d (multiples of 8, <= %d)", d, eff, 32 * 8 * MD_MAXG);
  PS_REQUIRE((expert_stride | gu_off | down_off) % 16 == 0 &&
                 (reinterpret_cast<uintptr_t>(expert_base) & 15) == 0,
             "ps_moe_decode_experts: expert bytes must be 16-byte aligned");
  if (!g_md_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_md_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_md_sms <= 0) g_md_sms = 148;
  }
  const int C = g_md_sms / k > 0 ? g_md_sms / k : 1;
  PS_REQUIRE(C <= PS_MOE_DECODE_TICKETS, "ps_moe_decode_experts: %d row blocks > ticket buffer", C);
  auto base = static_cast<const unsigned char*>(expert_base);
  cudaStream_t s = (cudaStream_t)stream;
  static size_t set0 = 0, set1 = 0;
  // gate/up: N = 2 * eff interleaved rows, even rows per CTA so pairs never straddle
  const int Rg = 2 * ((eff + C - 1) / C);
  const size_t sg = md_smem(Rg);
  if (sg > set0) {
    PS_CHECK_CUDA(cudaFuncSetAttribute(moe_decode_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sg));
    set0 = sg;
  }
  moe_decode_kernel<0><<<k * C, MD_THREADS, sg, s>>>(x, 0, ids, slot_of_expert, base, expert_stride, gu_off,
                                                     2 * eff, d, h, eff, C, Rg, nullptr, k, nullptr, nullptr);
  PS_CHECK_LAUNCH();
  const int Rd = (d + C - 1) / C;
  const size_t sd = md_smem(Rd);
  if (sd > set1) {
    PS_CHECK_CUDA(cudaFuncSetAttribute(moe_decode_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sd));
    set1 = sd;
  }
  moe_decode_kernel<1><<<k * C, MD_THREADS, sd, s>>>(h, eff, ids, slot_of_expert, base, expert_stride, down_off, d,
                                                     eff, out, d, C, Rd, w, k, y, tickets);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

}  // extern "C"

int ps_preload_moe_decode() {
  int n = 0;
  touch_kernel(moe_decode_kernel<0>, n);
  touch_kernel(moe_decode_kernel<1>, n);
  return n;
}
