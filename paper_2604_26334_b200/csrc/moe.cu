// K5: MoE router top-k and routed-expert compute (Qwen3-MoE style).
//
// Prices: MOE_ROUTE (t, d, E) and the expert MATMUL (t*k, d, mats*eff) of
// `pkg/src/shardplan/model_graph.py:181-200`. The plan charges a streamed
// expert group at ALL E experts (`:286-292`); the executor moves only the
// experts the router selects:
//   * decode (t <= 32): the expert kernels read the selected experts straight
//     from host-mapped memory (zero-copy, ~47-51 GB/s measured over PCIe
//     Gen5), so no expert byte crosses the link unless it is routed to;
//   * prefill (all experts touched): the group streams through the ring in
//     expert-aligned pieces and the same kernels run per piece, over the
//     work items of the experts that piece holds.
//
// Pipeline on device (no host round trip): router logits -> ps_moe_route_topk
// (softmax, top-k, renormalise) -> ps_moe_plan (group the T*k (token, slot)
// pairs by expert, tiles of <= 8 pairs) -> ps_moe_expert_gu (gate/up GEMV +
// SwiGLU per pair) -> ps_moe_expert_down -> ps_moe_combine (routing-weighted
// sum in fixed slot order: deterministic, no float atomics).
#include "common.cuh"
#include "../../include/pshard.h"

namespace ps {

constexpr int MOE_TILE = 8;     // pairs per work item
constexpr int MOE_WARPS = 8;
constexpr int MOE_ROWS = 2;     // rows per warp (one gate/up pair for stage A)

// ---- router: softmax over E, top-k (ties -> lower id), renormalise ----
__global__ void route_topk_kernel(const float* __restrict__ logits, int ldl, int T, int E, int k, int renorm,
                                  int* __restrict__ ids, float* __restrict__ w) {
  int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int lane = threadIdx.x & 31;
  if (t >= T) return;
  const float* row = logits + (long long)t * ldl;
  constexpr int MAXE = 256;
  float v[MAXE / 32];
  float mx = -INFINITY;
#pragma unroll
  for (int j = 0; j < MAXE / 32; ++j) {
    int e = lane + 32 * j;
    v[j] = e < E ? row[e] : -INFINITY;
    mx = fmaxf(mx, v[j]);
  }
  mx = warp_max(mx);
  float sum = 0.f;
#pragma unroll
  for (int j = 0; j < MAXE / 32; ++j) {
    int e = lane + 32 * j;
    v[j] = e < E ? __expf(v[j] - mx) : -1.f;   // probabilities are >= 0; -1 marks padding
    if (e < E) sum += v[j];
  }
  sum = warp_sum(sum);
  float inv = 1.f / sum;
  float picked_sum = 0.f;
  for (int r = 0; r < k; ++r) {
    float best = -2.f;
    int bi = 0x7fffffff;
#pragma unroll
    for (int j = 0; j < MAXE / 32; ++j) {
      int e = lane + 32 * j;
      if (v[j] > best || (v[j] == best && e < bi)) { best = v[j]; bi = e; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      float ob = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if ((bi & 31) == lane) v[bi >> 5] = -2.f;     // remove the winner
    float p = best * inv;
    picked_sum += p;
    if (lane == 0) { ids[t * k + r] = bi; w[t * k + r] = p; }
  }
  if (renorm) {
    __syncwarp();
    for (int r = lane; r < k; r += 32) w[t * k + r] = w[t * k + r] / picked_sum;
  }
}

// ---- plan: group pairs by expert; work items of <= MOE_TILE pairs ----
// layout of `plan` (ints): [0] n_items | [1 .. E+1] first_item per expert (E+1 entries)
//   | then items: (expert, start, count) * max_items | perm [P] | slot_of_pair [P]
__global__ void moe_plan_kernel(const int* __restrict__ ids, int P, int E, int max_items, int* __restrict__ plan) {
  extern __shared__ int sh[];
  int* count = sh;            // E
  int* offset = sh + E;       // E
  int* cursor = sh + 2 * E;   // E
  int* n_items_sh = sh + 3 * E;
  int* first = plan + 1;
  int* items = plan + 2 + E;
  int* perm = items + 3 * max_items;
  int* slot_of = perm + P;
  for (int e = threadIdx.x; e < E; e += blockDim.x) count[e] = 0;
  __syncthreads();
  for (int p = threadIdx.x; p < P; p += blockDim.x) atomicAdd(&count[ids[p]], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    int off = 0, it = 0;
    for (int e = 0; e < E; ++e) {
      offset[e] = off;
      cursor[e] = off;
      first[e] = it;
      for (int s = 0; s < count[e]; s += MOE_TILE) {
        items[3 * it] = e;
        items[3 * it + 1] = off + s;
        items[3 * it + 2] = min(MOE_TILE, count[e] - s);
        ++it;
      }
      off += count[e];
    }
    first[E] = it;
    *n_items_sh = it;
    plan[0] = it;
  }
  __syncthreads();
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    int pos = atomicAdd(&cursor[ids[p]], 1);
    perm[pos] = p;
    slot_of[p] = pos;
  }
}

__device__ __forceinline__ float load_x(const void* x, bool bf16, long long idx) {
  if (bf16) return __bfloat162float(static_cast<const __nv_bfloat16*>(x)[idx]);
  return static_cast<const float*>(x)[idx];
}

// Rows [row0, row0 + MOE_ROWS) of one expert matrix (row-major [rows x K] bf16) dotted
// with up to MOE_TILE activation rows; acc[r][i] per lane, reduced by the caller.
template <bool XBF16>
__device__ __forceinline__ void expert_dot(const __nv_bfloat16* __restrict__ Wm, int K, int row0, int nrows,
                                           const void* __restrict__ x, const long long* xoff, int n,
                                           float (&acc)[MOE_ROWS][MOE_TILE], int lane) {
#pragma unroll
  for (int r = 0; r < MOE_ROWS; ++r)
#pragma unroll
    for (int i = 0; i < MOE_TILE; ++i) acc[r][i] = 0.f;
  const __nv_bfloat16* wrow[MOE_ROWS];
#pragma unroll
  for (int r = 0; r < MOE_ROWS; ++r) wrow[r] = Wm + (long long)min(row0 + r, nrows - 1) * K;
  for (int k0 = lane * 8; k0 < K; k0 += 4 * 256) {
    uint4 wv[4][MOE_ROWS];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int r = 0; r < MOE_ROWS; ++r)
        wv[u][r] = (k0 + u * 256 < K) ? ld_stream(wrow[r] + k0 + u * 256) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int k = k0 + u * 256;
      if (k >= K) break;
#pragma unroll
      for (int i = 0; i < MOE_TILE; ++i) {
        if (i < n) {
          float xv[8];
          if (XBF16) {
            uint4 q = *reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(x) + xoff[i] + k);
            xv[0] = bf16_lo(q.x); xv[1] = bf16_hi(q.x); xv[2] = bf16_lo(q.y); xv[3] = bf16_hi(q.y);
            xv[4] = bf16_lo(q.z); xv[5] = bf16_hi(q.z); xv[6] = bf16_lo(q.w); xv[7] = bf16_hi(q.w);
          } else {
            const float4* xp = reinterpret_cast<const float4*>(static_cast<const float*>(x) + xoff[i] + k);
            float4 a = __ldg(xp), b = __ldg(xp + 1);
            xv[0] = a.x; xv[1] = a.y; xv[2] = a.z; xv[3] = a.w; xv[4] = b.x; xv[5] = b.y; xv[6] = b.z; xv[7] = b.w;
          }
#pragma unroll
          for (int r = 0; r < MOE_ROWS; ++r) {
            uint4 wq = wv[u][r];
            float s = acc[r][i];
            s = fmaf(xv[0], bf16_lo(wq.x), s); s = fmaf(xv[1], bf16_hi(wq.x), s);
            s = fmaf(xv[2], bf16_lo(wq.y), s); s = fmaf(xv[3], bf16_hi(wq.y), s);
            s = fmaf(xv[4], bf16_lo(wq.z), s); s = fmaf(xv[5], bf16_hi(wq.z), s);
            s = fmaf(xv[6], bf16_lo(wq.w), s); s = fmaf(xv[7], bf16_hi(wq.w), s);
            acc[r][i] = s;
          }
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < MOE_ROWS; ++r)
#pragma unroll
    for (int i = 0; i < MOE_TILE; ++i) acc[r][i] = warp_sum(acc[r][i]);
}

// Stage A: h[slot][j] = silu(x . Wg_e[j]) * (x . Wu_e[j]) for the pairs of each work item.
// Persistent CTAs walk units (item, row tile) over the item range [first[e_lo], first[e_hi]).
template <bool XBF16>
__global__ void __launch_bounds__(MOE_WARPS * 32)
expert_gu_kernel(const void* __restrict__ x, int ldx, const int* __restrict__ plan, int E, int P, int k,
                 int max_items, const unsigned char* __restrict__ expert_base, long long expert_stride,
                 long long gu_off, int eff, int d, float* __restrict__ h, int e_lo, int e_hi,
                 const int* __restrict__ slot_of_expert) {
  const int* first = plan + 1;
  const int* items = plan + 2 + E;
  const int* perm = items + 3 * max_items;
  const int it_lo = first[e_lo], it_hi = first[e_hi];
  const int rows = 2 * eff;
  const int rows_per_tile = MOE_WARPS * MOE_ROWS;
  const int tiles = (rows + rows_per_tile - 1) / rows_per_tile;
  const long long units = (long long)(it_hi - it_lo) * tiles;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (long long u = blockIdx.x; u < units; u += gridDim.x) {
    int it = it_lo + (int)(u / tiles);
    int tile = (int)(u % tiles);
    int e = items[3 * it], start = items[3 * it + 1], n = items[3 * it + 2];
    const long long slot = slot_of_expert ? slot_of_expert[e] : e;
    const __nv_bfloat16* Wg = reinterpret_cast<const __nv_bfloat16*>(expert_base + slot * expert_stride + gu_off);
    long long xoff[MOE_TILE];
#pragma unroll
    for (int i = 0; i < MOE_TILE; ++i) xoff[i] = (long long)(perm[start + min(i, n - 1)] / k) * ldx;
    int row0 = tile * rows_per_tile + warp * MOE_ROWS;
    float acc[MOE_ROWS][MOE_TILE];
    expert_dot<XBF16>(Wg, d, row0, rows, x, xoff, n, acc, lane);
    if (row0 + 1 < rows) {
#pragma unroll
      for (int i = 0; i < MOE_TILE; ++i)
        if (i < n && lane == i) h[(long long)(start + i) * eff + (row0 >> 1)] = silu(acc[0][i]) * acc[1][i];
    }
  }
}

// Stage B: out[slot][r] = h[slot] . Wd_e[r]
__global__ void __launch_bounds__(MOE_WARPS * 32)
expert_down_kernel(const float* __restrict__ h, const int* __restrict__ plan, int E, int max_items,
                   const unsigned char* __restrict__ expert_base, long long expert_stride, long long down_off,
                   int eff, int d, float* __restrict__ out, int e_lo, int e_hi,
                   const int* __restrict__ slot_of_expert) {
  const int* first = plan + 1;
  const int* items = plan + 2 + E;
  const int it_lo = first[e_lo], it_hi = first[e_hi];
  const int rows_per_tile = MOE_WARPS * MOE_ROWS;
  const int tiles = (d + rows_per_tile - 1) / rows_per_tile;
  const long long units = (long long)(it_hi - it_lo) * tiles;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (long long u = blockIdx.x; u < units; u += gridDim.x) {
    int it = it_lo + (int)(u / tiles);
    int tile = (int)(u % tiles);
    int e = items[3 * it], start = items[3 * it + 1], n = items[3 * it + 2];
    const long long slot = slot_of_expert ? slot_of_expert[e] : e;
    const __nv_bfloat16* Wd = reinterpret_cast<const __nv_bfloat16*>(expert_base + slot * expert_stride + down_off);
    long long xoff[MOE_TILE];
#pragma unroll
    for (int i = 0; i < MOE_TILE; ++i) xoff[i] = (long long)(start + min(i, n - 1)) * eff;
    int row0 = tile * rows_per_tile + warp * MOE_ROWS;
    float acc[MOE_ROWS][MOE_TILE];
    expert_dot<false>(Wd, eff, row0, d, h, xoff, n, acc, lane);
#pragma unroll
    for (int r = 0; r < MOE_ROWS; ++r)
      if (row0 + r < d) {
#pragma unroll
        for (int i = 0; i < MOE_TILE; ++i)
          if (i < n && lane == i) out[(long long)(start + i) * d + row0 + r] = acc[r][i];
      }
  }
}

// y[t] += sum_j w[t, j] * out[slot(t, j)], j in order (deterministic)
__global__ void moe_combine_kernel(const float* __restrict__ out, const int* __restrict__ plan, int E, int P,
                                   int max_items, const float* __restrict__ w, int k, int d, float* __restrict__ y,
                                   int ldy) {
  const int* slot_of = plan + 2 + E + 3 * max_items + P;
  int t = blockIdx.x;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    float s = 0.f;
    for (int j = 0; j < k; ++j) s += w[t * k + j] * out[(long long)slot_of[t * k + j] * d + i];
    y[(long long)t * ldy + i] += s;
  }
}

static int persistent_grid() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms * 4;
}

}  // namespace ps

using namespace ps;

extern "C" {

int ps_moe_route_topk(const float* logits, int ldl, int T, int E, int k, int renorm, int* ids, float* w,
                      void* stream) {
  PS_REQUIRE(E <= 256 && k <= E && k >= 1, "ps_moe_route_topk: E=%d k=%d unsupported", E, k);
  if (T <= 0) return PS_OK;
  int warps = 8;
  route_topk_kernel<<<(T + warps - 1) / warps, warps * 32, 0, (cudaStream_t)stream>>>(logits, ldl, T, E, k,
                                                                                      renorm, ids, w);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

int ps_moe_plan_ints(int P, int E, long long* n_ints) {
  int max_items = P / MOE_TILE + E;
  *n_ints = 2 + E + 3LL * max_items + 2LL * P;
  return PS_OK;
}

int ps_moe_plan(const int* ids, int P, int E, int* plan, void* stream) {
  PS_REQUIRE(P >= 1 && E >= 1 && E <= 1024, "ps_moe_plan: P=%d E=%d", P, E);
  int max_items = P / MOE_TILE + E;
  moe_plan_kernel<<<1, 1024, (3 * E + 1) * sizeof(int), (cudaStream_t)stream>>>(ids, P, E, max_items, plan);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

int ps_moe_expert_gu_mapped(const void* x, int ldx, int x_bf16, const int* plan, int E, int P, int k,
                            const void* expert_base, long long expert_stride, long long gu_off, int eff, int d,
                            float* h, int e_lo, int e_hi, const int* slot_of_expert, void* stream) {
  PS_REQUIRE(d % 8 == 0 && eff % 8 == 0, "ps_moe_expert_gu: d, eff must be multiples of 8");
  int max_items = P / MOE_TILE + E;
  auto base = static_cast<const unsigned char*>(expert_base);
  if (x_bf16)
    expert_gu_kernel<true><<<persistent_grid(), MOE_WARPS * 32, 0, (cudaStream_t)stream>>>(
        x, ldx, plan, E, P, k, max_items, base, expert_stride, gu_off, eff, d, h, e_lo, e_hi, slot_of_expert);
  else
    expert_gu_kernel<false><<<persistent_grid(), MOE_WARPS * 32, 0, (cudaStream_t)stream>>>(
        x, ldx, plan, E, P, k, max_items, base, expert_stride, gu_off, eff, d, h, e_lo, e_hi, slot_of_expert);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

int ps_moe_expert_gu(const void* x, int ldx, int x_bf16, const int* plan, int E, int P, int k,
                     const void* expert_base, long long expert_stride, long long gu_off, int eff, int d,
                     float* h, int e_lo, int e_hi, void* stream) {
  return ps_moe_expert_gu_mapped(x, ldx, x_bf16, plan, E, P, k, expert_base, expert_stride, gu_off, eff, d, h,
                                 e_lo, e_hi, nullptr, stream);
}

int ps_moe_expert_down_mapped(const float* h, const int* plan, int E, int P, const void* expert_base,
                              long long expert_stride, long long down_off, int eff, int d, float* out, int e_lo,
                              int e_hi, const int* slot_of_expert, void* stream) {
  int max_items = P / MOE_TILE + E;
  expert_down_kernel<<<persistent_grid(), MOE_WARPS * 32, 0, (cudaStream_t)stream>>>(
      h, plan, E, max_items, static_cast<const unsigned char*>(expert_base), expert_stride, down_off, eff, d, out,
      e_lo, e_hi, slot_of_expert);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

int ps_moe_expert_down(const float* h, const int* plan, int E, int P, const void* expert_base,
                       long long expert_stride, long long down_off, int eff, int d, float* out, int e_lo,
                       int e_hi, void* stream) {
  return ps_moe_expert_down_mapped(h, plan, E, P, expert_base, expert_stride, down_off, eff, d, out, e_lo, e_hi,
                                   nullptr, stream);
}

int ps_moe_combine(const float* out, const int* plan, int E, int P, const float* w, int T, int k, int d,
                   float* y, int ldy, void* stream) {
  int max_items = P / MOE_TILE + E;
  if (T <= 0) return PS_OK;
  moe_combine_kernel<<<T, 256, 0, (cudaStream_t)stream>>>(out, plan, E, P, max_items, w, k, d, y, ldy);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

}  // extern "C"

int ps_preload_moe() {
  using namespace ps;
  int n = 0;
  touch_kernel(route_topk_kernel, n);
  touch_kernel(moe_plan_kernel, n);
  touch_kernel(expert_gu_kernel<true>, n);
  touch_kernel(expert_gu_kernel<false>, n);
  touch_kernel(expert_down_kernel, n);
  touch_kernel(moe_combine_kernel, n);
  return n;
}
