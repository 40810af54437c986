// K1 / K8: decode GEMV and skinny GEMM, bf16 weights x fp32 activations.
//
// Prices: MATMUL requests of the attention projection, FFN and output head
// (`pkg/src/shardplan/model_graph.py:147-153,173-179,202-209`) at t <= 32
// new tokens. y[t, n] = sum_k x[t, k] * W[n, k], W row-major [N x K] bf16,
// fp32 accumulation. HBM-bound on resident or ring-staged weights: every
// weight byte is read exactly once with 128-bit non-allocating loads.
//
// Work decomposition: a CTA of 8 warps owns tiles of rows; inside a tile
// the 8 warps form (8 / KSPLIT) row groups of ROWS rows, and the KSPLIT
// warps of a group split K (partials reduced through shared memory). The
// host picks KSPLIT so one launch puts enough 16-byte loads in flight to
// cover HBM latency even for the ~50 MB ring pieces of a decode pass, and
// sizes the grid to the resident-CTA capacity (148 SMs x 6), looping over
// tiles (grid-stride) so warps do not retire after one short burst.
// ps_gemv_bf16 itself dispatches to the bulk-copy kernel (gemv_tma.cu) for device and
// host-mapped (K8, zero-copy) weights alike; this register-burst kernel stays reachable
// through ps_gemv_bf16_cfg (rows 2 | 4) as the test and tuning baseline.
//
// Epilogues: STORE (y = acc), ACCUM (y += acc, fused residual add),
// SWIGLU (rows interleaved gate/up: y[t, j] = silu(acc[2j]) * acc[2j+1]).
#include "common.cuh"
#include "../../include/pshard.h"

namespace ps {

constexpr int GEMV_WARPS = 8;

template <int T, int ROWS, int KSPLIT, int EPI>
__global__ void __launch_bounds__(GEMV_WARPS * 32)
gemv_bf16_kernel(const float* __restrict__ x, int ldx, int tt, const __nv_bfloat16* __restrict__ W,
                 int N, int K, long long ldw, int kpart, float* __restrict__ y, int ldy) {
  pdl_trigger();
  pdl_wait();
  constexpr int GROUPS = GEMV_WARPS / KSPLIT;
  constexpr int UNROLL = (T == 1) ? 8 : (T <= 4 ? 4 : 2);   // 16-byte loads in flight per row
  constexpr int STEP = 256;  // 32 lanes x 8 bf16
  __shared__ float part[GEMV_WARPS][ROWS * T];

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int grp = warp / KSPLIT, kp = warp - grp * KSPLIT;
  const int k_begin = kp * kpart;
  const int k_end = min(K, k_begin + kpart);
  const int rows_per_tile = GROUPS * ROWS;
  const int n_tiles = (N + rows_per_tile - 1) / rows_per_tile;

  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int row0 = tile * rows_per_tile + grp * ROWS;
    float acc[ROWS][T];
#pragma unroll
    for (int r = 0; r < ROWS; ++r)
#pragma unroll
      for (int t = 0; t < T; ++t) acc[r][t] = 0.f;
    const __nv_bfloat16* wrow[ROWS];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) wrow[r] = W + (long long)min(row0 + r, N - 1) * ldw;

    // bursts of UNROLL steps: all loads of a burst are issued (predicated) before use
    for (int kb = k_begin + lane * 8; kb < k_end; kb += UNROLL * STEP) {
      uint4 wv[UNROLL][ROWS];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u)
#pragma unroll
        for (int r = 0; r < ROWS; ++r)
          wv[u][r] = (kb + u * STEP < k_end) ? ld_stream(wrow[r] + kb + u * STEP) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const int k = kb + u * STEP;
        if (k >= k_end) break;
#pragma unroll
        for (int t = 0; t < T; ++t) {
          if (t < tt) {
            const float4* xp = reinterpret_cast<const float4*>(x + (long long)t * ldx + k);
            float4 a = __ldg(xp), b = __ldg(xp + 1);
#pragma unroll
            for (int r = 0; r < ROWS; ++r) {
              uint4 w = wv[u][r];
              float s = acc[r][t];
              s = fmaf(a.x, bf16_lo(w.x), s); s = fmaf(a.y, bf16_hi(w.x), s);
              s = fmaf(a.z, bf16_lo(w.y), s); s = fmaf(a.w, bf16_hi(w.y), s);
              s = fmaf(b.x, bf16_lo(w.z), s); s = fmaf(b.y, bf16_hi(w.z), s);
              s = fmaf(b.z, bf16_lo(w.w), s); s = fmaf(b.w, bf16_hi(w.w), s);
              acc[r][t] = s;
            }
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < ROWS; ++r)
#pragma unroll
      for (int t = 0; t < T; ++t) acc[r][t] = warp_sum(acc[r][t]);

    if (KSPLIT > 1) {
      if (lane == 0) {
#pragma unroll
        for (int r = 0; r < ROWS; ++r)
#pragma unroll
          for (int t = 0; t < T; ++t) part[warp][r * T + t] = acc[r][t];
      }
      __syncthreads();
      if (kp == 0) {
#pragma unroll
        for (int r = 0; r < ROWS; ++r)
#pragma unroll
          for (int t = 0; t < T; ++t) {
            float s = 0.f;
#pragma unroll
            for (int j = 0; j < KSPLIT; ++j) s += part[warp + j][r * T + t];
            acc[r][t] = s;
          }
      }
    }
    if (kp == 0) {
      if (EPI == PS_EPI_SWIGLU) {
#pragma unroll
        for (int r = 0; r < ROWS; r += 2) {
          if (row0 + r + 1 < N) {
#pragma unroll
            for (int t = 0; t < T; ++t)
              if (t < tt && lane == t) y[(long long)t * ldy + ((row0 + r) >> 1)] = silu(acc[r][t]) * acc[r + 1][t];
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
          if (row0 + r < N) {
#pragma unroll
            for (int t = 0; t < T; ++t) {
              if (t < tt && lane == t) {
                float* dst = y + (long long)t * ldy + row0 + r;
                if (EPI == PS_EPI_ACCUM) *dst += acc[r][t];
                else *dst = acc[r][t];
              }
            }
          }
        }
      }
    }
    if (KSPLIT > 1) __syncthreads();  // part[] is reused by the next tile
  }
}

static int g_sm_count = 0;

static int sm_count() {
  if (!g_sm_count) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, dev);
    if (g_sm_count <= 0) g_sm_count = 148;
  }
  return g_sm_count;
}

// Grid = min(tiles, resident CTA capacity of this instantiation): every CTA is
// resident from the start, so the grid-stride tile loop has no second wave.
template <int T, int ROWS, int KSPLIT, int EPI>
static void launch4(int n_tiles, int grid_cap, cudaStream_t s, const float* x, int ldx, int tt,
                    const __nv_bfloat16* W, int N, int K, long long ldw, int kpart, float* y, int ldy) {
  static int per_sm = 0;
  if (!per_sm) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gemv_bf16_kernel<T, ROWS, KSPLIT, EPI>,
                                                  GEMV_WARPS * 32, 0);
    if (per_sm <= 0) per_sm = 1;
  }
  int cap = grid_cap > 0 ? grid_cap : per_sm * sm_count();
  dim3 grid(n_tiles < cap ? n_tiles : cap);
  launch_k(gemv_bf16_kernel<T, ROWS, KSPLIT, EPI>, grid, GEMV_WARPS * 32, 0, s, x, ldx, tt, W, N, K, ldw, kpart, y,
           ldy);
}

template <int T, int ROWS, int KSPLIT>
static void launch3(int epi, int n_tiles, int grid_cap, cudaStream_t s, const float* x, int ldx, int tt,
                    const __nv_bfloat16* W, int N, int K, long long ldw, int kpart, float* y, int ldy) {
  if (epi == PS_EPI_STORE)
    launch4<T, ROWS, KSPLIT, PS_EPI_STORE>(n_tiles, grid_cap, s, x, ldx, tt, W, N, K, ldw, kpart, y, ldy);
  else if (epi == PS_EPI_ACCUM)
    launch4<T, ROWS, KSPLIT, PS_EPI_ACCUM>(n_tiles, grid_cap, s, x, ldx, tt, W, N, K, ldw, kpart, y, ldy);
  else
    launch4<T, ROWS, KSPLIT, PS_EPI_SWIGLU>(n_tiles, grid_cap, s, x, ldx, tt, W, N, K, ldw, kpart, y, ldy);
}

template <int T, int ROWS>
static void launch_ks(int ksplit, int epi, int n_tiles, int grid_cap, cudaStream_t s, const float* x, int ldx,
                      int tt, const __nv_bfloat16* W, int N, int K, long long ldw, int kpart, float* y, int ldy) {
  switch (ksplit) {
    case 1: launch3<T, ROWS, 1>(epi, n_tiles, grid_cap, s, x, ldx, tt, W, N, K, ldw, kpart, y, ldy); break;
    case 2: launch3<T, ROWS, 2>(epi, n_tiles, grid_cap, s, x, ldx, tt, W, N, K, ldw, kpart, y, ldy); break;
    case 4: launch3<T, ROWS, 4>(epi, n_tiles, grid_cap, s, x, ldx, tt, W, N, K, ldw, kpart, y, ldy); break;
    default: launch3<T, ROWS, 8>(epi, n_tiles, grid_cap, s, x, ldx, tt, W, N, K, ldw, kpart, y, ldy); break;
  }
}

// One launch for tt <= 8 tokens; rows/ksplit/grid chosen (or forced for tuning).
static int gemv_launch(const float* x, int ldx, int tt, const __nv_bfloat16* W, int N, int K, long long ldw,
                       float* y, int ldy, int epi, cudaStream_t s, int rows, int ksplit, int grid_cap) {
  const int ROWS = 2;
  if (rows != 2 && rows != 4) rows = ROWS;
  if (tt > 1) rows = 2;
  if (ksplit <= 0) {
    // enough warps to fill every SM (64 resident), keeping >= 512 columns per warp
    long long want = (long long)sm_count() * 64;
    long long row_groups = (N + rows - 1) / rows;
    ksplit = 1;
    while (ksplit < 8 && row_groups * ksplit < want && K / (ksplit * 2) >= 256) ksplit *= 2;
  }
  int kpart = ((K + ksplit - 1) / ksplit + 255) / 256 * 256;
  int rows_per_tile = (GEMV_WARPS / ksplit) * rows;
  int n_tiles = (N + rows_per_tile - 1) / rows_per_tile;
  if (tt == 1) {
    if (rows == 4) launch_ks<1, 4>(ksplit, epi, n_tiles, grid_cap, s, x, ldx, tt, W, N, K, ldw, kpart, y, ldy);
    else launch_ks<1, 2>(ksplit, epi, n_tiles, grid_cap, s, x, ldx, tt, W, N, K, ldw, kpart, y, ldy);
  } else if (tt == 2) {
    launch_ks<2, 2>(ksplit, epi, n_tiles, grid_cap, s, x, ldx, tt, W, N, K, ldw, kpart, y, ldy);
  } else if (tt <= 4) {
    launch_ks<4, 2>(ksplit, epi, n_tiles, grid_cap, s, x, ldx, tt, W, N, K, ldw, kpart, y, ldy);
  } else {
    launch_ks<8, 2>(ksplit, epi, n_tiles, grid_cap, s, x, ldx, tt, W, N, K, ldw, kpart, y, ldy);
  }
  PS_CHECK_LAUNCH();
  return PS_OK;
}

int gemv_tma_launch(const float* x, int ldx, int tt, const __nv_bfloat16* W, int N, int K, long long ldw, float* y,
                    int ldy, int epi, cudaStream_t s, int grid_cap);

// rows == 0 selects the bulk-copy kernel (gemv_tma.cu) for device-resident and host-mapped
// (zero-copy, K8) weights; rows = 2 | 4 use the register-burst kernel below.
static int gemv_checked(const float* x, int ldx, int t, const void* W, int N, int K, long long ldw, float* y,
                        int ldy, int epilogue, void* stream, int rows, int ksplit, int grid_cap) {
  PS_REQUIRE(t >= 1 && t <= 32, "ps_gemv_bf16: t=%d outside [1, 32]", t);
  PS_REQUIRE(K % 8 == 0 && ldw % 8 == 0 && ldx % 4 == 0, "ps_gemv_bf16: K/ldw must be multiples of 8, ldx of 4");
  PS_REQUIRE(((uintptr_t)W & 15) == 0 && ((uintptr_t)x & 15) == 0, "ps_gemv_bf16: W and x must be 16-byte aligned");
  PS_REQUIRE(epilogue == PS_EPI_STORE || epilogue == PS_EPI_ACCUM || epilogue == PS_EPI_SWIGLU,
             "ps_gemv_bf16: unsupported epilogue %d", epilogue);
  PS_REQUIRE(epilogue != PS_EPI_SWIGLU || N % 2 == 0, "ps_gemv_bf16: SWIGLU needs an even N");
  if (N <= 0) return PS_OK;
  auto Wb = static_cast<const __nv_bfloat16*>(W);
  cudaStream_t s = (cudaStream_t)stream;
  for (int t0 = 0; t0 < t; t0 += 8) {  // tokens in chunks of 8 (W re-read per chunk)
    int tt = t - t0 < 8 ? t - t0 : 8;
    // rows 0 (ps_gemv_bf16): the bulk-copy kernel, device or host-mapped weights alike, so a
    // zero-copy shard gives bit-identical outputs to its exponent-coded twin (ps_gemv_bf16c,
    // same decomposition) and to a VRAM copy; SM reads of host memory cap at ~50 GB/s
    // whatever the kernel. rows 2 | 4: the register-burst kernel (tests).
    if (rows == 0 || rows == -1) {
      int rc = gemv_tma_launch(x + (long long)t0 * ldx, ldx, tt, Wb, N, K, ldw, y + (long long)t0 * ldy, ldy,
                               epilogue, s, grid_cap);
      if (rc) return rc;
      continue;
    }
    int rc = gemv_launch(x + (long long)t0 * ldx, ldx, tt, Wb, N, K, ldw, y + (long long)t0 * ldy, ldy, epilogue,
                         s, rows, ksplit, grid_cap);
    if (rc) return rc;
  }
  return PS_OK;
}

}  // namespace ps

extern "C" int ps_gemv_bf16(const float* x, int ldx, int t, const void* W, int N, int K, long long ldw,
                            float* y, int ldy, int epilogue, void* stream) {
  return ps::gemv_checked(x, ldx, t, W, N, K, ldw, y, ldy, epilogue, stream, 0, 0, 0);
}

extern "C" int ps_gemv_bf16_cfg(const float* x, int ldx, int t, const void* W, int N, int K, long long ldw,
                                float* y, int ldy, int epilogue, void* stream, int rows, int ksplit,
                                int grid_cap) {
  return ps::gemv_checked(x, ldx, t, W, N, K, ldw, y, ldy, epilogue, stream, rows, ksplit, grid_cap);
}

int ps_preload_gemv() {
  using namespace ps;
  int n = 0;
#define PS_T4(T, R, K)                                         \
  touch_kernel(gemv_bf16_kernel<T, R, K, PS_EPI_STORE>, n);    \
  touch_kernel(gemv_bf16_kernel<T, R, K, PS_EPI_ACCUM>, n);    \
  touch_kernel(gemv_bf16_kernel<T, R, K, PS_EPI_SWIGLU>, n);
#define PS_TK(T, R) PS_T4(T, R, 1) PS_T4(T, R, 2) PS_T4(T, R, 4) PS_T4(T, R, 8)
  PS_TK(1, 4) PS_TK(1, 2) PS_TK(2, 2) PS_TK(4, 2) PS_TK(8, 2)
#undef PS_TK
#undef PS_T4
  return n;
}
