// K1 / K8: decode GEMV and skinny GEMM, bf16 weights x fp32 activations.
//
// Prices: MATMUL requests of the attention projection, FFN and output head
// (`pkg/src/shardplan/model_graph.py:147-153,173-179,202-209`) at t <= 32
// new tokens. y[t, n] = sum_k x[t, k] * W[n, k], W row-major [N x K] bf16,
// fp32 accumulation. HBM-bound on resident or ring-staged weights: every
// weight byte is read exactly once with 128-bit non-allocating loads, each
// lane keeping UNROLL x ROWS loads in flight, and each warp reduces its
// rows with shuffles. The same kernel reads host-mapped weights (K8,
// zero-copy over PCIe) when W points into cudaHostAllocMapped memory.
//
// Epilogues: STORE (y = acc), ACCUM (y += acc, fused residual add),
// SWIGLU (rows interleaved gate/up: y[t, j] = silu(acc[2j]) * acc[2j+1]).
#include "common.cuh"
#include "../../include/pshard.h"

namespace ps {

constexpr int GEMV_WARPS = 8;

template <int T, int ROWS, int EPI>
__global__ void __launch_bounds__(GEMV_WARPS * 32)
gemv_bf16_kernel(const float* __restrict__ x, int ldx, const __nv_bfloat16* __restrict__ W,
                 int N, int K, long long ldw, float* __restrict__ y, int ldy) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int row0 = (blockIdx.x * GEMV_WARPS + warp) * ROWS;
  if (row0 >= N) return;

  float acc[ROWS][T];
#pragma unroll
  for (int r = 0; r < ROWS; ++r)
#pragma unroll
    for (int t = 0; t < T; ++t) acc[r][t] = 0.f;

  const __nv_bfloat16* wrow[ROWS];
#pragma unroll
  for (int r = 0; r < ROWS; ++r) {
    int rr = row0 + r < N ? row0 + r : N - 1;  // clamp; result discarded
    wrow[r] = W + (long long)rr * ldw;
  }

  constexpr int UNROLL = (T <= 2) ? 4 : 2;
  constexpr int STEP = 256;  // 32 lanes x 8 bf16
  int k = lane * 8;
  // main body: UNROLL steps per iteration, all weight loads issued first
  for (; k + (UNROLL - 1) * STEP < K; k += UNROLL * STEP) {
    uint4 wv[UNROLL][ROWS];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u)
#pragma unroll
      for (int r = 0; r < ROWS; ++r) wv[u][r] = ld_stream(wrow[r] + k + u * STEP);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const float4* xp = reinterpret_cast<const float4*>(x + (long long)t * ldx + k + u * STEP);
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
  // tail: single steps (K is a multiple of 8)
  for (; k < K; k += STEP) {
    uint4 wv[ROWS];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) wv[r] = ld_stream(wrow[r] + k);
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const float4* xp = reinterpret_cast<const float4*>(x + (long long)t * ldx + k);
      float4 a = __ldg(xp), b = __ldg(xp + 1);
#pragma unroll
      for (int r = 0; r < ROWS; ++r) {
        uint4 w = wv[r];
        float s = acc[r][t];
        s = fmaf(a.x, bf16_lo(w.x), s); s = fmaf(a.y, bf16_hi(w.x), s);
        s = fmaf(a.z, bf16_lo(w.y), s); s = fmaf(a.w, bf16_hi(w.y), s);
        s = fmaf(b.x, bf16_lo(w.z), s); s = fmaf(b.y, bf16_hi(w.z), s);
        s = fmaf(b.z, bf16_lo(w.w), s); s = fmaf(b.w, bf16_hi(w.w), s);
        acc[r][t] = s;
      }
    }
  }

#pragma unroll
  for (int r = 0; r < ROWS; ++r)
#pragma unroll
    for (int t = 0; t < T; ++t) acc[r][t] = warp_sum(acc[r][t]);

  // lanes t < T write token t (spreads the stores over lanes)
  if (EPI == PS_EPI_SWIGLU) {
#pragma unroll
    for (int r = 0; r < ROWS; r += 2) {
      int j = (row0 + r) >> 1;
      if (row0 + r + 1 < N) {
#pragma unroll
        for (int t = 0; t < T; ++t)
          if (lane == (t & 31)) y[(long long)t * ldy + j] = silu(acc[r][t]) * acc[r + 1][t];
      }
    }
  } else {
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      if (row0 + r < N) {
#pragma unroll
        for (int t = 0; t < T; ++t) {
          if (lane == (t & 31)) {
            float* dst = y + (long long)t * ldy + row0 + r;
            if (EPI == PS_EPI_ACCUM) *dst += acc[r][t];
            else *dst = acc[r][t];
          }
        }
      }
    }
  }
}

template <int T, int ROWS>
static int launch_gemv(const float* x, int ldx, const __nv_bfloat16* W, int N, int K,
                       long long ldw, float* y, int ldy, int epi, cudaStream_t s) {
  int rows_per_block = GEMV_WARPS * ROWS;
  dim3 grid((N + rows_per_block - 1) / rows_per_block);
  dim3 block(GEMV_WARPS * 32);
  switch (epi) {
    case PS_EPI_STORE:
      gemv_bf16_kernel<T, ROWS, PS_EPI_STORE><<<grid, block, 0, s>>>(x, ldx, W, N, K, ldw, y, ldy);
      break;
    case PS_EPI_ACCUM:
      gemv_bf16_kernel<T, ROWS, PS_EPI_ACCUM><<<grid, block, 0, s>>>(x, ldx, W, N, K, ldw, y, ldy);
      break;
    case PS_EPI_SWIGLU:
      gemv_bf16_kernel<T, ROWS, PS_EPI_SWIGLU><<<grid, block, 0, s>>>(x, ldx, W, N, K, ldw, y, ldy);
      break;
    default:
      ps_set_error("ps_gemv_bf16: unsupported epilogue %d", epi);
      return PS_ERR_ARG;
  }
  PS_CHECK_LAUNCH();
  return PS_OK;
}

}  // namespace ps

extern "C" int ps_gemv_bf16(const float* x, int ldx, int t, const void* W, int N, int K,
                            long long ldw, float* y, int ldy, int epilogue, void* stream) {
  using namespace ps;
  PS_REQUIRE(t >= 1 && t <= 32, "ps_gemv_bf16: t=%d outside [1, 32]", t);
  PS_REQUIRE(K % 8 == 0 && ldw % 8 == 0 && ldx % 4 == 0, "ps_gemv_bf16: K/ldw must be multiples of 8, ldx of 4");
  PS_REQUIRE(((uintptr_t)W & 15) == 0 && ((uintptr_t)x & 15) == 0, "ps_gemv_bf16: W and x must be 16-byte aligned");
  PS_REQUIRE(epilogue != PS_EPI_SWIGLU || N % 2 == 0, "ps_gemv_bf16: SWIGLU needs an even N");
  if (N <= 0) return PS_OK;
  auto Wb = static_cast<const __nv_bfloat16*>(W);
  cudaStream_t s = (cudaStream_t)stream;
  int rc;
  if (t == 1) rc = launch_gemv<1, 2>(x, ldx, Wb, N, K, ldw, y, ldy, epilogue, s);
  else if (t == 2) rc = launch_gemv<2, 2>(x, ldx, Wb, N, K, ldw, y, ldy, epilogue, s);
  else if (t <= 4) {
    // pad to 4 rows by launching per exact size class
    if (t == 4) rc = launch_gemv<4, 2>(x, ldx, Wb, N, K, ldw, y, ldy, epilogue, s);
    else rc = launch_gemv<3, 2>(x, ldx, Wb, N, K, ldw, y, ldy, epilogue, s);
  } else {
    // t in (4, 32]: chunks of 8 tokens
    rc = PS_OK;
    for (int t0 = 0; t0 < t && rc == PS_OK; t0 += 8) {
      int tt = t - t0 < 8 ? t - t0 : 8;
      const float* xs = x + (long long)t0 * ldx;
      float* ys = y + (long long)t0 * ldy;
      switch (tt) {
        case 8: rc = launch_gemv<8, 2>(xs, ldx, Wb, N, K, ldw, ys, ldy, epilogue, s); break;
        case 7: rc = launch_gemv<7, 2>(xs, ldx, Wb, N, K, ldw, ys, ldy, epilogue, s); break;
        case 6: rc = launch_gemv<6, 2>(xs, ldx, Wb, N, K, ldw, ys, ldy, epilogue, s); break;
        case 5: rc = launch_gemv<5, 2>(xs, ldx, Wb, N, K, ldw, ys, ldy, epilogue, s); break;
        case 4: rc = launch_gemv<4, 2>(xs, ldx, Wb, N, K, ldw, ys, ldy, epilogue, s); break;
        case 3: rc = launch_gemv<3, 2>(xs, ldx, Wb, N, K, ldw, ys, ldy, epilogue, s); break;
        case 2: rc = launch_gemv<2, 2>(xs, ldx, Wb, N, K, ldw, ys, ldy, epilogue, s); break;
        default: rc = launch_gemv<1, 2>(xs, ldx, Wb, N, K, ldw, ys, ldy, epilogue, s); break;
      }
    }
  }
  return rc;
}
