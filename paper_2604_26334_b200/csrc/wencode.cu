// GPU encoder of the exponent-coded weight rows (format: runtime/wcomp.py, decoded by
// wcodec.cuh). Byte-identical to wcomp.encode, which stays the CPU reference; model load
// encodes on the GPU (one H2D of the bf16 matrix, two kernels, one D2H of the coded rows)
// instead of ~20 s of numpy for Llama-3.1-8B, and a model whose bf16 and coded host copies
// do not fit host memory together (Llama-3.3-70B on a 196 GB box) is generated and coded
// on the GPU without ever holding its bf16 blob on the host.
//
//   ps_wencode_stats: per row, the window base (the 15 exponents below the row's largest;
//                     a row escaping more than 8 weights that way takes the 15-wide window
//                     covering the most weights, ties to the highest) and its escape count
//   ps_wencode_rows:  sign|mantissa bytes, 4-bit codes (low nibble = even column), and the
//                     trailer [base | n << 8, (col << 8 | exp) ascending, 0xFFFFFFFF ...]
//
// One CTA per row; thread i of n owns the contiguous columns [i * K / n, (i + 1) * K / n),
// so a scan of per-thread escape counts places every escape at its ascending-column
// slot. Bound: HBM (K*2 in, K*1.5 + trailer out per row), far from the host link.
#include "common.cuh"
#include "../../include/pshard.h"

namespace ps {

constexpr int WE_THREADS = 256;
constexpr int WE_RECHECK = 8;     // wcomp.row_bases(recheck=8)

__device__ __forceinline__ int we_exp(uint16_t b) { return (b >> 7) & 0xFF; }

// block-wide sum / max over WE_THREADS threads (warp shuffles + one smem round)
template <bool MAX>
__device__ __forceinline__ int we_reduce(int v, int* red) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const int u = __shfl_xor_sync(0xffffffffu, v, o);
    v = MAX ? max(v, u) : v + u;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  v = lane < WE_THREADS / 32 ? red[lane] : (MAX ? 0 : 0);
#pragma unroll
  for (int o = 4; o >= 1; o >>= 1) {
    const int u = __shfl_xor_sync(0xffffffffu, v, o);
    v = MAX ? max(v, u) : v + u;
  }
  return __shfl_sync(0xffffffffu, v, 0);
}

__global__ void __launch_bounds__(WE_THREADS)
wencode_stats_kernel(const uint16_t* __restrict__ bits, int K, long long ld, int* __restrict__ base_out,
                     int* __restrict__ count_out) {
  __shared__ int red[WE_THREADS / 32];
  __shared__ int hist[256];
  const uint16_t* row = bits + blockIdx.x * ld;
  int mx = 0;
  for (int c = threadIdx.x; c < K; c += WE_THREADS) mx = max(mx, we_exp(row[c]));
  mx = we_reduce<true>(mx, red);
  int base = max(0, mx - 14);
  int low = 0;
  for (int c = threadIdx.x; c < K; c += WE_THREADS) low += we_exp(row[c]) < base;
  low = we_reduce<false>(low, red);
  if (low > WE_RECHECK) {   // an outlier far above the bulk: the best-covering window
    hist[threadIdx.x] = 0;
    __syncthreads();
    for (int c = threadIdx.x; c < K; c += WE_THREADS) atomicAdd(&hist[we_exp(row[c])], 1);
    __syncthreads();
    // cover[b] = hist[b .. b+14], b in [0, 241]; argmax, ties to the highest b
    int best = -1, best_b = 0;
    const int b = threadIdx.x;
    if (b <= 241) {
      int cov = 0;
      for (int i = 0; i < 15; ++i) cov += hist[b + i];
      best = cov;
      best_b = b;
    }
    // pack (cover, b) so that max picks the larger cover, then the larger b
    int key = best < 0 ? -1 : (best << 8) | best_b;
    key = we_reduce<true>(key, red);
    base = key & 0xFF;
  }
  int esc = 0;
  for (int c = threadIdx.x; c < K; c += WE_THREADS) {
    const int e = we_exp(row[c]) - base;
    esc += (e < 0) | (e > 14);
  }
  esc = we_reduce<false>(esc, red);
  if (threadIdx.x == 0) {
    base_out[blockIdx.x] = base;
    count_out[blockIdx.x] = esc;
  }
}

// blockDim.x threads (256, or 128 when K / 256 is odd) so each thread owns an even number
// of columns: a code byte (two nibbles) never straddles two threads
__global__ void __launch_bounds__(WE_THREADS)
wencode_rows_kernel(const uint16_t* __restrict__ bits, int K, long long ld, const int* __restrict__ base_in,
                    int tb, uint8_t* __restrict__ out, long long ld_out) {
  __shared__ int scan[WE_THREADS];
  const int nt = blockDim.x;
  const uint16_t* row = bits + blockIdx.x * ld;
  uint8_t* o = out + blockIdx.x * ld_out;
  const int base = base_in[blockIdx.x];
  const int per = K / nt;
  const int c0 = threadIdx.x * per;
  int mine = 0;
  for (int c = c0; c < c0 + per; c += 2) {
    const uint16_t a = row[c], b = row[c + 1];
    const int ea = we_exp(a) - base, eb = we_exp(b) - base;
    const bool xa = ea < 0 || ea > 14, xb = eb < 0 || eb > 14;
    mine += xa + xb;
    o[c] = (uint8_t)(((a >> 8) & 0x80) | (a & 0x7F));
    o[c + 1] = (uint8_t)(((b >> 8) & 0x80) | (b & 0x7F));
    o[K + c / 2] = (uint8_t)((xa ? 15 : ea) | ((xb ? 15 : eb) << 4));
  }
  // inclusive scan of the escape counts in thread (= column) order
  scan[threadIdx.x] = mine;
  __syncthreads();
  for (int off = 1; off < nt; off <<= 1) {
    const int v = threadIdx.x >= off ? scan[threadIdx.x - off] : 0;
    __syncthreads();
    scan[threadIdx.x] += v;
    __syncthreads();
  }
  const int total = scan[nt - 1];
  int slot = 1 + scan[threadIdx.x] - mine;
  uint32_t* tr = reinterpret_cast<uint32_t*>(o + (long long)K * 3 / 2);
  if (mine) {
    for (int c = c0; c < c0 + per; ++c) {
      const int e = we_exp(row[c]);
      if (e - base < 0 || e - base > 14) tr[slot++] = ((uint32_t)c << 8) | (uint32_t)e;
    }
  }
  for (int w = 1 + total + threadIdx.x; w < tb / 4; w += nt) tr[w] = 0xFFFFFFFFu;
  if (threadIdx.x == 0) tr[0] = (uint32_t)base | ((uint32_t)total << 8);
}

}  // namespace ps

extern "C" int ps_wencode_stats(const void* bits, int N, int K, long long ld, int* base_out, int* count_out,
                                void* stream) {
  using namespace ps;
  PS_REQUIRE(K > 0 && K % 256 == 0 && ld >= K, "ps_wencode_stats: K %d (multiple of 256), ld %lld", K, ld);
  if (N <= 0) return PS_OK;
  wencode_stats_kernel<<<N, WE_THREADS, 0, (cudaStream_t)stream>>>(static_cast<const uint16_t*>(bits), K, ld,
                                                                   base_out, count_out);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

extern "C" int ps_wencode_rows(const void* bits, int N, int K, long long ld, const int* base, int trailer_bytes,
                               void* out, long long ld_out, void* stream) {
  using namespace ps;
  PS_REQUIRE(K > 0 && K % 256 == 0 && ld >= K, "ps_wencode_rows: K %d (multiple of 256), ld %lld", K, ld);
  PS_REQUIRE(trailer_bytes >= 16 && trailer_bytes % 16 == 0 && ld_out >= (long long)K * 3 / 2 + trailer_bytes,
             "ps_wencode_rows: trailer %d, ld_out %lld", trailer_bytes, ld_out);
  if (N <= 0) return PS_OK;
  const int nt = (K / 256) % 2 == 0 ? WE_THREADS : WE_THREADS / 2;
  wencode_rows_kernel<<<N, nt, 0, (cudaStream_t)stream>>>(static_cast<const uint16_t*>(bits), K, ld, base,
                                                                  trailer_bytes, static_cast<uint8_t*>(out), ld_out);
  PS_CHECK_LAUNCH();
  return PS_OK;
}
