// Huffman-coded exponents ("hx", runtime/hxcodec.py): ~10.1 bits per bf16 weight on the
// host link and in VRAM, lossless. The decoder expands a run of 64-row blocks to bf16 in
// VRAM ahead of the bf16 kernels (bulk-copy GEMV, one-pass tcgen05 GEMV, tcgen05 GEMM),
// which therefore see exactly the bf16 weights: results are bit-identical to bf16.
//
//   ps_hx_expand  decode: one lane per 256-weight sub-block (bit offset = prefix of the
//                 row header's sub-block lengths) decodes its exponents into shared memory
//                 (a 4096-entry table turns the next 12 bits of the LSB-first stream into
//                 one symbol, or two when both codes fit; exponent = rowmax - symbol), then the
//                 warp assembles bf16 rows with coalesced loads and stores
//   ps_hx_stats   encoder pass 1: row max exponent + histogram of d = rowmax - exponent
//   ps_hx_sizes   encoder pass 2: bits per sub-block, bytes per row (host: Huffman code,
//                 row and block offsets)
//   ps_hx_write   encoder pass 3: block headers, row headers, sign|mantissa bytes, the
//                 bit streams (atomicOr into a zeroed buffer: sub-blocks share words)
//
// Bound: link bytes. The expand kernel runs at HBM-class speed (it writes 2 bytes per
// weight and reads ~1.26), microseconds per piece against the milliseconds a piece takes
// to cross PCIe; prefill passes run it ahead of the GEMM on every piece.
#include "common.cuh"
#include "wcodec.cuh"
#include "../../include/pshard.h"

namespace ps {

constexpr int HX_SUB = 256, HX_BLOCK_ROWS = 64, HX_LUT = 4096, HX_THREADS = 256;

__device__ __forceinline__ int hx_header_bytes(int K) { return ((4 + 2 * (K / HX_SUB)) + 15) / 16 * 16; }

// expand: CTA (b, part) of HX_EXP_WARPS warps takes tasks [part * 32 * HX_EXP_WARPS, ...)
// of block b of a piece, task = (row r, sub-block s), r = task / (K / 256); blk[b] = byte
// offset of block b from `piece`. Two phases per warp of 32 tasks:
//   1. each lane decodes ITS sub-block's 256 exponents (serial: the bit stream is a chain)
//      into a shared-memory row of its own (65 words: conflict-free), from a 64-bit bit
//      buffer with one word of look-ahead, one 4096-entry table lookup per symbol;
//   2. the warp assembles the 32 sub-blocks one at a time, lane l taking 8 columns: the
//      sign|mantissa loads (256 B) and the bf16 stores (512 B) are coalesced.
constexpr int HX_EXP_WARPS = 4;
constexpr int HX_CHUNK = 64;                        // symbols per decode round
constexpr int HX_EXP_ROW_WORDS = HX_CHUNK / 4 + 1;  // 16 exponent words + 1 (bank offset)

// One CTA's share (`part`) of one 64-row block: `block` = the block's bytes, `nr` rows,
// `out` = bf16 row 0 of the block (ld_out elements per row); lut = the 4096-entry table
// already in shared memory. Every thread reaches both barriers (the CTA loops over items).
__device__ __forceinline__ void hx_expand_item(const uint8_t* __restrict__ block, int nr, int K, int part,
                                               const uint32_t* __restrict__ lut, uint32_t* __restrict__ row_start,
                                               uint32_t (*exps)[32][HX_EXP_ROW_WORDS],
                                               __nv_bfloat16* __restrict__ out, long long ld_out) {
  const int nsub = K / HX_SUB;
  const int hb = hx_header_bytes(K);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = 0;
  if (warp == 0) {   // row starts: exclusive scan of the 64 row sizes
    const uint32_t* sizes = reinterpret_cast<const uint32_t*>(block);
    uint32_t a = lane < nr ? sizes[lane] : 0u;
    uint32_t b = lane + 32 < nr ? sizes[lane + 32] : 0u;
    uint32_t sa = a, sb = b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t ua = __shfl_up_sync(0xffffffffu, sa, o), ub = __shfl_up_sync(0xffffffffu, sb, o);
      if (lane >= o) { sa += ua; sb += ub; }
    }
    const uint32_t tot_a = __shfl_sync(0xffffffffu, sa, 31);
    row_start[lane] = 256 + sa - a;
    row_start[lane + 32] = 256 + tot_a + sb - b;
  }
  __syncthreads();
  const int task0 = (part * HX_EXP_WARPS + warp) * 32;
  if (task0 < nr * nsub) {   // (warps past the block's tasks skip to the closing barrier)
    // Four rounds of 64 symbols: each lane decodes the next 64 exponents of ITS sub-block
    // (serial: the bit stream is a chain) into its 64-byte shared row (17 words:
    // conflict-free), then the warp assembles those 64 columns of all 32 sub-blocks —
    // 8 lanes per sub-block, 16-B coalesced loads and stores. A 2 KB buffer per warp
    // instead of 8 KB keeps ~2x the warps resident to hide the decode chain.
    uint32_t* my = exps[warp][lane];
    uint8_t* myb = reinterpret_cast<uint8_t*>(my);
    const int ntask = min(32, nr * nsub - task0);
    const int task = task0 + lane;
    const int r = task / nsub, s = task - (task / nsub) * nsub;
    const bool live = lane < ntask;
    uint32_t rowmax = 0;
    const uint32_t* p = nullptr;
    uint64_t buf = 0;
    int avail = 64;
    uint32_t nextw = 0, nextw2 = 0;
    int carry = -1;   // a symbol decoded past the previous round's end
    if (live) {
      const uint8_t* row = block + row_start[r];
      const uint16_t* hdr = reinterpret_cast<const uint16_t*>(row);
      rowmax = hdr[0];
      uint32_t pos = 0;
      for (int i = 0; i < s; ++i) pos += hdr[2 + i];
      // 64-bit bit buffer, refilled one word at a time with one word of look-ahead; the
      // refill test runs once per two lookups (a lane refills every few lookups, but in
      // a warp SOME lane almost always does, so a per-lookup test costs every lane the
      // refill path): after it the buffer holds >= 32 bits, enough for two 12-bit
      // windows. One lookup resolves one symbol, or two when both codes fit the window.
      p = reinterpret_cast<const uint32_t*>(row + hb + K) + (pos >> 5);
      buf = (((uint64_t)p[1] << 32) | p[0]) >> (pos & 31);
      avail = 64 - (int)(pos & 31);
      nextw = p[2];     // two words of look-ahead (~28 symbols): a refill's load has the time
      nextw2 = p[3];    // of ~14 lookups to come back from L2 (the stream lines rarely stay in L1)
      p += 4;
    }
    const int q = lane >> 3, l8 = lane & 7;   // phase 2: sub-block 4 i + q, columns 8 l8 ..
    // phase-2 addresses of the (up to) 8 sub-blocks this lane assembles, once per item
    const uint8_t* src8[8];
    __nv_bfloat16* dst8[8];
    uint32_t rmax4[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int j = 4 * i + q;
      const int tj = task0 + min(j, ntask - 1), rj = tj / nsub, sj = tj - (tj / nsub) * nsub;
      src8[i] = block + row_start[rj] + hb + sj * HX_SUB + 8 * l8;
      dst8[i] = out + (long long)(r0 + rj) * ld_out + sj * HX_SUB + 8 * l8;
      rmax4[i] = __shfl_sync(0xffffffffu, rowmax, min(j, 31)) * 0x01010101u;   // sub-block j's rowmax
    }
#pragma unroll 1
    for (int c0 = 0; c0 < HX_SUB; c0 += HX_CHUNK) {
      if (live) {   // symbols (rowmax - exponent) of this lane's next 64 weights
        // A lookup always stores two symbol bytes and advances by the count it resolved
        // (a lone symbol's second byte is overwritten by the next lookup); a pair that
        // straddles the round's end leaves its second symbol in byte 64, carried to
        // byte 0 of the next round. No per-lookup end test beyond the loop's.
        int k = 0;
        if (carry >= 0) { myb[0] = (uint8_t)carry; k = 1; }
#pragma unroll 1
        while (k < HX_CHUNK) {
          if (avail < 32) {
            buf |= (uint64_t)nextw << avail;
            avail += 32;
            nextw = nextw2;
            nextw2 = *p++;
          }
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            if (k < HX_CHUNK) {
              const uint32_t e = lut[(uint32_t)buf & (HX_LUT - 1)];
              const int len = (int)((e >> 16) & 0xFFu);
              myb[k] = (uint8_t)e;
              myb[k + 1] = (uint8_t)(e >> 8);
              buf >>= len;
              avail -= len;
              k += (int)(e >> 24);
            }
          }
        }
        carry = k > HX_CHUNK ? (int)myb[HX_CHUNK] : -1;
      }
      __syncwarp();
      uint2 mm[8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        mm[i] = 4 * i + q < ntask ? *reinterpret_cast<const uint2*>(src8[i] + c0) : make_uint2(0u, 0u);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int j = 4 * i + q;
        if (j < ntask) {
          // exponents = rowmax - symbol, four bytes per instruction; then two weights per
          // word as in wcodec.cuh: a sign-replicating PRMT keeps sign << 15 | mantissa
          // under & 0x807F807F, a PRMT spreads two exponents, a shift places them
          const uint32_t e0 = __vsub4(rmax4[i], exps[warp][j][2 * l8]);
          const uint32_t e1 = __vsub4(rmax4[i], exps[warp][j][2 * l8 + 1]);
          uint4 w;
          w.x = (prmt(mm[i].x, 0u, 0x9180u) & 0x807F807Fu) | (prmt(e0, 0u, 0x4140u) << 7);
          w.y = (prmt(mm[i].x, 0u, 0xB3A2u) & 0x807F807Fu) | (prmt(e0, 0u, 0x4342u) << 7);
          w.z = (prmt(mm[i].y, 0u, 0x9180u) & 0x807F807Fu) | (prmt(e1, 0u, 0x4140u) << 7);
          w.w = (prmt(mm[i].y, 0u, 0xB3A2u) & 0x807F807Fu) | (prmt(e1, 0u, 0x4342u) << 7);
          *reinterpret_cast<uint4*>(dst8[i] + c0) = w;
        }
      }
      __syncwarp();   // the next round overwrites the rows
    }
  }
  __syncthreads();   // row_start / exps are reused by the CTA's next item
}

// The table is loaded once per CTA and CTAs loop over items (one part of a 64-row block):
// a CTA per item read the 16 KB table per 128 sub-blocks (32 KB of weights) — ncu r02:
// the top stall of the expert expansion.
__device__ __forceinline__ void hx_load_lut(const uint32_t* __restrict__ lut_g, uint32_t* lut) {
  const uint4* src = reinterpret_cast<const uint4*>(lut_g);
  uint4* dst = reinterpret_cast<uint4*>(lut);
  for (int i = threadIdx.x; i < HX_LUT / 4; i += 32 * HX_EXP_WARPS) dst[i] = src[i];
  __syncthreads();
}

// Minimum resident CTAs per SM the expansion kernels are compiled for (build-time
// experiment knob: -DPS_HX_MIN_CTAS=6 trades ~20 spilled bytes for a sixth CTA per SM).
// (Default: the one-argument bound. `__launch_bounds__(128, 1)` is not equivalent in
// practice: ptxas then takes 128 / 141 registers instead of 94 / 128.)
#ifndef PS_HX_MIN_CTAS
#define PS_HX_MIN_CTAS 1
#endif
#if PS_HX_MIN_CTAS > 1
#define PS_HX_BOUNDS __launch_bounds__(32 * HX_EXP_WARPS, PS_HX_MIN_CTAS)
#else
#define PS_HX_BOUNDS __launch_bounds__(32 * HX_EXP_WARPS)
#endif

__global__ void PS_HX_BOUNDS
hx_expand_kernel(const uint8_t* __restrict__ piece, const uint32_t* __restrict__ blk, int rows, int K,
                 const uint32_t* __restrict__ lut_g, __nv_bfloat16* __restrict__ out, long long ld_out) {
  __shared__ uint32_t lut[HX_LUT];   // s1 | s2 << 8 | bits << 16 | n << 24
  __shared__ uint32_t row_start[HX_BLOCK_ROWS];
  extern __shared__ uint32_t hx_exps[];   // [warp][lane][65] exponent rows (dynamic: > 48 KB static)
  auto exps = reinterpret_cast<uint32_t (*)[32][HX_EXP_ROW_WORDS]>(hx_exps);
  hx_load_lut(lut_g, lut);
  const int parts = (HX_BLOCK_ROWS * (K / HX_SUB) + 32 * HX_EXP_WARPS - 1) / (32 * HX_EXP_WARPS);
  const int nb = (rows + HX_BLOCK_ROWS - 1) / HX_BLOCK_ROWS;
  for (int item = blockIdx.x; item < nb * parts; item += gridDim.x) {
    const int b = item / parts, part = item - b * parts;
    const int r0 = b * HX_BLOCK_ROWS;
    hx_expand_item(piece + blk[b], min(HX_BLOCK_ROWS, rows - r0), K, part, lut, row_start, exps,
                   out + (long long)r0 * ld_out, ld_out);
  }
}

__device__ __forceinline__ int hx_exp(uint16_t b) { return (b >> 7) & 0xFF; }

__global__ void __launch_bounds__(HX_THREADS)
hx_stats_kernel(const uint16_t* __restrict__ bits, int K, long long ld, int* __restrict__ rowmax,
                unsigned long long* __restrict__ hist) {
  __shared__ int red[HX_THREADS / 32];
  __shared__ unsigned int h[256];
  const uint16_t* row = bits + blockIdx.x * ld;
  h[threadIdx.x] = 0;
  int mx = 0;
  for (int c = threadIdx.x; c < K; c += HX_THREADS) mx = max(mx, hx_exp(row[c]));
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = 0;
  for (int i = 0; i < HX_THREADS / 32; ++i) mx = max(mx, red[i]);
  for (int c = threadIdx.x; c < K; c += HX_THREADS) atomicAdd(&h[mx - hx_exp(row[c])], 1u);
  __syncthreads();
  if (h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], (unsigned long long)h[threadIdx.x]);
  if (threadIdx.x == 0) rowmax[blockIdx.x] = mx;
}

__global__ void __launch_bounds__(HX_THREADS)
hx_sizes_kernel(const uint16_t* __restrict__ bits, int K, long long ld, const int* __restrict__ rowmax,
                const uint32_t* __restrict__ table, uint16_t* __restrict__ sublen, uint32_t* __restrict__ rowbytes) {
  __shared__ uint32_t tot;
  const uint16_t* row = bits + blockIdx.x * ld;
  const int nsub = K / HX_SUB, mx = rowmax[blockIdx.x];
  if (threadIdx.x == 0) tot = 0;
  __syncthreads();
  for (int s = threadIdx.x; s < nsub; s += HX_THREADS) {
    uint32_t n = 0;
    for (int c = s * HX_SUB; c < (s + 1) * HX_SUB; ++c) n += table[mx - hx_exp(row[c])] >> 16;
    sublen[(long long)blockIdx.x * nsub + s] = (uint16_t)n;
    atomicAdd(&tot, n);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t stream = ((tot + 7) / 8 + 24 + 15) / 16 * 16;   // >= 24 spare bytes: the decoder reads ahead
    rowbytes[blockIdx.x] = (uint32_t)hx_header_bytes(K) + (uint32_t)K + stream;
  }
}

__global__ void __launch_bounds__(HX_THREADS)
hx_write_kernel(const uint16_t* __restrict__ bits, int K, long long ld, const int* __restrict__ rowmax,
                const uint32_t* __restrict__ table, const uint16_t* __restrict__ sublen,
                const uint32_t* __restrict__ rowbytes, const unsigned long long* __restrict__ row_off, int N,
                uint8_t* __restrict__ out) {
  const int r = blockIdx.x;
  const uint16_t* row = bits + r * ld;
  const int nsub = K / HX_SUB, mx = rowmax[r], hb = hx_header_bytes(K);
  uint8_t* o = out + row_off[r];
  if (r % HX_BLOCK_ROWS == 0) {   // the block header: 64 row sizes (0 past N)
    uint32_t* bh = reinterpret_cast<uint32_t*>(o - 256);
    for (int i = threadIdx.x; i < HX_BLOCK_ROWS; i += HX_THREADS) bh[i] = r + i < N ? rowbytes[r + i] : 0u;
  }
  uint16_t* hdr = reinterpret_cast<uint16_t*>(o);
  for (int i = threadIdx.x; i < hb / 2; i += HX_THREADS)
    hdr[i] = i == 0 ? (uint16_t)mx : (i >= 2 && i < 2 + nsub ? sublen[(long long)r * nsub + i - 2] : 0);
  for (int c = threadIdx.x; c < K; c += HX_THREADS) {
    const uint16_t b = row[c];
    o[hb + c] = (uint8_t)(((b >> 8) & 0x80) | (b & 0x7F));
  }
  uint32_t* sw = reinterpret_cast<uint32_t*>(o + hb + K);
  for (int s = threadIdx.x; s < nsub; s += HX_THREADS) {
    uint32_t pos = 0;
    for (int i = 0; i < s; ++i) pos += sublen[(long long)r * nsub + i];
    for (int c = s * HX_SUB; c < (s + 1) * HX_SUB; ++c) {
      const uint32_t t = table[mx - hx_exp(row[c])];
      const uint32_t len = t >> 16, code = t & 0xFFFFu;
      const uint32_t sh = pos & 31, idx = pos >> 5;
      atomicOr(&sw[idx], code << sh);
      if (sh + len > 32) atomicOr(&sw[idx + 1], code >> (32 - sh));
      pos += len;
    }
  }
}

// The routed experts of one MoE layer, fetched hx-coded into slots (expert rank j in slot
// j, or slot_of_rank[j] when the fetcher placed it — a speculative prefetch hit): each slot holds a span [uint32 block offsets of both matrices][...][hx matrices];
// item (j, b, part) expands block b of expert j's matrix into scratch expert j (out_off
// bytes into it, rows of K bf16) for the bf16 one-token expert kernels.
// Both matrices of the routed experts (gate/up, down) in ONE launch: the expansion is
// latency-bound (a 256-weight serial decode per lane), so two back-to-back launches cost
// two decode latencies on the routing chain; here CTAs [0, grid_a) expand matrix A with
// its table, the rest matrix B with its own.
struct HxExpertMat {
  int hdr_word;
  long long mat_off;
  int rows, K;
  const uint32_t* lut;
  long long out_off;
};

__global__ void PS_HX_BOUNDS
hx_expand_experts2_kernel(const uint8_t* __restrict__ slots, long long slot_stride, const int* __restrict__ slot_of_rank,
                          int k, HxExpertMat a, HxExpertMat b, int grid_a, uint8_t* __restrict__ scratch,
                          long long scratch_stride) {
  __shared__ uint32_t lut[HX_LUT];
  __shared__ uint32_t row_start[HX_BLOCK_ROWS];
  extern __shared__ uint32_t hx_exps[];
  auto exps = reinterpret_cast<uint32_t (*)[32][HX_EXP_ROW_WORDS]>(hx_exps);
  const bool is_a = (int)blockIdx.x < grid_a;
  const HxExpertMat& m = is_a ? a : b;
  const int cta = is_a ? blockIdx.x : blockIdx.x - grid_a, ncta = is_a ? grid_a : gridDim.x - grid_a;
  hx_load_lut(m.lut, lut);
  const int parts = (HX_BLOCK_ROWS * (m.K / HX_SUB) + 32 * HX_EXP_WARPS - 1) / (32 * HX_EXP_WARPS);
  const int nb = (m.rows + HX_BLOCK_ROWS - 1) / HX_BLOCK_ROWS;
  for (int item = cta; item < k * nb * parts; item += ncta) {
    const int part = item % parts, jb = item / parts;
    const int j = jb / nb, bb = jb - (jb / nb) * nb;
    const uint8_t* span = slots + (long long)(slot_of_rank ? slot_of_rank[j] : j) * slot_stride;
    const uint32_t off = reinterpret_cast<const uint32_t*>(span)[m.hdr_word + bb];
    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(scratch + j * scratch_stride + m.out_off) +
                       (long long)bb * HX_BLOCK_ROWS * m.K;
    hx_expand_item(span + m.mat_off + off, min(HX_BLOCK_ROWS, m.rows - bb * HX_BLOCK_ROWS), m.K, part, lut,
                   row_start, exps, o, m.K);
  }
}

// resident CTAs of the expand kernels (8 per SM at ~25 KB of shared memory each)
static int hx_grid_cap() {
  static int cap = 0;
  if (!cap) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cap = 8 * (sms > 0 ? sms : 148);
  }
  return cap;
}

}  // namespace ps

extern "C" int ps_hx_expand(const void* piece, const unsigned* block_off, int rows, int K, const void* lut,
                            void* out, long long ld_out, void* stream) {
  using namespace ps;
  PS_REQUIRE(K > 0 && K % HX_SUB == 0 && ld_out >= K && ld_out % 8 == 0, "ps_hx_expand: K %d, ld_out %lld", K,
             ld_out);
  PS_REQUIRE(((uintptr_t)piece & 15) == 0 && ((uintptr_t)out & 15) == 0 && ((uintptr_t)lut & 15) == 0,
             "ps_hx_expand: piece, out and lut must be 16-byte aligned");
  if (rows <= 0) return PS_OK;
  const int nblocks = (rows + HX_BLOCK_ROWS - 1) / HX_BLOCK_ROWS;
  const int per_cta = 32 * HX_EXP_WARPS;
  const int parts = (HX_BLOCK_ROWS * (K / HX_SUB) + per_cta - 1) / per_cta;
  constexpr int smem = HX_EXP_WARPS * 32 * HX_EXP_ROW_WORDS * 4;
  static bool smem_set = false;
  if (!smem_set) {
    PS_CHECK_CUDA(cudaFuncSetAttribute(hx_expand_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    if (PS_HX_MIN_CTAS > 5)
      PS_CHECK_CUDA(cudaFuncSetAttribute(hx_expand_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                         cudaSharedmemCarveoutMaxShared));
    smem_set = true;
  }
  const int grid = min(nblocks * parts, hx_grid_cap());
  hx_expand_kernel<<<grid, per_cta, smem, (cudaStream_t)stream>>>(
      static_cast<const uint8_t*>(piece), block_off, rows, K, static_cast<const uint32_t*>(lut),
      static_cast<__nv_bfloat16*>(out), ld_out);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

extern "C" int ps_hx_expand_experts2(const void* slots, long long slot_stride, const int* slot_of_rank, int k,
                                     int hdr_a, long long mat_a,
                                     int rows_a, int K_a, const void* lut_a, long long out_a, int hdr_b,
                                     long long mat_b, int rows_b, int K_b, const void* lut_b, long long out_b,
                                     void* scratch, long long scratch_stride, void* stream) {
  using namespace ps;
  PS_REQUIRE(K_a > 0 && K_a % HX_SUB == 0 && K_b > 0 && K_b % HX_SUB == 0 && rows_a > 0 && rows_b > 0 && k >= 0,
             "ps_hx_expand_experts2: K %d / %d rows %d / %d k %d", K_a, K_b, rows_a, rows_b, k);
  PS_REQUIRE(((uintptr_t)slots & 15) == 0 && (slot_stride & 255) == 0 && ((mat_a | mat_b) & 15) == 0 &&
                 ((uintptr_t)scratch & 15) == 0 && (scratch_stride & 15) == 0 && ((out_a | out_b) & 15) == 0,
             "ps_hx_expand_experts2: alignment");
  if (k == 0) return PS_OK;
  const int per_cta = 32 * HX_EXP_WARPS;
  auto items = [&](int rows, int K) {
    return k * ((rows + HX_BLOCK_ROWS - 1) / HX_BLOCK_ROWS) * ((HX_BLOCK_ROWS * (K / HX_SUB) + per_cta - 1) / per_cta);
  };
  const int ia = items(rows_a, K_a), ib = items(rows_b, K_b);
  const int cap = hx_grid_cap();
  // resident CTAs split between the two matrices in proportion to their items
  int ga = (int)((long long)cap * ia / (ia + ib));
  ga = ga < 1 ? 1 : (ga > ia ? ia : ga);
  int gb = cap - ga;
  gb = gb < 1 ? 1 : (gb > ib ? ib : gb);
  constexpr int smem = HX_EXP_WARPS * 32 * HX_EXP_ROW_WORDS * 4;
  static bool smem_set = false;
  if (!smem_set) {
    PS_CHECK_CUDA(cudaFuncSetAttribute(hx_expand_experts2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    if (PS_HX_MIN_CTAS > 5)
      PS_CHECK_CUDA(cudaFuncSetAttribute(hx_expand_experts2_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                         cudaSharedmemCarveoutMaxShared));
    smem_set = true;
  }
  const HxExpertMat a{hdr_a, mat_a, rows_a, K_a, static_cast<const uint32_t*>(lut_a), out_a};
  const HxExpertMat b{hdr_b, mat_b, rows_b, K_b, static_cast<const uint32_t*>(lut_b), out_b};
  hx_expand_experts2_kernel<<<ga + gb, per_cta, smem, (cudaStream_t)stream>>>(
      static_cast<const uint8_t*>(slots), slot_stride, slot_of_rank, k, a, b, ga, static_cast<uint8_t*>(scratch),
      scratch_stride);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

extern "C" int ps_hx_stats(const void* bits, int N, int K, long long ld, int* rowmax, unsigned long long* hist,
                           void* stream) {
  using namespace ps;
  PS_REQUIRE(K > 0 && ld >= K, "ps_hx_stats: K %d ld %lld", K, ld);
  if (N <= 0) return PS_OK;
  hx_stats_kernel<<<N, HX_THREADS, 0, (cudaStream_t)stream>>>(static_cast<const uint16_t*>(bits), K, ld, rowmax,
                                                               hist);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

extern "C" int ps_hx_sizes(const void* bits, int N, int K, long long ld, const int* rowmax, const unsigned* table,
                           unsigned short* sublen, unsigned* rowbytes, void* stream) {
  using namespace ps;
  PS_REQUIRE(K > 0 && K % HX_SUB == 0 && ld >= K, "ps_hx_sizes: K %d ld %lld", K, ld);
  if (N <= 0) return PS_OK;
  hx_sizes_kernel<<<N, HX_THREADS, 0, (cudaStream_t)stream>>>(static_cast<const uint16_t*>(bits), K, ld, rowmax,
                                                               table, sublen, rowbytes);
  PS_CHECK_LAUNCH();
  return PS_OK;
}

extern "C" int ps_hx_write(const void* bits, int N, int K, long long ld, const int* rowmax, const unsigned* table,
                           const unsigned short* sublen, const unsigned* rowbytes, const unsigned long long* row_off,
                           void* out, void* stream) {
  using namespace ps;
  PS_REQUIRE(K > 0 && K % HX_SUB == 0 && ld >= K, "ps_hx_write: K %d ld %lld", K, ld);
  if (N <= 0) return PS_OK;
  hx_write_kernel<<<N, HX_THREADS, 0, (cudaStream_t)stream>>>(static_cast<const uint16_t*>(bits), K, ld, rowmax,
                                                               table, sublen, rowbytes, row_off, N,
                                                               static_cast<uint8_t*>(out));
  PS_CHECK_LAUNCH();
  return PS_OK;
}

int ps_preload_hx() {
  using namespace ps;
  int n = 0;
  touch_kernel(hx_expand_kernel, n);
  touch_kernel(hx_expand_experts2_kernel, n);
  return n;
}
