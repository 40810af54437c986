// Decoder of the exponent-coded weight rows (runtime/wcomp.py), shared by the coded
// GEMV (gemv_tma.cu, t <= 8) and the tensor-core decode GEMM (gemv_tc.cu, t <= 32).
// A coded row: K sign|mantissa bytes, K/2 bytes of 4-bit codes (exponent - base, 15 =
// escape), a trailer [base | n_esc << 8, (col << 8 | exp) x n_esc] of uint32 words.
#pragma once

#include <stdint.h>

namespace ps {

// 8 coded weights -> 8 bf16 (uint4). sm: their sign|mantissa bytes, nb: their eight
// 4-bit codes, base7 = (base | base << 16) << 7 of the row (gt_pair below). A code of 15
// (escape) sends the group to gt_patch_escapes, which reads the exponent from the row's
// trailer.
static __device__ __forceinline__ uint4 gt_patch_escapes(uint4 v, uint2 sm, uint32_t nb,
                                                         const uint32_t* __restrict__ trailer, int col) {
  const uint32_t n = trailer[0] >> 8;
  uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 8; ++i) {   // unrolled: every index below is a constant (no local memory)
    if (((nb >> (4 * i)) & 0xFu) != 15u) continue;
    uint32_t e = 0;
#pragma unroll 1
    for (uint32_t j = 1; j <= n; ++j) {
      const uint32_t ent = trailer[j];
      if ((int)(ent >> 8) == col + i) { e = ent & 0xFFu; break; }
    }
    const uint32_t b = (((i < 4) ? sm.x : sm.y) >> (8 * (i & 3))) & 0xFFu;
    const uint32_t half = ((b & 0x80u) << 8) | (e << 7) | (b & 0x7Fu);
    const int sh = 16 * (i & 1);
    w[i >> 1] = (w[i >> 1] & ~(0xFFFFu << sh)) | (half << sh);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// PTX prmt in its default mode: a selector nibble with bit 3 set replicates the sign of
// the selected byte (CUDA's __byte_perm documents only 3-bit selectors), so a byte
// whose msb is 0 becomes 0x00 — a zero byte without a zero operand.
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

// Two weights per 32-bit word, four instructions: one sign-replicating PRMT lays the two
// sm bytes out as [b0, sign(b0) x 8, b1, sign(b1) x 8] (so & 0x807F keeps sign << 15 |
// mantissa per half), one PRMT spreads the two codes, one IMAD adds the base and shifts,
// one LOP3 merges: (bb & 0x807F807F) | e7.
__device__ __forceinline__ uint32_t gt_pair(uint32_t smw, uint32_t sm_sel, uint32_t lo, uint32_t hi, uint32_t e_sel,
                                            uint32_t base7) {
  const uint32_t bb = prmt(smw, 0u, sm_sel);                  // [b0, s0, b1, s1]
  const uint32_t ep = prmt(lo, hi, e_sel);                    // [code0, 0, code1, 0]
  const uint32_t e7 = ep * 128u + base7;                       // (code + base) << 7, per half
  return (bb & 0x807F807Fu) | e7;
}

// Fast path only: escapes (code 15) come out wrong and are patched by the caller once
// per row when gt_escapes() flags any of the row's groups.
__device__ __forceinline__ uint4 gt_decode8(uint2 sm, uint32_t nb, uint32_t base7) {
  const uint32_t lo = nb & 0x0F0F0F0Fu, hi = (nb >> 4) & 0x0F0F0F0Fu;   // codes 0,2,4,6 | 1,3,5,7
  uint4 v;
  v.x = gt_pair(sm.x, 0x9180u, lo, hi, 0x8480u, base7);
  v.y = gt_pair(sm.x, 0xB3A2u, lo, hi, 0x9591u, base7);
  v.z = gt_pair(sm.y, 0x9180u, lo, hi, 0xA6A2u, base7);
  v.w = gt_pair(sm.y, 0xB3A2u, lo, hi, 0xB7B3u, base7);
  return v;
}

__device__ __forceinline__ uint32_t gt_escapes(uint32_t nb) {   // non-zero: some code is 15
  return nb & (nb >> 1) & (nb >> 2) & (nb >> 3) & 0x11111111u;
}

}  // namespace ps
