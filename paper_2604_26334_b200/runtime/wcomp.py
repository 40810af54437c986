"""Exponent-coded bf16 weights: 12 bits per weight on the host link, bit-exact.

A bf16 weight is sign (1) | exponent (8) | mantissa (7). Over the streamed
tensors of these models the exponent field takes ~25 values with ~2.1 bits of
entropy; 15 consecutive exponents [base, base + 14] cover
99.996 % of the weights. The coded row of a [N, K] matrix is

    K bytes  sign << 7 | mantissa          (one per weight)
    K/2 bytes 4-bit codes, low nibble first (exponent - base, or 15 = escape)

and an escape table gives the exact exponent of every weight outside the window:
`esc_off[N + 1]` (int32 row offsets) into `esc_ent` (int32, col << 8 | exponent,
sorted by column within a row). `ps_gemv_bf16c` (csrc/gemv_tma.cu) decodes rows
in shared memory inside the bulk-copy GEMV and accumulates in the same order as
`ps_gemv_bf16`, so its outputs are bit-identical while the matrix moves 25 % fewer
bytes. Wiring it into the executor's ring (coded host blob, coded pieces) is the
next step; this module and the kernel are its tested building blocks.
"""

from __future__ import annotations

import numpy as np

ESCAPE = 15


def choose_base(bits: np.ndarray) -> int:
    """Start of the 15-exponent window that covers the most weights (ties: lowest)."""
    exp = ((bits >> 7) & 0xFF).astype(np.int64).reshape(-1)
    hist = np.bincount(exp, minlength=256)
    cover = np.convolve(hist, np.ones(15, np.int64), mode="valid")   # cover[b] = sum hist[b:b+15]
    return int(np.argmax(cover))


def encode(bits: np.ndarray, base: int | None = None):
    """bf16 bit patterns (uint16 [N, K], K % 2 == 0) -> (coded uint8 [N, 1.5 K], base,
    esc_off int32 [N + 1], esc_ent int32 [n_escapes])."""
    bits = np.ascontiguousarray(bits, dtype=np.uint16)
    n, k = bits.shape
    if k % 2:
        raise ValueError("K must be even")
    if base is None:
        base = choose_base(bits)
    if not 0 <= base <= 255 - 14:
        raise ValueError(f"base exponent {base} outside [0, 241]")
    b32 = bits.astype(np.uint32)
    sm = (((b32 >> 8) & 0x80) | (b32 & 0x7F)).astype(np.uint8)
    exp = ((b32 >> 7) & 0xFF).astype(np.int64)
    code = exp - base
    esc = (code < 0) | (code > 14)
    code = np.where(esc, ESCAPE, code).astype(np.uint8)
    nib = (code[:, 0::2] | (code[:, 1::2] << 4)).astype(np.uint8)
    coded = np.concatenate([sm, nib], axis=1)
    rows, cols = np.nonzero(esc)                       # row-major: sorted by row, then column
    esc_off = np.zeros(n + 1, np.int32)
    np.add.at(esc_off, rows + 1, 1)
    esc_off = np.cumsum(esc_off, dtype=np.int64).astype(np.int32)
    esc_ent = ((cols.astype(np.int64) << 8) | exp[rows, cols]).astype(np.int32)
    return coded, base, esc_off, esc_ent


def decode(coded: np.ndarray, base: int, esc_off: np.ndarray, esc_ent: np.ndarray) -> np.ndarray:
    """Inverse of `encode` (CPU reference for the kernel's decoder)."""
    n, kk = coded.shape
    k = kk * 2 // 3
    sm = coded[:, :k].astype(np.uint32)
    nib = coded[:, k:]
    code = np.empty((n, k), np.uint32)
    code[:, 0::2] = nib & 0xF
    code[:, 1::2] = nib >> 4
    exp = code + base
    for r in range(n):
        for e in esc_ent[esc_off[r]:esc_off[r + 1]]:
            exp[r, e >> 8] = e & 0xFF
    return (((sm & 0x80) << 8) | (exp << 7) | (sm & 0x7F)).astype(np.uint16)


def coded_bytes(n: int, k: int, n_escapes: int) -> int:
    """Bytes a coded matrix moves: rows plus its escape table."""
    return n * k * 3 // 2 + (n + 1) * 4 + n_escapes * 4
