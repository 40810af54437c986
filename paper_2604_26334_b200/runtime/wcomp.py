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
bytes. `CodedShards` keeps coded copies of a model's dense shards in pinned host
memory; the executor streams them in GEMV (decode) passes.
"""

from __future__ import annotations

import numpy as np

ESCAPE = 15


def choose_base(bits: np.ndarray) -> int:
    """Start of the 15-exponent window that covers the most weights (ties: lowest)."""
    exp = (bits.reshape(-1) >> 7).astype(np.uint8)          # the uint8 cast drops the sign bit
    hist = np.bincount(exp, minlength=256)
    cover = np.convolve(hist, np.ones(15, np.int64), mode="valid")   # cover[b] = sum hist[b:b+15]
    return int(np.argmax(cover))


def encode(bits: np.ndarray, base: int | None = None, out: np.ndarray | None = None):
    """bf16 bit patterns (uint16 [N, K], K % 2 == 0) -> (coded uint8 [N, 1.5 K], base,
    esc_off int32 [N + 1], esc_ent int32 [n_escapes]). `out`: optional destination
    (uint8, N * 1.5 K bytes) written in place."""
    bits = np.ascontiguousarray(bits, dtype=np.uint16)
    n, k = bits.shape
    if k % 2:
        raise ValueError("K must be even")
    if base is None:
        base = choose_base(bits)
    if not 0 <= base <= 255 - 14:
        raise ValueError(f"base exponent {base} outside [0, 241]")
    coded = np.empty((n, k * 3 // 2), np.uint8) if out is None else out.reshape(n, k * 3 // 2)
    hi = (bits >> 8).astype(np.uint8)                       # sign | exponent[7:1]
    lo = bits.astype(np.uint8)                              # exponent[0] | mantissa
    np.bitwise_or(hi & 0x80, lo & 0x7F, out=coded[:, :k])
    exp = ((hi & 0x7F) << 1) | (lo >> 7)                    # uint8 exponent
    code = exp - np.uint8(base)                             # wraps for exponents below base
    esc = code > 14
    code[esc] = 15
    np.bitwise_or(code[:, 0::2], code[:, 1::2] << 4, out=coded[:, k:])
    rows, cols = np.nonzero(esc)                            # row-major: by row, then column
    esc_off = np.zeros(n + 1, np.int64)
    np.add.at(esc_off, rows + 1, 1)
    esc_off = np.cumsum(esc_off).astype(np.int32)
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


class CodedShards:
    """Exponent-coded copies of a model's dense weight shards in pinned host memory,
    for GEMV (decode) passes that stream them (`Executor`, PS_CODED=1).

    Per shard the tensors keep the blob's order, 256-byte aligned: matrices (K a
    multiple of 256) as coded rows (`tensors[sid][name] = (offset, row_bytes, base,
    off_index)`, base >= 0), norm vectors and other tensors as raw bf16 (base -1).
    All escape tables are concatenated: `esc_off` holds, for every coded matrix,
    rows + 1 absolute offsets into `esc_ent` starting at its `off_index`."""

    def __init__(self, weights, kinds, threads: int = 16):
        from concurrent.futures import ThreadPoolExecutor

        from . import lib as L
        layout = weights.layout
        up = lambda n: (n + 255) // 256 * 256  # noqa: E731
        self.tensors, self.shard_off, self.shard_bytes = {}, {}, {}
        jobs, off = [], 0
        for sid, blob in layout.blobs.items():
            if blob.kind not in kinds:
                continue
            self.shard_off[sid] = off
            t_off, meta = 0, {}
            for name, t in blob.tensors.items():
                if t.rows > 1 and t.cols % 256 == 0:
                    meta[name] = [t_off, t.cols * 3 // 2, 0, 0]
                    jobs.append((sid, name))
                    t_off += up(t.rows * t.cols * 3 // 2)
                else:
                    meta[name] = [t_off, t.cols * 2, -1, 0]
                    t_off += up(t.rows * t.cols * 2)
            self.tensors[sid] = meta
            self.shard_bytes[sid] = t_off
            off += t_off
        self.nbytes = max(1, off)
        self.host = L.host_alloc(self.nbytes, mapped=False)
        buf = np.ctypeslib.as_array((np.ctypeslib.ctypes.c_uint8 * self.nbytes).from_address(self.host))

        def work(job):
            sid, name = job
            bits = weights.host_view(sid, name)
            o = self.shard_off[sid] + self.tensors[sid][name][0]
            n_b = bits.shape[0] * bits.shape[1] * 3 // 2
            _, base, e_off, e_ent = encode(bits, out=buf[o:o + n_b])
            return base, e_off, e_ent

        with ThreadPoolExecutor(max_workers=threads) as pool:
            results = list(pool.map(work, jobs))
        offs, ents, n_off, n_ent = [], [], 0, 0
        for (sid, name), (base, e_off, e_ent) in zip(jobs, results):
            m = self.tensors[sid][name]
            m[2], m[3] = base, n_off
            offs.append(e_off.astype(np.int64) + n_ent)
            ents.append(e_ent)
            n_off += len(e_off)
            n_ent += len(e_ent)
        for sid, blob in layout.blobs.items():   # raw tensors: bytes as they are
            if sid not in self.tensors:
                continue
            for name, t in blob.tensors.items():
                m = self.tensors[sid][name]
                if m[2] < 0:
                    o = self.shard_off[sid] + m[0]
                    buf[o:o + t.rows * t.cols * 2] = weights.host_view(sid, name).reshape(-1).view(np.uint8)
        self.esc_off = (np.concatenate(offs) if offs else np.zeros(1, np.int64)).astype(np.int32)
        self.esc_ent = np.concatenate(ents).astype(np.int32) if ents and n_ent else np.zeros(1, np.int32)
        self.coded_bytes = sum(self.shard_bytes.values())
        # escape tables in host-mapped memory: the GEMV touches them only for the rare
        # escaped weight (zero-copy), so they cost no VRAM budget
        self.esc_ptrs = []
        for arr in (self.esc_off, self.esc_ent):
            ptr = L.host_alloc(max(16, arr.nbytes), mapped=True)
            np.ctypeslib.as_array((np.ctypeslib.ctypes.c_uint8 * arr.nbytes).from_address(ptr))[:] = \
                arr.view(np.uint8)
            self.esc_ptrs.append(ptr)
        self.esc_off_ptr, self.esc_ent_ptr = self.esc_ptrs

    def shard_ptr(self, sid: int) -> int:
        return self.host + self.shard_off[sid]

    def close(self) -> None:
        from . import lib as L
        if self.host:
            L.host_free(self.host)
            self.host = 0
        for ptr in getattr(self, "esc_ptrs", []):
            L.host_free(ptr)
        self.esc_ptrs = []
