"""Huffman-coded exponents ("hx"): ~10.1 bits per bf16 weight, lossless.

The 12-bit format (runtime/wcomp.py) spends 4 bits on an exponent whose entropy over
these weights is ~2 bits. hx codes it with a per-matrix canonical
Huffman code instead, keeping the sign|mantissa byte raw:

    symbol  d = rowmax_r - exponent      (rowmax_r = the row's largest exponent)
    code    canonical Huffman over the matrix's histogram of d, lengths <= 12 bits,
            packed LSB-first (bit-reversed codes), so a decoder peeks 12 bits and
            looks the symbol up in a 4096-entry table

Layout of one [N, K] matrix (K % 256 == 0), rows in blocks of 64:

    block   64 x uint32 row byte sizes (rows past N: 0), then the block's rows
    row     header: uint16 rowmax, uint16 0, uint16 bit length of each 256-weight
            sub-block (K / 256 of them), padded to 16 bytes
            K bytes sign << 7 | mantissa
            the bit stream, padded (after >= 24 spare bytes: the decoder reads up
            to 95 bits ahead) to 16 bytes

Every 64-row block is self-contained: a ring piece is a run of whole blocks, and the
decoder (`ps_hx_expand`, csrc/hx.cu) needs only the block offsets of its piece and
the matrix's code table (256 x uint32: length << 16 | bit-reversed code). A sub-block
decodes independently of its neighbours (its bit offset is a prefix sum of the
header's lengths), so one thread decodes 256 weights.

This module is the format's CPU reference (encoder + decoder, test sizes only); the
GPU encoder (`ps_hx_stats` / `ps_hx_sizes` / `ps_hx_write`) must produce the same bytes.
"""

from __future__ import annotations

import numpy as np

MAX_LEN = 12
SUB = 256                 # weights per independently decodable sub-block
BLOCK_ROWS = 64


def code_lengths(hist: np.ndarray, max_len: int = MAX_LEN) -> np.ndarray:
    """Huffman code lengths (uint8 [256]) for a symbol histogram, limited to max_len
    bits by package-merge; symbols with count 0 get length 0. A single used symbol gets
    length 1. Deterministic: ties break on the symbol index."""
    hist = np.asarray(hist, dtype=np.int64)
    used = [int(s) for s in np.nonzero(hist)[0]]
    lengths = np.zeros(256, np.uint8)
    if not used:
        return lengths
    if len(used) == 1:
        lengths[used[0]] = 1
        return lengths
    # package-merge (boundary-free form): max_len rounds of pairing
    leaves = sorted((int(hist[s]), s) for s in used)
    items = [(w, (s,)) for w, s in leaves]
    cur = list(items)
    for _ in range(max_len - 1):
        pk = [(cur[i][0] + cur[i + 1][0], cur[i][1] + cur[i + 1][1]) for i in range(0, len(cur) - 1, 2)]
        cur = sorted(items + pk, key=lambda t: (t[0], len(t[1]), t[1]))
    take = cur[:2 * len(used) - 2]
    for _, syms in take:
        for s in syms:
            lengths[s] += 1
    return lengths


def canonical_table(lengths: np.ndarray) -> np.ndarray:
    """uint32 [256]: length << 16 | code bit-reversed (LSB-first), canonical order
    (by length, then symbol); 0 for unused symbols."""
    table = np.zeros(256, np.uint32)
    order = sorted((int(lengths[s]), s) for s in range(256) if lengths[s])
    code, prev = 0, 0
    for ln, s in order:
        code <<= (ln - prev)
        prev = ln
        rev = int(f"{code:0{ln}b}"[::-1], 2)
        table[s] = (ln << 16) | rev
        code += 1
    return table


def _exp(bits: np.ndarray) -> np.ndarray:
    return ((bits >> 7) & 0xFF).astype(np.int32)


def histogram(bits: np.ndarray) -> tuple:
    """(rowmax int32 [N], histogram int64 [256] of d = rowmax - exponent)."""
    e = _exp(bits)
    rowmax = e.max(axis=1)
    d = rowmax[:, None] - e
    return rowmax, np.bincount(d.reshape(-1), minlength=256).astype(np.int64)


def header_bytes(k: int) -> int:
    return -(-(4 + 2 * (k // SUB)) // 16) * 16


def row_bytes(k: int, nbits: int) -> int:
    return header_bytes(k) + k + -(-(-(-nbits // 8) + 24) // 16) * 16


def encode(bits: np.ndarray, table: np.ndarray | None = None):
    """bf16 bits uint16 [N, K] -> (blob uint8, block offsets uint64 [nblocks + 1], table).
    Pure Python bit packing: test sizes only."""
    bits = np.ascontiguousarray(bits, dtype=np.uint16)
    n, k = bits.shape
    if k % SUB:
        raise ValueError("K must be a multiple of 256")
    rowmax, hist = histogram(bits)
    if table is None:
        table = canonical_table(code_lengths(hist))
    e = _exp(bits)
    d = rowmax[:, None] - e
    lens = (table[d] >> 16).astype(np.int64)
    codes = (table[d] & 0xFFFF).astype(np.int64)
    sublen = lens.reshape(n, k // SUB, SUB).sum(axis=2)            # bits per sub-block
    rbytes = [row_bytes(k, int(sublen[r].sum())) for r in range(n)]
    nblocks = -(-n // BLOCK_ROWS)
    offs = np.zeros(nblocks + 1, np.uint64)
    for b in range(nblocks):
        offs[b + 1] = offs[b] + 256 + sum(rbytes[b * BLOCK_ROWS:(b + 1) * BLOCK_ROWS])
    blob = np.zeros(int(offs[-1]), np.uint8)
    hb = header_bytes(k)
    sm = (((bits >> 8) & 0x80) | (bits & 0x7F)).astype(np.uint8)
    for b in range(nblocks):
        r0, r1 = b * BLOCK_ROWS, min(n, (b + 1) * BLOCK_ROWS)
        pos = int(offs[b])
        blob[pos:pos + 4 * (r1 - r0)] = np.array(rbytes[r0:r1], np.uint32).view(np.uint8)
        pos += 256
        for r in range(r0, r1):
            hdr = np.zeros(hb // 2, np.uint16)
            hdr[0] = rowmax[r]
            hdr[2:2 + k // SUB] = sublen[r]
            blob[pos:pos + hb] = hdr.view(np.uint8)
            blob[pos + hb:pos + hb + k] = sm[r]
            acc, nacc, out = 0, 0, bytearray()
            for c in range(k):
                acc |= int(codes[r, c]) << nacc
                nacc += int(lens[r, c])
                while nacc >= 8:
                    out.append(acc & 0xFF)
                    acc >>= 8
                    nacc -= 8
            if nacc:
                out.append(acc & 0xFF)
            s0 = pos + hb + k
            blob[s0:s0 + len(out)] = np.frombuffer(bytes(out), np.uint8)
            pos += rbytes[r]
    return blob, offs, table


def decode(blob: np.ndarray, offs: np.ndarray, table: np.ndarray, n: int, k: int) -> np.ndarray:
    """Inverse of `encode` (CPU reference of ps_hx_expand): uint16 bf16 bits [N, K]."""
    lut = {}
    for s in range(256):
        if table[s]:
            lut[(int(table[s]) >> 16, int(table[s]) & 0xFFFF)] = s
    out = np.zeros((n, k), np.uint16)
    hb = header_bytes(k)
    for b in range(len(offs) - 1):
        pos = int(offs[b])
        r0, r1 = b * BLOCK_ROWS, min(n, (b + 1) * BLOCK_ROWS)
        sizes = blob[pos:pos + 4 * (r1 - r0)].view(np.uint32)
        pos += 256
        for i, r in enumerate(range(r0, r1)):
            hdr = blob[pos:pos + hb].view(np.uint16)
            rowmax = int(hdr[0])
            sm = blob[pos + hb:pos + hb + k].astype(np.uint16)
            stream = blob[pos + hb + k:pos + int(sizes[i])]
            bitpos = 0
            for c in range(k):
                code, ln = 0, 0
                while (ln, code) not in lut:
                    byte = int(stream[bitpos >> 3])
                    code |= ((byte >> (bitpos & 7)) & 1) << ln
                    ln += 1
                    bitpos += 1
                    if ln > MAX_LEN:
                        raise ValueError("bad code")
                e = rowmax - lut[(ln, code)]
                out[r, c] = ((sm[c] & 0x80) << 8) | (e << 7) | (sm[c] & 0x7F)
            pos += int(sizes[i])
    return out


def pair_table(table: np.ndarray) -> np.ndarray:
    """The decoder's 4096-entry table (uint32) of `ps_hx_expand`: for every 12-bit
    LSB-first window, s1 | s2 << 8 | bits << 16 | n << 24 — the first symbol and, when the
    second code also lies inside the window, the second (n = 2), with the bits they take."""
    single = lookup_table(table).astype(np.uint32)
    x = np.arange(1 << MAX_LEN, dtype=np.uint32)
    s1, l1 = single & 0xFF, single >> 8
    rest = x >> l1
    e2 = single[rest]
    s2, l2 = e2 & 0xFF, e2 >> 8
    two = (l2 <= MAX_LEN - l1).astype(np.uint32)
    return (s1 | (np.where(two, s2, 0) << 8) | (np.where(two, l1 + l2, l1) << 16)
            | ((1 + two) << 24)).astype(np.uint32)


def lookup_table(table: np.ndarray) -> np.ndarray:
    """The decoder's 4096-entry table (uint16: symbol | length << 8) for a code table:
    every 12-bit LSB-first window whose low `length` bits are a symbol's reversed code."""
    lut = np.zeros(1 << MAX_LEN, np.uint16)
    for s in range(256):
        t = int(table[s])
        if not t:
            continue
        ln, rev = t >> 16, t & 0xFFFF
        lut[rev | (np.arange(1 << (MAX_LEN - ln)) << ln)] = s | (ln << 8)
    return lut


class HxMatrix:
    """One hx-coded matrix: its geometry, code table, decoder table, block offsets
    (uint64 [nblocks + 1], bytes from the matrix start) and size."""

    def __init__(self, n: int, k: int, table: np.ndarray, block_off: np.ndarray):
        self.n, self.k, self.table = n, k, table
        self._lut = None
        self.block_off = block_off
        self.nbytes = int(block_off[-1])

    @property
    def lut(self) -> np.ndarray:
        """The decoder table (pair_table), built on first use."""
        if self._lut is None:
            self._lut = pair_table(self.table)
        return self._lut

    def blocks_for_rows(self, r0: int, r1: int) -> tuple:
        """(first block, end block) covering rows [r0, r1) (r0 on a block boundary)."""
        return r0 // BLOCK_ROWS, -(-r1 // BLOCK_ROWS)


class GpuHxEncoder:
    """The hx encoder on the GPU (csrc/hx.cu: ps_hx_stats, ps_hx_sizes, ps_hx_write),
    byte-identical to `encode`. A matrix is staged whole in device memory (model load,
    before the capped arena exists); `src` is its pinned host address or a device
    filler fill(dst_dev, r0, r1) (host_format='coded' generation)."""

    def __init__(self):
        import torch

        from . import lib as L
        self.L, self.torch = L, torch
        self.stream = torch.cuda.current_stream().cuda_stream

    def _stage(self, src, n: int, k: int):
        t = self.torch.empty(n * k, dtype=self.torch.int16, device="cuda")
        if callable(src):
            step = max(1, (256 << 20) // (2 * k))
            for r0 in range(0, n, step):
                src(t.data_ptr() + r0 * k * 2, r0, min(n, r0 + step))
        else:
            self.L.memcpy_async(t.data_ptr(), src, n * k * 2, self.stream)
        return t

    def _sizes(self, bits, n: int, k: int, table: np.ndarray | None):
        torch, L = self.torch, self.L
        rowmax = torch.empty(n, dtype=torch.int32, device="cuda")
        hist = torch.zeros(256, dtype=torch.int64, device="cuda")
        L.call("ps_hx_stats", bits.data_ptr(), n, k, k, rowmax.data_ptr(), hist.data_ptr(), self.stream)
        if table is None:
            table = canonical_table(code_lengths(hist.cpu().numpy()))
        tab = torch.from_numpy(table.view(np.int32)).cuda()
        sublen = torch.empty(n * (k // SUB), dtype=torch.int16, device="cuda")
        rowbytes = torch.empty(n, dtype=torch.int32, device="cuda")
        L.call("ps_hx_sizes", bits.data_ptr(), n, k, k, rowmax.data_ptr(), tab.data_ptr(), sublen.data_ptr(),
               rowbytes.data_ptr(), self.stream)
        return table, tab, rowmax, sublen, rowbytes

    def histogram(self, src, n: int, k: int) -> np.ndarray:
        """Histogram (int64 [256]) of d = rowmax - exponent over a matrix."""
        torch, L = self.torch, self.L
        bits = self._stage(src, n, k)
        rowmax = torch.empty(n, dtype=torch.int32, device="cuda")
        hist = torch.zeros(256, dtype=torch.int64, device="cuda")
        L.call("ps_hx_stats", bits.data_ptr(), n, k, k, rowmax.data_ptr(), hist.data_ptr(), self.stream)
        return hist.cpu().numpy()

    def plan(self, src, n: int, k: int, table: np.ndarray | None = None) -> HxMatrix:
        """Layout of the matrix coded with its own Huffman code, or with `table` (a code
        shared by several matrices, e.g. the experts of one MoE layer)."""
        bits = self._stage(src, n, k)
        table, _, _, _, rowbytes = self._sizes(bits, n, k, table)
        rb = rowbytes.cpu().numpy().view(np.uint32).astype(np.uint64)
        nb = -(-n // BLOCK_ROWS)
        per_block = np.zeros(nb, np.uint64)
        np.add.at(per_block, np.arange(n) // BLOCK_ROWS, rb)
        block_off = np.zeros(nb + 1, np.uint64)
        np.cumsum(per_block + 256, out=block_off[1:])
        return HxMatrix(n, k, table, block_off)

    def write(self, src, m: HxMatrix, dst_host: int) -> None:
        """Encode the matrix again (same table) and copy its m.nbytes bytes to dst_host."""
        torch, L = self.torch, self.L
        n, k = m.n, m.k
        bits = self._stage(src, n, k)
        _, tab, rowmax, sublen, rowbytes = self._sizes(bits, n, k, m.table)
        rb = rowbytes.cpu().numpy().view(np.uint32).astype(np.uint64)
        row_off = np.empty(n, np.uint64)
        for b in range(len(m.block_off) - 1):
            r0, r1 = b * BLOCK_ROWS, min(n, (b + 1) * BLOCK_ROWS)
            row_off[r0:r1] = m.block_off[b] + 256 + np.concatenate(([0], np.cumsum(rb[r0:r1 - 1])))
        ro = torch.from_numpy(row_off.view(np.int64)).cuda()
        out = torch.zeros(m.nbytes, dtype=torch.uint8, device="cuda")
        L.call("ps_hx_write", bits.data_ptr(), n, k, k, rowmax.data_ptr(), tab.data_ptr(), sublen.data_ptr(),
               rowbytes.data_ptr(), ro.data_ptr(), out.data_ptr(), self.stream)
        L.memcpy_async(dst_host, out.data_ptr(), m.nbytes, self.stream)
        L.call("ps_stream_synchronize", self.stream)


from .wcomp import GpuEncoder  # noqa: E402  (raw-tensor copies of generated weights)


class HxShards:
    """hx-coded copies of a model's dense weight shards (attention, FFN, head) in pinned
    host memory: matrices with K % 256 == 0 as hx blobs, everything else (norm vectors)
    raw bf16, tensors 256-byte aligned in blob order. `tensors[sid][name]` = (offset,
    HxMatrix) or (offset, None) for raw bytes; `luts` holds every matrix's 16 KB decoder
    table back to back (`lut_off[(sid, name)]`), uploaded once to VRAM by the executor.

    Source: the bf16 host blob, or — host_format='coded' (runtime/model.py) — each
    tensor's deterministic init run on the GPU (no bf16 blob on the host at all).
    `shared`: a node-wide /dev/shm segment (model.SharedHostBlob): every replica plans
    the layout (GPU, ~1 s), the creator writes, the others wait for the ready flag."""

    def __init__(self, weights, kinds, shared: str | None = None):
        from ..planning.graph import ShardKind
        from . import lib as L
        self.host, self.seg = 0, None
        layout = weights.layout
        generated = getattr(weights, "host_format", "bf16") == "coded"
        enc = GpuHxEncoder()
        up = lambda n: (n + 255) // 256 * 256  # noqa: E731

        def source(sid, name):
            t = layout.blobs[sid].tensors[name]
            if generated:
                return weights.tensor_filler(t, enc.stream)
            return weights.tensor_ptr(sid, name)

        self.tensors, self.shard_off, self.shard_bytes, self.lut_off = {}, {}, {}, {}
        self.experts = {}      # MoE group sid -> expert span geometry (see _plan_experts)
        luts, off = [], 0
        for sid, blob in layout.blobs.items():
            if blob.kind is ShardKind.MOE_EXPERT_GROUP and blob.kind in kinds:
                geo = self._plan_experts(enc, source, sid, blob, luts)
                if geo is not None:
                    self.experts[sid] = geo
                    self.shard_off[sid] = off
                    self.shard_bytes[sid] = geo["n_experts"] * geo["stride"]
                    off += self.shard_bytes[sid]
                continue
            if blob.kind not in kinds:
                continue
            self.shard_off[sid] = off
            t_off, meta = 0, {}
            for name, t in blob.tensors.items():
                if t.rows > 1 and t.cols % SUB == 0:
                    m = enc.plan(source(sid, name), t.rows, t.cols)
                    meta[name] = (t_off, m)
                    self.lut_off[(sid, name)] = len(luts) * m.lut.nbytes
                    luts.append(m.lut)
                    t_off += up(m.nbytes)
                else:
                    meta[name] = (t_off, None)
                    t_off += up(t.rows * t.cols * 2)
            self.tensors[sid] = meta
            self.shard_bytes[sid] = t_off
            off += t_off
        self.nbytes = max(1, off)
        self.luts = np.concatenate(luts) if luts else np.zeros(8, np.uint16)
        if shared is not None:
            from .model import SharedHostBlob
            self.seg = SharedHostBlob(shared, self.nbytes)
            self.host = self.seg.addr
            if not self.seg.creator:
                try:
                    self.seg.wait_ready()          # another replica of this node writes
                except BaseException:
                    self.close()
                    raise
                return
        else:
            self.host = L.host_alloc(self.nbytes, mapped=True)
        try:
            for sid, geo in self.experts.items():
                self._write_experts(enc, source, sid, geo)
            for sid, meta in self.tensors.items():
                for name, (o, m) in meta.items():
                    dst = self.host + self.shard_off[sid] + o
                    t = layout.blobs[sid].tensors[name]
                    if m is not None:
                        enc.write(source(sid, name), m, dst)
                    elif generated:
                        GpuEncoder(chunk_bytes=max(1 << 20, t.rows * t.cols * 2)).bf16_to(
                            source(sid, name), t.rows, t.cols, dst)
                    else:
                        import ctypes
                        ctypes.memmove(dst, weights.tensor_ptr(sid, name), t.rows * t.cols * 2)
        except BaseException:
            self.close()
            raise
        if self.seg is not None:
            self.seg.mark_ready()

    def _plan_experts(self, enc, source, sid, blob, luts) -> dict | None:
        """Routed experts of one MoE group, hx-coded with one Huffman code per matrix kind
        (gate/up, down) shared by the group's experts, so one decoder table serves every
        expert a layer routes to. Expert e is a uniform-stride span
            [uint32 block offsets of gate/up, then of down | pad to 256]
            [gate/up hx, padded to the group's largest][down hx, padded likewise]
        (the padding is < 0.5 % here), so the fetcher copies expert e from e * stride, and
        the expansion kernel finds each block from the offsets that travel with it."""
        layer = blob.layer
        names = {kind: [f"L{layer}.e{e}.{kind}" for e in range(sum(1 for n in blob.tensors
                                                                   if n.endswith(".wgu")))]
                 for kind in ("wgu", "wdown")}
        ts = {n: blob.tensors[n] for kind in names for n in names[kind]}
        if any(t.cols % SUB for t in ts.values()):
            return None
        plans, tables = {}, {}
        for kind, ns in names.items():
            hist = sum(enc.histogram(source(sid, n), ts[n].rows, ts[n].cols) for n in ns)
            tables[kind] = canonical_table(code_lengths(hist))
            for n in ns:
                plans[n] = enc.plan(source(sid, n), ts[n].rows, ts[n].cols, table=tables[kind])
        up = lambda v: (v + 255) // 256 * 256  # noqa: E731
        g0 = plans[names["wgu"][0]]
        d0 = plans[names["wdown"][0]]
        nb_gu, nb_dn = len(g0.block_off) - 1, len(d0.block_off) - 1
        H = up(4 * (nb_gu + nb_dn))
        G = up(max(plans[n].nbytes for n in names["wgu"]))
        D = up(max(plans[n].nbytes for n in names["wdown"]))
        geo = {"n_experts": len(names["wgu"]), "stride": H + G + D, "gu_off": H, "dn_off": H + G,
               "nb_gu": nb_gu, "nb_dn": nb_dn, "gu_rows": g0.n, "dn_rows": d0.n, "gu_k": g0.k, "dn_k": d0.k,
               "names": names, "plans": plans, "actual_bytes": sum(H + plans[g].nbytes + plans[d].nbytes
                                                                   for g, d in zip(names["wgu"], names["wdown"]))}
        for kind in ("wgu", "wdown"):
            lut = pair_table(tables[kind])
            self.lut_off[(sid, kind)] = len(luts) * lut.nbytes
            luts.append(lut)
        return geo

    def _write_experts(self, enc, source, sid, geo) -> None:
        import ctypes
        base = self.host + self.shard_off[sid]
        ctypes.memset(base, 0, self.shard_bytes[sid])
        for e, (g, d) in enumerate(zip(geo["names"]["wgu"], geo["names"]["wdown"])):
            span = base + e * geo["stride"]
            mg, md = geo["plans"][g], geo["plans"][d]
            hdr = np.concatenate([mg.block_off[:-1], md.block_off[:-1]]).astype(np.uint32)
            ctypes.memmove(span, hdr.ctypes.data, hdr.nbytes)
            enc.write(source(sid, g), mg, span + geo["gu_off"])
            enc.write(source(sid, d), md, span + geo["dn_off"])

    @property
    def hx_bytes(self) -> int:
        """Bytes of the dense shards' hx copies."""
        return sum(self.shard_bytes[sid] for sid in self.tensors)

    def shard_ptr(self, sid: int) -> int:
        return self.host + self.shard_off[sid]

    def close(self) -> None:
        from . import lib as L
        if self.seg is not None:
            self.seg.close()
            self.seg, self.host = None, 0
        elif self.host:
            L.host_free(self.host)
            self.host = 0
