"""Exponent-coded bf16 weights: 12 bits per weight on the host link, bit-exact.

A bf16 weight is sign (1) | exponent (8) | mantissa (7). Over the streamed
tensors of these models the exponent field takes ~25 values with ~2.1 bits of
entropy: within one row, the 15 exponents just below the row's
largest cover all but ~1e-4 of the weights. A coded [N, K] matrix is N rows of
`row_bytes(K, trailer)` bytes, each self-contained:

    K bytes      sign << 7 | mantissa                 (one per weight)
    K/2 bytes    4-bit codes, low nibble first: exponent - base_r, or 15 = escape
    T bytes      trailer, uint32 words: [0] = base_r | n_escapes << 8, then
                 n_escapes words col << 8 | exponent (ascending col), the rest
                 0xFFFFFFFF; T = 16 * ceil((1 + max escapes of any row) / 4)

base_r = max(0, largest exponent of row r - 14). Everything a row needs travels
with it, so the GEMV (`ps_gemv_bf16c`, csrc/gemv_tma.cu) resolves escapes from the
same shared-memory stage as the row — no side tables, no host-mapped reads — and
rows of very different magnitude (heavy-tailed heads, real checkpoints) each get
their own window. A matrix with a row of more than MAX_ESCAPES escapes is not
coded (streams as bf16). The kernel decodes in the consumer loop and accumulates
in the same order as `ps_gemv_bf16`, so its outputs are bit-identical while the
matrix moves ~25 % fewer bytes. `CodedShards` keeps coded copies of a model's
dense shards in pinned host memory; the executor streams them in GEMV (decode)
passes.
"""

from __future__ import annotations

import numpy as np

ESCAPE = 15
MAX_ESCAPES = 63                 # per row: trailer <= 256 bytes


def trailer_bytes(max_escapes: int) -> int:
    return 16 * -(-(1 + max_escapes) // 4)


def row_bytes(k: int, trailer: int) -> int:
    return k * 3 // 2 + trailer


def encode(bits: np.ndarray, out: np.ndarray | None = None, max_escapes: int = MAX_ESCAPES,
           trailer: int | None = None):
    """bf16 bit patterns (uint16 [N, K], K % 32 == 0) -> (coded uint8 [N, row_bytes],
    trailer bytes), or None when a row needs more than `max_escapes` escapes (or more
    than a forced `trailer` holds: experts of one MoE group share one row size). `out`:
    optional destination (uint8, at least N * row_bytes) written in place."""
    bits = np.ascontiguousarray(bits, dtype=np.uint16)
    n, k = bits.shape
    if k % 32:
        raise ValueError("K must be a multiple of 32")
    hi = (bits >> 8).astype(np.uint8)                       # sign | exponent[7:1]
    lo = bits.astype(np.uint8)                              # exponent[0] | mantissa
    exp = ((hi & 0x7F) << 1) | (lo >> 7)                    # uint8 exponent
    base = row_bases(exp)
    code = exp.astype(np.int16) - base[:, None]
    esc = (code < 0) | (code > 14)
    counts = np.count_nonzero(esc, axis=1)
    top = int(counts.max()) if n else 0
    if top > max_escapes:
        return None
    tb = trailer_bytes(top)
    if trailer is not None:
        if trailer < tb:
            return None
        tb = trailer
    rb = row_bytes(k, tb)
    coded = (np.empty((n, rb), np.uint8) if out is None else out[:n * rb].reshape(n, rb))
    np.bitwise_or(hi & 0x80, lo & 0x7F, out=coded[:, :k])
    code[esc] = ESCAPE
    code = code.astype(np.uint8)
    np.bitwise_or(code[:, 0::2], code[:, 1::2] << 4, out=coded[:, k:k + k // 2])
    trailer = coded[:, k + k // 2:].view(np.uint32)         # [n, tb / 4], row-major
    trailer[:] = 0xFFFFFFFF
    trailer[:, 0] = base.astype(np.uint32) | (counts.astype(np.uint32) << 8)
    if top:
        rows, cols = np.nonzero(esc)                        # by row, then ascending column
        first = np.zeros(n + 1, np.int64)
        np.cumsum(counts, out=first[1:])
        slot = np.arange(len(rows)) - first[rows]
        trailer[rows, 1 + slot] = (cols.astype(np.uint32) << 8) | exp[rows, cols]
    return coded, tb


def row_bases(exp: np.ndarray, recheck: int = 8) -> np.ndarray:
    """Per-row window start (int16 [N]) for uint8 exponents [N, K]: the 15 exponents
    below the row's largest; a row that would escape more than `recheck` weights that
    way (an outlier far above the bulk) gets the window covering the most weights
    (ties: the highest)."""
    base = np.maximum(exp.max(axis=1).astype(np.int16) - 14, 0)
    low = np.count_nonzero(exp.astype(np.int16) < base[:, None], axis=1)
    for r in np.nonzero(low > recheck)[0]:
        hist = np.bincount(exp[r], minlength=256)
        cover = np.convolve(hist, np.ones(15, np.int64), mode="valid")   # cover[b] = hist[b:b+15]
        base[r] = len(cover) - 1 - int(np.argmax(cover[::-1]))
    return base


def decode(coded: np.ndarray, k: int) -> np.ndarray:
    """Inverse of `encode` (CPU reference for the kernel's decoder): uint8 [N, row
    bytes] -> bf16 bits uint16 [N, K]."""
    n = coded.shape[0]
    sm = coded[:, :k].astype(np.uint32)
    nib = coded[:, k:k + k // 2]
    trailer = np.ascontiguousarray(coded[:, k + k // 2:]).view(np.uint32)
    code = np.empty((n, k), np.uint32)
    code[:, 0::2] = nib & 0xF
    code[:, 1::2] = nib >> 4
    base = (trailer[:, 0] & 0xFF)[:, None]
    exp = code + base
    for r in range(n):
        for e in trailer[r, 1:1 + (trailer[r, 0] >> 8)]:
            exp[r, e >> 8] = e & 0xFF
    return (((sm & 0x80) << 8) | ((exp & 0xFF) << 7) | (sm & 0x7F)).astype(np.uint16)


class CodedShards:
    """Exponent-coded copies of a model's dense weight shards in pinned host memory,
    for GEMV (decode) passes that stream them (`Executor`, PS_CODED=1).

    Per shard the tensors keep the blob's order, 256-byte aligned: matrices (K a
    multiple of 256) as coded rows (`tensors[sid][name] = (offset, row_bytes,
    coded)`, coded = True), norm vectors, other tensors and matrices with too many
    escapes as raw bf16 (coded = False, row_bytes = 2 K)."""

    def __init__(self, weights, kinds, threads: int = 16, shared: str | None = None, use_gpu: bool = True,
                 chunk_bytes: int = 256 << 20):
        """`shared`: name of a node-wide /dev/shm segment (model.SharedHostBlob): the
        replica that creates it encodes, the others map it and wait for the ready flag,
        so a node holds ONE coded copy however many replicas stream from it."""
        from concurrent.futures import ThreadPoolExecutor

        from . import lib as L
        layout = weights.layout
        self.host = 0
        self.seg = None
        up = lambda n: (n + 255) // 256 * 256  # noqa: E731
        from ..planning.graph import ShardKind
        moe_kind = ShardKind.MOE_EXPERT_GROUP
        # dense shards: every matrix; MoE expert groups: the expert matrices only (the
        # router and norm are read from the bf16 blob by the routing step)
        mats = [(sid, name) for sid, blob in layout.blobs.items() if blob.kind in kinds
                for name, t in blob.tensors.items() if t.rows > 1 and t.cols % 256 == 0 and
                (blob.kind is not moe_kind or ".e" in name)]

        gpu = None
        # host_format="coded" (runtime/model.py): no bf16 blob; tensors come from their
        # device-side init, generated once per pass
        generated = getattr(weights, "host_format", "bf16") == "coded"
        if use_gpu or generated:
            import torch
            if torch.cuda.is_available():
                gpu = GpuEncoder(chunk_bytes)
        if generated and gpu is None:
            raise RuntimeError("host_format='coded' encodes on the GPU")
        self.encoder = "gpu" if gpu is not None else "numpy"

        def source(sid, name):
            if generated:
                return weights.tensor_filler(layout.blobs[sid].tensors[name], gpu.stream)
            return weights.tensor_ptr(sid, name)

        def plan(job):   # the trailer each matrix needs (a counting pass, no output)
            sid, name = job
            if gpu is not None:
                t = layout.blobs[sid].tensors[name]
                top = gpu.max_escapes(source(sid, name), t.rows, t.cols)
                return job, None if top > MAX_ESCAPES else trailer_bytes(top)
            return job, _trailer_or_none(weights.host_view(sid, name))

        if gpu is not None:
            trailers = dict(plan(job) for job in mats)
        else:
            with ThreadPoolExecutor(max_workers=threads) as pool:
                trailers = dict(pool.map(plan, mats))
        # one row size per expert matrix kind within a group (uniform expert stride, so
        # the fetcher copies expert e from e * stride): the group's largest trailer
        self.experts = {}
        for sid, blob in layout.blobs.items():
            if blob.kind is not moe_kind or blob.kind not in kinds:
                continue
            for suffix in ("wgu", "wdown"):
                names = [n for n in blob.tensors if n.endswith("." + suffix) and ".e" in n]
                tbs = [trailers.get((sid, n)) for n in names]   # absent: not codable (K % 256)
                top = None if any(tb is None for tb in tbs) else max(tbs)
                for n in names:
                    trailers[(sid, n)] = top
        self.tensors, self.shard_off, self.shard_bytes = {}, {}, {}
        off = 0
        for sid, blob in layout.blobs.items():
            if blob.kind not in kinds:
                continue
            self.shard_off[sid] = off
            t_off, meta = 0, {}
            for name, t in blob.tensors.items():
                tb = trailers.get((sid, name))
                if tb is not None:
                    meta[name] = (t_off, row_bytes(t.cols, tb), True)
                    t_off += up(t.rows * row_bytes(t.cols, tb))
                else:
                    meta[name] = (t_off, t.cols * 2, False)
                    t_off += up(t.rows * t.cols * 2)
            self.tensors[sid] = meta
            self.shard_bytes[sid] = t_off
            off += t_off
            if blob.kind is moe_kind:
                self._expert_geometry(sid, blob, meta)
        self.nbytes = max(1, off)
        self.n_uncoded = sum(1 for job in mats if trailers[job] is None)
        if shared is not None:
            from .model import SharedHostBlob
            self.seg = SharedHostBlob(shared, self.nbytes)
            self.host = self.seg.addr
            if not self.seg.creator:
                if gpu is not None:
                    gpu.close()
                try:
                    self.seg.wait_ready()          # another replica of this node encodes
                except BaseException:
                    self.close()
                    raise
                self.mapped = True                 # registered mapped by SharedHostBlob
                self.coded_bytes = sum(self.shard_bytes.values())
                return
        else:
            # mapped: a CPU-placed (zero-copy) shard's GEMV reads its coded rows from here
            self.host = L.host_alloc(self.nbytes, mapped=True)
        self.mapped = True        # both private (mapped alloc) and shared (registered mapped)
        try:
            buf = np.ctypeslib.as_array((np.ctypeslib.ctypes.c_uint8 * self.nbytes).from_address(self.host))

            def work(item):
                sid, name = item
                t = layout.blobs[sid].tensors[name]
                o, rb, is_coded = self.tensors[sid][name]
                if generated:
                    dst = self.host + self.shard_off[sid] + o
                    if is_coded:
                        gpu.encode_to(source(sid, name), t.rows, t.cols, rb - t.cols * 3 // 2, dst)
                    else:
                        gpu.bf16_to(source(sid, name), t.rows, t.cols, dst)
                    return
                src = weights.host_view(sid, name)
                if is_coded and gpu is not None:
                    gpu.encode_to(source(sid, name), t.rows, t.cols, rb - t.cols * 3 // 2,
                                  self.host + self.shard_off[sid] + o)
                elif is_coded:
                    res = encode(src, out=buf[o + self.shard_off[sid]:], trailer=rb - t.cols * 3 // 2)
                    assert res is not None and res[1] == rb - t.cols * 3 // 2
                else:
                    start = self.shard_off[sid] + o
                    buf[start:start + t.rows * t.cols * 2] = src.reshape(-1).view(np.uint8)

            items = [(sid, name) for sid, meta in self.tensors.items() for name in meta]
            if gpu is not None:
                for item in items:
                    work(item)
            else:
                with ThreadPoolExecutor(max_workers=threads) as pool:
                    list(pool.map(work, items))
        except BaseException:
            self.close()
            raise
        finally:
            if gpu is not None:
                gpu.close()
        if self.seg is not None:
            self.seg.mark_ready()
        self.coded_bytes = sum(self.shard_bytes.values())

    def _expert_geometry(self, sid, blob, meta) -> None:
        """experts[sid] = (offset of expert 0 in the coded shard, expert stride, offset of
        wdown in an expert, bytes of one expert, gate/up row bytes, down row bytes), when
        every expert matrix of the group is coded."""
        layer = blob.layer
        names = [f"L{layer}.e{e}.{m}" for e in range(2) for m in ("wgu", "wdown")]
        if not all(n in meta and meta[n][2] for n in names if n in blob.tensors):
            return
        e0, d0 = meta[f"L{layer}.e0.wgu"][0], meta[f"L{layer}.e0.wdown"][0]
        stride = (meta[f"L{layer}.e1.wgu"][0] - e0) if f"L{layer}.e1.wgu" in meta else None
        if stride is None or any(not meta[n][2] for n in meta if ".e" in n):
            return
        wd = blob.tensors[f"L{layer}.e0.wdown"]
        ebytes = d0 - e0 + wd.rows * meta[f"L{layer}.e0.wdown"][1]
        self.experts[sid] = (e0, stride, d0 - e0, ebytes, meta[f"L{layer}.e0.wgu"][1],
                             meta[f"L{layer}.e0.wdown"][1])

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


class GpuEncoder:
    """`encode` on the GPU (csrc/wencode.cu: ps_wencode_stats + ps_wencode_rows), byte-
    identical to the numpy encoder: matrices go up in row chunks of <= `chunk_bytes`
    through a device staging buffer, coded rows come back with one D2H per chunk.
    Used at model load (before the capped arena exists, so the staging is not budget)."""

    def __init__(self, chunk_bytes: int = 256 << 20):
        import torch

        from . import lib as L
        self.L = L
        self.torch = torch
        self.stream = torch.cuda.current_stream().cuda_stream
        self.chunk_bytes = chunk_bytes
        self.src = torch.empty(chunk_bytes, dtype=torch.uint8, device="cuda")
        self.out = torch.empty(chunk_bytes * 3 // 4 + (chunk_bytes // 512) * 256 + 4096, dtype=torch.uint8,
                               device="cuda")
        self.rows_cap = 1 << 16
        self._ints(self.rows_cap)

    def _ints(self, n: int) -> None:
        self.base = self.torch.empty(n, dtype=self.torch.int32, device="cuda")
        self.count = self.torch.empty(n, dtype=self.torch.int32, device="cuda")
        self.rows_cap = n

    def _chunks(self, n: int, k: int):
        step = max(1, min(self.chunk_bytes // (2 * k), self.rows_cap))
        for r0 in range(0, n, step):
            yield r0, min(n, r0 + step)

    def _source(self, src, k: int):
        """fill(dst_dev, r0, r1) for a pinned host matrix address or a device filler."""
        if callable(src):
            return src
        return lambda dst, r0, r1: self.L.memcpy_async(dst, src + r0 * k * 2, (r1 - r0) * k * 2, self.stream)

    def _stats(self, fill, r0: int, r1: int, k: int) -> None:
        fill(self.src.data_ptr(), r0, r1)
        self.L.call("ps_wencode_stats", self.src.data_ptr(), r1 - r0, k, k, self.base.data_ptr(),
                    self.count.data_ptr(), self.stream)

    def max_escapes(self, src, n: int, k: int) -> int:
        """Largest per-row escape count of a bf16 matrix [n, k]: `src` is its pinned host
        address, or fill(dst_dev, r0, r1) producing its rows on the device."""
        fill, top = self._source(src, k), 0
        for r0, r1 in self._chunks(n, k):
            self._stats(fill, r0, r1, k)
            top = max(top, int(self.count[:r1 - r0].max().item()))
        return top

    def bf16_to(self, src, n: int, k: int, dst_host: int) -> None:
        """The raw bf16 rows of a device-filled matrix copied to `dst_host`."""
        fill = self._source(src, k)
        for r0, r1 in self._chunks(n, k):
            fill(self.src.data_ptr(), r0, r1)
            self.L.memcpy_async(dst_host + r0 * k * 2, self.src.data_ptr(), (r1 - r0) * k * 2, self.stream)
        self.L.call("ps_stream_synchronize", self.stream)

    def encode_to(self, src, n: int, k: int, tb: int, dst_host: int) -> None:
        """Coded rows (trailer `tb` bytes) of a bf16 matrix (`src` as in max_escapes)
        written to `dst_host` (n * row_bytes(k, tb) bytes, pinned)."""
        L = self.L
        rb = row_bytes(k, tb)
        fill = self._source(src, k)
        for r0, r1 in self._chunks(n, k):
            if (r1 - r0) * rb > self.out.numel():
                raise ValueError("GpuEncoder: output staging too small")
            self._stats(fill, r0, r1, k)
            L.call("ps_wencode_rows", self.src.data_ptr(), r1 - r0, k, k, self.base.data_ptr(), tb,
                   self.out.data_ptr(), rb, self.stream)
            L.memcpy_async(dst_host + r0 * rb, self.out.data_ptr(), (r1 - r0) * rb, self.stream)
        L.call("ps_stream_synchronize", self.stream)   # stream order protects the staging reuse

    def close(self) -> None:
        self.src = self.out = self.base = self.count = None


def _trailer_or_none(bits: np.ndarray) -> int | None:
    """Trailer bytes `encode` would use for this matrix, or None (too many escapes)."""
    bits = np.ascontiguousarray(bits, dtype=np.uint16)
    exp = ((bits >> 7) & 0xFF).astype(np.uint8)
    base = row_bases(exp)
    e = exp.astype(np.int16) - base[:, None]
    top = int(np.count_nonzero((e < 0) | (e > 14), axis=1).max()) if len(bits) else 0
    return None if top > MAX_ESCAPES else trailer_bytes(top)
