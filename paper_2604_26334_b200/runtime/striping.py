"""NVLink-striped streaming across the GPUs of a node.

Batch-1 decode is bound by ONE host link (every config of BASELINE.json runs at
0.95-0.995 of it). A node has one PCIe link per GPU: with striping, the executing
GPU (the *leader*) splits every weight piece of its ring into N stripes; it
copies stripe 0 itself and each *helper* process (one per other GPU) copies its
stripe over its own PCIe link straight into the leader's ring through a CUDA-IPC
mapping (peer writes over NVLink / NVSwitch). The native side is
`csrc/striper.cu`; this module owns the processes and the shared memory:

* the weights live in one node-shared /dev/shm blob (`model.SharedHostBlob`),
  so every GPU can read any byte of the plan;
* a small control segment (/dev/shm) carries the leader's piece commands and the
  go-sequence its GPU writes once a ring region is free;
* `StripeLeader` plugs into `CopyRing.upload` (weight pieces only; KV caches
  live in the leader's private host memory and stay unstriped); a striped
  piece's consumer waits on the leader's own-stripe event AND on
  `ps_stripe_wait` (helpers' done flags, 2 s timeout, never a hang).

Pieces below `min_bytes` are not worth a cross-process round trip and go up
unstriped. On one GPU the same code runs N processes against one device (the
functional test); the bandwidth gain needs N physical links.
"""

from __future__ import annotations

import ctypes as C
import mmap
import os
import time

from . import lib as L


class _ShmSegment:
    def __init__(self, name: str, nbytes: int, create: bool, timeout_s: float = 120.0):
        self.path = f"/dev/shm/{name}"
        self.nbytes = nbytes
        self.creator = create
        if create:
            self.fd = os.open(self.path, os.O_CREAT | os.O_EXCL | os.O_RDWR, 0o600)
            os.ftruncate(self.fd, nbytes)
            os.posix_fallocate(self.fd, 0, nbytes)   # populated pages pin safely in parallel
        else:
            t0 = time.time()
            while True:
                try:
                    self.fd = os.open(self.path, os.O_RDWR)
                    if os.fstat(self.fd).st_size >= nbytes:
                        break
                    os.close(self.fd)
                except FileNotFoundError:
                    pass
                if time.time() - t0 > timeout_s:
                    raise TimeoutError(f"{self.path} never appeared")
                time.sleep(0.01)
        self.mm = mmap.mmap(self.fd, nbytes)
        self.addr = C.addressof(C.c_char.from_buffer(self.mm))
        L.call("ps_host_register", self.addr, nbytes, 1)

    def close(self) -> None:
        if self.addr:
            L.call("ps_host_unregister", self.addr)
            self.addr = 0
            try:
                self.mm.close()
            except BufferError:
                pass
            os.close(self.fd)
            if self.creator:
                try:
                    os.unlink(self.path)
                except FileNotFoundError:
                    pass


def ctl_bytes() -> int:
    n = C.c_longlong()
    L.call("ps_stripe_ctl_bytes", C.byref(n))
    return n.value


class StripeLeader:
    """Leader side of a stripe group of `n_helpers` helper processes."""

    def __init__(self, ctl_name: str, n_helpers: int, min_bytes: int = 4 << 20, align: int = 4096):
        self.ctl = _ShmSegment(ctl_name, ctl_bytes(), create=True)
        self.n_helpers = n_helpers
        self.min_bytes = min_bytes
        self.align = align
        self.done = 0
        self.seq = 0
        self.blob_base = 0
        self.blob_bytes = 0
        self.arena_base = 0
        self.striped_pieces = 0
        self.striped_bytes = 0

    def attach(self, arena_base: int, blob_base: int, blob_bytes: int) -> None:
        """Export the leader's VRAM arena (the ring is carved from it) to the helpers."""
        done = C.c_void_p()
        L.call("ps_stripe_leader_init", self.ctl.addr, self.n_helpers, arena_base, C.byref(done))
        self.done = done.value
        self.arena_base, self.blob_base, self.blob_bytes = arena_base, blob_base, blob_bytes

    def wait_helpers(self, timeout_s: float = 120.0) -> None:
        """Block until every helper has mapped the leader's ring (after attach)."""
        n = C.c_int()
        t0 = time.time()
        while True:
            L.call("ps_stripe_ready", self.ctl.addr, C.byref(n))
            if n.value >= self.n_helpers:
                return
            if time.time() - t0 > timeout_s:
                raise TimeoutError(f"{n.value} of {self.n_helpers} stripe helpers attached")
            time.sleep(0.005)

    def covers(self, src_host: int, nbytes: int) -> bool:
        return (self.done and nbytes >= self.min_bytes and
                self.blob_base <= src_host and src_host + nbytes <= self.blob_base + self.blob_bytes)

    def upload(self, dst: int, src_host: int, nbytes: int, stream: int) -> tuple:
        """After the ring's release waits on `stream`: post the piece, signal it,
        copy stripe 0. Returns the sequence number the consumer must wait for."""
        self.seq = (self.seq + 1) & 0xFFFFFFFF or 1
        n = self.n_helpers + 1
        stripe = -(-nbytes // n)
        stripe = -(-stripe // self.align) * self.align
        L.call("ps_stripe_post", self.ctl.addr, self.seq, src_host - self.blob_base, dst - self.arena_base,
               nbytes, stripe)
        L.call("ps_stripe_signal", self.ctl.addr, self.seq, stream)
        L.memcpy_async(dst, src_host, min(stripe, nbytes), stream)
        self.striped_pieces += 1
        self.striped_bytes += nbytes
        return self.seq

    def wait(self, seq: int, stream: int) -> None:
        L.call("ps_stripe_wait", self.done, self.n_helpers, seq, stream)

    def error_seq(self) -> int:
        v = C.c_uint()
        L.call("ps_stripe_error", self.done, C.byref(v))
        return v.value

    def close(self) -> None:
        if self.ctl.addr:
            L.call("ps_stripe_stop", self.ctl.addr)
            time.sleep(0.05)
            if self.done:
                L.call("ps_stripe_leader_free", self.done)
                self.done = 0
            self.ctl.close()


def helper_main(ctl_name: str, j: int, blob_name: str, blob_bytes: int) -> int:
    """Helper process body: map the control block and the node-shared weight blob,
    serve stripe j of every posted piece until the leader stops; returns bytes copied."""
    L.lib()
    ctl = _ShmSegment(ctl_name, ctl_bytes(), create=False)
    blob = _ShmSegment(blob_name, blob_bytes, create=False)
    copied = C.c_longlong()
    try:
        L.call("ps_stripe_helper_run", ctl.addr, j, blob.addr, C.byref(copied))
    finally:
        blob.close()
        ctl.close()
    return copied.value
