"""Copy-engine weight streamer: a byte ring in VRAM fed by cudaMemcpyAsync.

Row a17 of SURVEY.md §8. The reference models streaming as a two-slot
double buffer — upload k waits for upload k-1 and for the compute of
streamed shard k-2 to release its slot (`pkg/src/shardplan/simulator.py:156-175`).
This build generalises it to an N-deep ring of variable-size pieces:

* pieces are byte ranges of the pinned host blob (row-aligned slices of a
  shard, <= `chunk_bytes`), copied on a dedicated H2D stream;
* each piece records an `arrived` event on the copy stream; the compute
  stream waits on it right before the kernel that reads the piece;
* each piece's region is released by events recorded after its last
  consumer (compute, or the D2H KV write-back); a new piece waits on the
  release events of every older region it overlaps before its copy starts.

The copy stream therefore runs as far ahead of compute as the ring allows
(across shards and across passes), which keeps the copy engine busy
back-to-back — the property the roofline of every BASELINE config rests on.
"""

from __future__ import annotations

from collections import deque

from ..planning.faults import ShardPlanError
from . import lib as L


class RingTooSmall(ShardPlanError):
    """A piece would overwrite a region whose consumers are not yet enqueued."""


class EventPool:
    """Round-robin CUDA events; a record is always consumed long before reuse."""

    def __init__(self, n: int = 8192):
        self.events = [L.event_create(False) for _ in range(n)]
        self.i = 0

    def next(self) -> int:
        ev = self.events[self.i]
        self.i = (self.i + 1) % len(self.events)
        return ev


class Region:
    __slots__ = ("start", "end", "release", "sealed", "tag")

    def __init__(self, start: int, end: int, tag: str):
        self.start, self.end, self.tag = start, end, tag
        self.release: list[int] = []
        self.sealed = False          # True once every consumer has been enqueued


class CopyRing:
    def __init__(self, base: int, capacity: int, h2d_stream: int, events: EventPool):
        self.base, self.capacity = base, capacity
        self.stream = h2d_stream
        self.events = events
        self.head = 0
        self.live: deque[Region] = deque()
        self.bytes_copied = 0
        self.copies = 0
        self.tracer = None
        self.striper = None        # runtime.striping.StripeLeader on a striped node

    def _reserve(self, nbytes: int, tag: str) -> Region:
        n = (nbytes + 255) // 256 * 256
        if n > self.capacity:
            raise RingTooSmall(f"piece '{tag}' of {n} B exceeds the {self.capacity} B ring")
        start = self.head if self.head + n <= self.capacity else 0
        end = start + n
        keep: deque[Region] = deque()
        waits: list[int] = []
        for r in self.live:
            if r.start < end and start < r.end:
                if not r.sealed:
                    raise RingTooSmall(
                        f"ring of {self.capacity} B too small: piece '{tag}' would overwrite "
                        f"'{r.tag}' whose consumers are not enqueued yet")
                waits.extend(r.release)
            else:
                keep.append(r)
        self.live = keep
        for ev in waits:
            L.call("ps_stream_wait_event", self.stream, ev)
        region = Region(start, end, tag)
        self.live.append(region)
        self.head = end
        return region

    def upload(self, src_host: int, nbytes: int, tag: str, reserve: int = 0
               ) -> tuple[Region, int, int]:
        """Copy `nbytes` from pinned host memory into a region of
        max(nbytes, reserve) bytes. Returns (region, device address, arrived): an
        event, or (event, stripe sequence) for a piece striped across GPUs."""
        region = self._reserve(max(nbytes, reserve), tag)
        dst = self.base + region.start
        tr = self.tracer
        ev0 = tr.begin(self.stream) if tr is not None and nbytes else None
        seq = None
        if self.striper is not None and self.striper.covers(src_host, nbytes):
            # stripe 0 here, stripes 1.. by the helper GPUs (runtime/striping.py)
            seq = self.striper.upload(dst, src_host, nbytes, self.stream)
        else:
            L.memcpy_async(dst, src_host, nbytes, self.stream)
        if ev0 is not None:
            tr.end(f"{tag} ({nbytes >> 20} MiB)", "h2d", ev0, self.stream)
        ev = self.events.next()
        L.call("ps_event_record", ev, self.stream)
        self.bytes_copied += nbytes
        self.copies += 1
        # "arrived" is the copy-stream event, plus the helpers' sequence when striped
        return region, dst, (ev if seq is None else (ev, seq))

    def upload_runs(self, src_base: int, runs: list, nbytes: int, tag: str) -> tuple[Region, int, int]:
        """One region of `nbytes` filled by several copies: runs = [(offset, bytes)] of
        the host range at `src_base`, each landing at the same offset in the region (a
        paged KV window: pages keep their pool offsets). Returns (region, device
        address, arrived event)."""
        region = self._reserve(max(1, nbytes), tag)
        dst = self.base + region.start
        tr = self.tracer
        total = sum(n for _, n in runs)
        ev0 = tr.begin(self.stream) if tr is not None and total else None
        for off, n in runs:
            L.memcpy_async(dst + off, src_base + off, n, self.stream)
        if ev0 is not None:
            tr.end(f"{tag} ({total >> 20} MiB, {len(runs)} runs)", "h2d", ev0, self.stream)
        ev = self.events.next()
        L.call("ps_event_record", ev, self.stream)
        self.bytes_copied += total
        self.copies += len(runs)
        return region, dst, ev

    def reserve_only(self, nbytes: int, tag: str) -> tuple[Region, int]:
        """Ring space without an upload (e.g. room for appended KV rows)."""
        region = self._reserve(nbytes, tag)
        return region, self.base + region.start

    def seal(self, region: Region, release_events: list[int]) -> None:
        region.release = list(release_events)
        region.sealed = True
