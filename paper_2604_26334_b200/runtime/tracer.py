"""Copy / compute overlap timeline from CUDA events (nsys is not installed).

When a `Tracer` is attached to an executor, every ring upload (copy-engine
stream), every kernel group of a consumer (compute stream) and every KV
write-back (D2H stream) is bracketed by timing events. `dump()` converts them
to a Chrome trace (chrome://tracing / Perfetto) and `summary()` reports, over
the traced window, how busy the copy engine was and how much compute ran while
a copy was in flight — the evidence that the stream hides the math.
"""

from __future__ import annotations

import json

from . import lib as L


class Tracer:
    def __init__(self):
        self.spans: list = []      # (name, lane, ev_begin, ev_end)
        self.base = None

    def begin(self, stream: int) -> int:
        ev = L.event_create(True)
        L.call("ps_event_record", ev, stream)
        if self.base is None:
            self.base = ev
        return ev

    def end(self, name: str, lane: str, ev0: int, stream: int) -> None:
        ev1 = L.event_create(True)
        L.call("ps_event_record", ev1, stream)
        self.spans.append((name, lane, ev0, ev1))

    def _resolved(self):
        out = []
        for name, lane, e0, e1 in self.spans:
            L.call("ps_event_synchronize", e1)
            t0 = L.event_elapsed_ms(self.base, e0) * 1e3
            t1 = L.event_elapsed_ms(self.base, e1) * 1e3
            out.append((name, lane, t0, t1))
        return out

    def dump(self, path: str) -> dict:
        spans = self._resolved()
        events = [{"name": n, "ph": "X", "pid": 0, "tid": lane, "ts": round(t0, 3),
                   "dur": round(max(0.0, t1 - t0), 3)} for n, lane, t0, t1 in spans]
        with open(path, "w") as fh:
            json.dump({"traceEvents": events, "displayTimeUnit": "ms"}, fh)
        return self.summary(spans)

    def summary(self, spans=None) -> dict:
        spans = spans if spans is not None else self._resolved()
        if not spans:
            return {}

        def union(iv):
            iv = sorted(iv)
            merged = []
            for a, b in iv:
                if merged and a <= merged[-1][1]:
                    merged[-1][1] = max(merged[-1][1], b)
                else:
                    merged.append([a, b])
            return merged

        def total(m):
            return sum(b - a for a, b in m)

        def intersect(m1, m2):
            i = j = 0
            s = 0.0
            while i < len(m1) and j < len(m2):
                a, b = max(m1[i][0], m2[j][0]), min(m1[i][1], m2[j][1])
                if b > a:
                    s += b - a
                if m1[i][1] < m2[j][1]:
                    i += 1
                else:
                    j += 1
            return s

        copy = union([(t0, t1) for _, lane, t0, t1 in spans if lane == "h2d"])
        comp = union([(t0, t1) for _, lane, t0, t1 in spans if lane == "compute"])
        start = min(t0 for _, _, t0, _ in spans)
        end = max(t1 for _, _, _, t1 in spans)
        window = end - start
        return {"window_us": round(window, 1),
                "copy_engine_busy_frac": round(total(copy) / window, 4),
                "compute_busy_frac": round(total(comp) / window, 4),
                "compute_hidden_under_copy_frac": round(intersect(copy, comp) / max(total(comp), 1e-9), 4),
                "spans": len(spans)}

    def close(self) -> None:
        for _, _, e0, e1 in self.spans:
            L.call("ps_event_destroy", e0)
            L.call("ps_event_destroy", e1)
        self.spans = []
