"""Where does the host link sit idle? Reads a CUPTI chrome trace (tools/cupti_trace.py)
and reports the link's idle gaps (no H2D copy in flight on any stream) and which
kernels ran during them.

    python tools/trace_gaps.py gpurun_out/cupti_cfg3.json [--min-us 2]"""
import argparse
import collections
import gzip
import json

ap = argparse.ArgumentParser()
ap.add_argument("trace")
ap.add_argument("--min-us", type=float, default=2.0)
ap.add_argument("--show", type=int, default=3)
a = ap.parse_args()
op = gzip.open if a.trace.endswith(".gz") else open
d = json.load(op(a.trace))
ev = d["traceEvents"] if isinstance(d, dict) else d
copies = sorted((e["ts"], e["ts"] + e["dur"]) for e in ev
                if e.get("cat") == "gpu_memcpy" and "HtoD" in e.get("name", ""))
kernels = sorted((e["ts"], e["ts"] + e["dur"], e["name"].split("(")[0].split("<")[0][-48:]) for e in ev
                 if e.get("cat") == "kernel")
busy, gaps = 0.0, []
cur0, cur1 = copies[0]
for s, e in copies[1:]:
    if s > cur1:
        busy += cur1 - cur0
        if s - cur1 >= a.min_us:
            gaps.append((cur1, s))
        cur0, cur1 = s, e
    else:
        cur1 = max(cur1, e)
busy += cur1 - cur0
span = copies[-1][1] - copies[0][0]
by = collections.defaultdict(float)
for g0, g1 in gaps:
    for s, e, n in kernels:
        ov = min(e, g1) - max(s, g0)
        if ov > 0:
            by[n] += ov
hist = collections.Counter(min(int((g1 - g0) // 10) * 10, 200) for g0, g1 in gaps)
print(json.dumps({"span_us": round(span, 1), "link_busy_us": round(busy, 1), "busy_frac": round(busy / span, 4),
                  "gaps": len(gaps), "gap_us": round(sum(g1 - g0 for g0, g1 in gaps), 1),
                  "gap_hist_10us": dict(sorted(hist.items())),
                  "kernel_us_in_gaps": {k: round(v, 1) for k, v in sorted(by.items(), key=lambda kv: -kv[1])[:15]}},
                 indent=1))
for g0, g1 in sorted(gaps, key=lambda g: g[0] - g[1])[:a.show]:
    print(f"gap {g1 - g0:.1f} us")
    for s, e, n in kernels:
        if e > g0 - 20 and s < g1:
            print(f"   {s - g0:8.1f} {e - s:7.1f}  {n}")
