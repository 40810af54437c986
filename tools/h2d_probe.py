"""Host->device copy bandwidth vs number of concurrent copy streams (copy engines).
Pinned source, 1 GiB total per trial split evenly across S streams, best of 5."""
import json, sys
import torch
sys.path.insert(0, ".")
from paper_2604_26334_b200.runtime import lib as L
total = 1 << 30
host = L.host_alloc(total, mapped=False)
dev = torch.empty(total, dtype=torch.uint8, device="cuda")
streams = [L.stream_create() for _ in range(8)]
evs = [L.event_create(True) for _ in range(16)]
for S in (1, 2, 3, 4, 8):
    for chunk_mb in (16, 64, 1024):
        best = 0.0
        for _ in range(5):
            torch.cuda.synchronize()
            start = L.event_create(True)
            L.call("ps_event_record", start, streams[0])
            for s in streams[1:S]:
                L.call("ps_stream_wait_event", s, start)
            per = total // S
            chunk = min(chunk_mb << 20, per)
            for i in range(S):
                off = i * per
                done = 0
                while done < per:
                    n = min(chunk, per - done)
                    L.memcpy_async(dev.data_ptr() + off + done, host + off + done, n, streams[i])
                    done += n
            ends = []
            for i in range(S):
                L.call("ps_event_record", evs[i], streams[i]); ends.append(evs[i])
            for e in ends:
                L.call("ps_event_synchronize", e)
            t = max(L.event_elapsed_ms(start, e) for e in ends) / 1e3
            best = max(best, total / t / 1e9)
        print(json.dumps({"streams": S, "chunk_MB": chunk_mb, "GBps": round(best, 2)}), flush=True)
