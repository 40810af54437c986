"""Concurrent host -> device bandwidth on N GPUs of one node — the denominator of the
batched-mode (replica) and striped-streaming rooflines on 2/4/8 B200s (SURVEY.md §7 hard
part 9). Run with one process per GPU:

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/h2d_multi_gpu.py

Each rank pins 1 GiB of host memory (on its own), times pinned cudaMemcpyAsync H2D alone
(rank by rank, the others idle) and then all ranks at once after a barrier (gloo
bookkeeping, no NCCL); rank 0 prints one JSON line with per-rank GB/s and the aggregate.
Works at N = 1 (this pool's boxes)."""
import json
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26334_b200.runtime import lib as L  # noqa: E402

rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
if world > 1:
    dist.init_process_group("gloo")
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
nbytes, reps = 1 << 30, 5
host = L.host_alloc(nbytes, mapped=False)
dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
s = L.stream_create()
e0, e1 = L.event_create(True), L.event_create(True)


def best():
    out = 0.0
    for _ in range(reps):
        L.call("ps_event_record", e0, s)
        L.memcpy_async(dev.data_ptr(), host, nbytes, s)
        L.call("ps_event_record", e1, s)
        L.call("ps_event_synchronize", e1)
        out = max(out, nbytes / (L.event_elapsed_ms(e0, e1) / 1e3) / 1e9)
    return out


alone = [0.0] * world
for r in range(world):
    if world > 1:
        dist.barrier()
    if r == rank:
        alone[r] = best()
together_t0 = time.time()
if world > 1:
    dist.barrier()
together = best()
vals = torch.tensor([alone[rank], together], dtype=torch.float64)
if world > 1:
    allv = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(allv, vals)
else:
    allv = [vals]
if rank == 0:
    print(json.dumps({"gpus": world, "bytes": nbytes, "alone_gbs": [round(float(v[0]), 2) for v in allv],
                      "together_gbs": [round(float(v[1]), 2) for v in allv],
                      "aggregate_together_gbs": round(sum(float(v[1]) for v in allv), 2),
                      "how": "pinned cudaMemcpyAsync 1 GiB, best of 5 per rank; 'together' = all ranks at once"}))
L.host_free(host)
if world > 1:
    dist.destroy_process_group()
