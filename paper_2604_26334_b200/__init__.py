"""B200-native pipelined-sharding inference (arxiv 2604.26334).

* `planning`  — the reference-compatible placement planner (`shardplan` API).
* `runtime`   — the C-ABI bindings, capped VRAM arena, copy-engine weight
  streamer and the executor that runs a plan's passes on the GPU.
* `csrc`      — hand-written sm_100a CUDA kernels behind `include/pshard.h`.
"""

__version__ = "0.1.0"
