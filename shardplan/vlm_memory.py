"""`shardplan.vlm_memory` — OUT OF SCOPE in this build.

The vision-encoder peak-memory model (`pkg/src/shardplan/vlm_memory.py`)
is not on the LLM streaming path. The names exist so modules
importing them load; every call raises NotImplementedError.
"""


def _out_of_scope(*_a, **_k):
    raise NotImplementedError("the VLM memory model is out of scope in this build "
                              "(SURVEY.md §2, DESIGN.md §7)")


class VisionSpec:  # noqa: D101
    def __init__(self, *a, **k):
        _out_of_scope()


(choose_chunk, flash_attn_peak_bytes, load_vision, naive_attn_peak_bytes, peak_vram,
 vision_encode_time, vision_peak_bytes, vision_token_count, vision_from_dict, vision_to_dict,
 save_vision, query_chunk_candidates) = (_out_of_scope,) * 12
