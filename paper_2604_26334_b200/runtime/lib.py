"""ctypes binding of the C-ABI in include/pshard.h (libpshard.so, built in-tree).

There is no fallback: if the shared library is missing or fails to load,
importing the runtime raises. Every call's status is checked and a
non-zero status raises `PshardError` with the library's thread-local
message.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PSHARD_LIB") or os.path.join(os.path.dirname(_HERE), "_lib", "libpshard.so")

PS_EPI_STORE, PS_EPI_ACCUM, PS_EPI_SWIGLU, PS_EPI_STORE_BF16 = 0, 1, 2, 3

_p, _i, _ll, _sz, _f, _ull = C.c_void_p, C.c_int, C.c_longlong, C.c_size_t, C.c_float, C.c_ulonglong
_pp = C.POINTER(C.c_void_p)

# name -> argtypes (all return int status)
_SIGS = {
    "ps_abi_version": [],
    "ps_device_info": [_i, C.POINTER(_i), C.POINTER(_i), C.POINTER(_i), C.POINTER(_sz)],
    "ps_set_device": [_i],
    "ps_preload_kernels": [C.POINTER(_i)],
    "ps_host_alloc": [_sz, _i, _pp],
    "ps_host_free": [_p],
    "ps_host_register": [_p, _sz, _i],
    "ps_host_unregister": [_p],
    "ps_host_device_pointer": [_p, _pp],
    "ps_device_alloc": [_sz, _pp],
    "ps_device_free": [_p],
    "ps_memcpy_async": [_p, _p, _sz, _p],
    "ps_memset_async": [_p, _i, _sz, _p],
    "ps_stream_create": [_i, _pp],
    "ps_stream_destroy": [_p],
    "ps_stream_synchronize": [_p],
    "ps_device_synchronize": [],
    "ps_event_create": [_i, _pp],
    "ps_event_destroy": [_p],
    "ps_event_record": [_p, _p],
    "ps_stream_wait_event": [_p, _p],
    "ps_event_synchronize": [_p],
    "ps_event_query": [_p],
    "ps_event_elapsed_ms": [_p, _p, C.POINTER(_f)],
    "ps_gemv_bf16": [_p, _i, _i, _p, _i, _i, _ll, _p, _i, _i, _p],
    "ps_gemv_bf16_cfg": [_p, _i, _i, _p, _i, _i, _ll, _p, _i, _i, _p, _i, _i, _i],
    "ps_gemm_bf16": [_p, _i, _i, _ll, _p, _i, _ll, _p, _i, _i, _p],
    "ps_gemm_bf16_cfg": [_p, _i, _i, _ll, _p, _i, _ll, _p, _i, _i, _p, _i],
    "ps_rmsnorm": [_p, _i, _p, _i, _p, _i, _f, _p, _i, _i, _p],
    "ps_qkv_rope_append": [_p, _i, _i, _i, _i, _i, _p, _p, _p, _i, _p, _i, _i, _p, _p, _p, _f, _p],
    "ps_attn_decode": [_p, _i, _i, _i, _i, _i, _p, _p, _i, _p, _i, _i, _p, _i, _f, _p, _i, _p, _ll, _p],
    "ps_attn_prefill_tc": [_p, _i, _i, _p, _p, _p, _i, _i, _i, _i, _p, _i, _p, _i, _i, _i, _f, _p, _i, _i, _p],
    "ps_attn_tc_watchdog": [C.POINTER(C.c_uint), _i],
    "ps_fault_status": [C.POINTER(C.c_uint), _i],
    "ps_attn_decode_workspace": [_i, _i, _i, _i, C.POINTER(_ll)],
    "ps_attn_prefill": [_p, _i, _i, _p, _p, _p, _i, _i, _i, _i, _p, _i, _p, _i, _i, _f, _p, _i, _i, _p],
    "ps_upload_small": [_p, _p, _i, _p],
    "ps_moe_route_topk": [_p, _i, _i, _i, _i, _i, _p, _p, _p],
    "ps_moe_plan_ints": [_i, _i, C.POINTER(_ll)],
    "ps_moe_plan": [_p, _i, _i, _p, _p],
    "ps_moe_expert_gu": [_p, _i, _i, _p, _i, _i, _i, _p, _ll, _ll, _i, _i, _p, _i, _i, _p],
    "ps_moe_expert_down": [_p, _p, _i, _i, _p, _ll, _ll, _i, _i, _p, _i, _i, _p],
    "ps_moe_expert_gu_mapped": [_p, _i, _i, _p, _i, _i, _i, _p, _ll, _ll, _i, _i, _p, _i, _i, _p, _p],
    "ps_moe_expert_down_mapped": [_p, _p, _i, _i, _p, _ll, _ll, _i, _i, _p, _i, _i, _p, _p],
    "ps_fetcher_create": [_i, _pp],
    "ps_fetcher_destroy": [_p],
    "ps_fetcher_info": [_p, _pp, _pp, C.POINTER(_ll), C.POINTER(_ll), C.POINTER(_i)],
    "ps_fetcher_submit": [_p, C.c_uint, _p, _ll, _ll, _p, _ll],
    "ps_fetcher_submit_split": [_p, C.c_uint, _p, _ll, _ll, _p, _ll, _i],
    "ps_moe_publish": [_p, _p, _i, _i, _p, C.c_uint, _p],
    "ps_fetcher_submit_spec": [_p, C.c_uint, _p, _ll, _ll, _p, _ll, _i, _p, _ll, _ll],
    "ps_moe_publish_spec": [_p, _p, _i, _i, _p, C.c_uint, _p, _i, _p, _i, _i, _i, _p, _p],
    "ps_fetcher_seq_bytes": [_p, C.c_uint, C.POINTER(_ll)],
    "ps_wait_flag": [_p, C.c_uint, _p],
    "ps_fetcher_device_error": [_p, C.POINTER(C.c_uint)],
    "ps_stripe_ctl_bytes": [C.POINTER(_ll)],
    "ps_stripe_leader_init": [_p, _i, _p, _pp],
    "ps_stripe_leader_free": [_p],
    "ps_stripe_post": [_p, C.c_uint, _ll, _ll, _ll, _ll],
    "ps_stripe_signal": [_p, C.c_uint, _p],
    "ps_stripe_wait": [_p, _i, C.c_uint, _p],
    "ps_stripe_error": [_p, C.POINTER(C.c_uint)],
    "ps_stripe_helper_run": [_p, _i, _p, C.POINTER(_ll)],
    "ps_stripe_stop": [_p],
    "ps_stripe_ready": [_p, C.POINTER(_i)],
    "ps_moe_combine": [_p, _p, _i, _i, _p, _i, _i, _i, _p, _i, _p],
    "ps_set_pdl": [_i],
    "ps_expand_coded": [_p, _ll, _i, _i, _p, _ll, _p],
    "ps_gemv_head_early": [_p, _i, _p, _i, _ll, _i, _p, _i, _p, C.c_uint, _p],
    "ps_set_flag": [_p, C.c_uint, _p],
    "ps_wencode_stats": [_p, _i, _i, _ll, _p, _p, _p],
    "ps_wencode_rows": [_p, _i, _i, _ll, _p, _i, _p, _ll, _p],
    "ps_hx_expand": [_p, _p, _i, _i, _p, _p, _ll, _p],
    "ps_hx_expand_experts2": [_p, _ll, _p, _i, _i, _ll, _i, _i, _p, _ll, _i, _ll, _i, _i, _p, _ll, _p, _ll, _p],
    "ps_hx_stats": [_p, _i, _i, _ll, _p, _p, _p],
    "ps_hx_sizes": [_p, _i, _i, _ll, _p, _p, _p, _p, _p],
    "ps_hx_write": [_p, _i, _i, _ll, _p, _p, _p, _p, _p, _p, _p],
    "ps_gemv_tc": [_p, _i, _i, _p, _i, _i, _ll, _i, _p, _i, _i, _p, _ll, _p],
    "ps_gemv_tc_workspace": [_i, _i, C.POINTER(_ll)],
    "ps_gemv_bf16c": [_p, _i, _i, _p, _i, _i, _ll, _p, _i, _i, _p],
    "ps_moe_decode_experts": [_p, _p, _i, _p, _p, _ll, _ll, _ll, _i, _i, _p, _p, _p, _p],
    "ps_moe_decode_experts_c": [_p, _p, _i, _p, _p, _ll, _ll, _ll, _i, _i, _i, _i, _p, _p, _p, _p],
    "ps_moe_decode_experts_phase": [_p, _p, _i, _p, _p, _ll, _ll, _ll, _i, _i, _p, _p, _p, _i, _i, _i, _p],
    "ps_embed_gather": [_p, _p, _i, _i, _p, _i, _p],
    "ps_argmax": [_p, _i, _i, _i, _p, _p],
    "ps_cast_f32_bf16": [_p, _i, _p, _i, _i, _i, _p],
    "ps_add_f32": [_p, _p, _ll, _p],
    "ps_init_uniform_bf16": [_p, _sz, _ull, _ull, _f, _f, _p],
    "ps_init_rowscaled_bf16": [_p, _sz, _ull, _ull, _ll, _f, _p],
    "ps_init_interleaved_bf16": [_p, _ll, _ll, _ll, _i, _ull, _ull, _f, _f, _p],
}

EXPORTED = tuple(["ps_last_error"] + list(_SIGS))


class PshardError(RuntimeError):
    """A C-ABI call returned a non-zero status."""


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c \"import __graft_entry__ as g; g.build()\"` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    lib.ps_last_error.restype = C.c_char_p
    lib.ps_last_error.argtypes = []
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    return lib


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = _load()
    return _lib


KERNEL_CALLS = frozenset({
    "ps_gemv_bf16", "ps_gemm_bf16", "ps_rmsnorm", "ps_qkv_rope_append", "ps_attn_decode",
    "ps_attn_prefill", "ps_embed_gather", "ps_argmax", "ps_cast_f32_bf16", "ps_add_f32",
    "ps_upload_small", "ps_init_uniform_bf16", "ps_init_interleaved_bf16", "ps_init_rowscaled_bf16", "ps_gemv_bf16_cfg", "ps_gemm_bf16_cfg",
    "ps_moe_route_topk", "ps_moe_plan", "ps_moe_expert_gu", "ps_moe_expert_down", "ps_moe_combine", "ps_moe_decode_experts", "ps_moe_decode_experts_c", "ps_moe_decode_experts_phase", "ps_gemv_bf16c", "ps_gemv_tc", "ps_expand_coded", "ps_gemv_head_early", "ps_set_flag",
    "ps_wencode_stats", "ps_wencode_rows", "ps_hx_expand", "ps_hx_expand_experts2", "ps_hx_stats", "ps_hx_sizes", "ps_hx_write",
    "ps_moe_expert_gu_mapped", "ps_moe_expert_down_mapped", "ps_moe_publish", "ps_moe_publish_spec", "ps_wait_flag",
    "ps_stripe_signal", "ps_stripe_wait", "ps_attn_prefill_tc"})
counters = {"kernel_calls": 0, "memcpy_calls": 0}


def call(name: str, *args) -> int:
    if name in KERNEL_CALLS:
        counters["kernel_calls"] += 1
    elif name == "ps_memcpy_async":
        counters["memcpy_calls"] += 1
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        msg = lib().ps_last_error().decode(errors="replace")
        raise PshardError(f"{name} failed ({rc}): {msg}")
    return rc


class DeviceFault(PshardError):
    """A device-side spin-wait gave up (expert fetch, stripe, tcgen05 attention
    barrier) or the fetcher's host thread timed out: the pass's results are invalid."""


FAULT_NAMES = ("expert-fetch wait timed out at sequence", "stripe wait timed out at sequence",
               "tcgen05 attention barrier watchdog code", "fetcher host thread never saw sequence",
               "early-head GEMV flag wait timed out at pass")


def fault_status(reset: bool = False) -> tuple:
    """The five host-mapped fault words (csrc/common.cuh); a plain host read."""
    w = (C.c_uint * 5)()
    call("ps_fault_status", w, 1 if reset else 0)
    return tuple(int(x) for x in w)


def raise_on_fault() -> None:
    w = fault_status()
    if any(w):
        fault_status(reset=True)
        raise DeviceFault("; ".join(f"{n} {v:#x}" for n, v in zip(FAULT_NAMES, w) if v))


def attn_decode_workspace(batch: int, n_heads: int, head_dim: int, max_len: int) -> int:
    """Floats of workspace ps_attn_decode needs (split-KV partials)."""
    n = C.c_longlong(0)
    call("ps_attn_decode_workspace", batch, n_heads, head_dim, max_len, C.byref(n))
    return n.value


def out_ptr() -> C.c_void_p:
    return C.c_void_p()


# -- thin typed helpers ---------------------------------------------------------------

def host_alloc(nbytes: int, mapped: bool = True) -> int:
    p = C.c_void_p()
    call("ps_host_alloc", nbytes, 1 if mapped else 0, C.byref(p))
    return p.value


def host_free(ptr: int) -> None:
    call("ps_host_free", ptr)


def memcpy_async(dst: int, src: int, nbytes: int, stream: int) -> None:
    if nbytes:
        call("ps_memcpy_async", dst, src, nbytes, stream)


def stream_create(high_priority: bool = False) -> int:
    p = C.c_void_p()
    call("ps_stream_create", 1 if high_priority else 0, C.byref(p))
    return p.value


def event_create(timing: bool = False) -> int:
    p = C.c_void_p()
    call("ps_event_create", 1 if timing else 0, C.byref(p))
    return p.value


def event_elapsed_ms(a: int, b: int) -> float:
    v = C.c_float()
    call("ps_event_elapsed_ms", a, b, C.byref(v))
    return float(v.value)


def event_query(ev: int) -> bool:
    r = lib().ps_event_query(ev)
    if r < 0:
        raise PshardError(lib().ps_last_error().decode())
    return r == 1


def device_info(device: int = 0) -> dict:
    sm, ma, mi, mem = C.c_int(), C.c_int(), C.c_int(), C.c_size_t()
    call("ps_device_info", device, C.byref(sm), C.byref(ma), C.byref(mi), C.byref(mem))
    return {"sm_count": sm.value, "cc": (ma.value, mi.value), "total_mem": mem.value}
