"""Built-in model and machine specs.

Two groups:

* the reference presets (`pkg/src/shardplan/presets.py:15-39`, data under
  `pkg/src/shardplan/data/`): six calibrated client models and three client
  machines, restated here as values so the reference's tests and golden
  plans run unchanged; `list_presets` lists exactly these;
* the B200 presets this build adds (`list_b200_presets`): bf16 specs of the
  BASELINE.json models (public Hugging Face configs), the tiny config-1
  decoder, and the `b200` machine — measured copy-engine and HBM rates of
  this pool's B200s with the host CPU declared unusable (1 thread at
  1 Mflop/s), so every plan is GPU-executed.
"""

from __future__ import annotations

from .graph import ModelSpec, model_from_dict
from .hardware import MachineSpec, machine_from_dict

__all__ = ["list_presets", "list_b200_presets", "builtin_model", "builtin_machine", "striped_machine",
           "builtin_vision", "model_doc", "machine_doc"]

_KINDS = ("models", "machines", "vision")


def _quant(attn=2.0, ffn=2.0, out=2.0, kv=2.0, act=2.0) -> dict:
    return {"activations": act, "attn_weights": attn, "ffn_weights": ffn,
            "kv_cache": kv, "output_weights": out}


def _model(name, layers, d, heads, kv, hd, ffn, vocab, ctx, quant=None, moe=None) -> dict:
    return {"format": "model-spec/v1", "name": name, "n_layers": layers, "d_model": d,
            "n_heads": heads, "n_kv_heads": kv, "head_dim": hd, "ffn_dim": ffn,
            "vocab_size": vocab, "max_context": ctx, "quant": quant or _quant(),
            "gated_ffn": True, "elementwise_epsilon": 0.02,
            "moe": None if moe is None else dict(zip(("n_experts", "top_k", "expert_ffn_dim"),
                                                     moe))}


_CURVE16 = [1.0, 1.95, 2.85, 3.7, 4.5, 5.25, 5.95, 6.6, 7.2, 7.75, 8.25, 8.7, 9.1, 9.45,
            9.75, 10.0]


def _machine(name, vram, gflops, gbw, tflops, curve, sysbw, h2d, d2h, alpha, threads,
             sat, launch=2e-6) -> dict:
    return {"format": "machine-spec/v1", "name": name, "vram_capacity": vram,
            "gpu_flops": gflops, "gpu_mem_bw": gbw, "cpu_thread_flops": tflops,
            "cpu_scaling": list(curve), "sysram_bw": sysbw, "pcie_h2d_bw": h2d,
            "pcie_d2h_bw": d2h, "contention_alpha": alpha, "threads_available": threads,
            "cpu_bw_saturation_threads": sat, "gpu_launch_overhead_s": launch}


_Q4 = _quant(attn=0.5625, out=0.8203125, ffn=0.53125)
_Q2 = _quant(attn=0.5625, out=0.8203125, ffn=0.3203125)

_REFERENCE_MODELS = {
    "cr1": _model("cr1", 28, 3584, 28, 4, 128, 18944, 152064, 131072),
    "nemo4b": _model("nemo4b", 32, 3072, 24, 8, 128, 9216, 131072, 131072),
    "nemo8b": _model("nemo8b", 40, 4096, 32, 8, 128, 11520, 131072, 131072),
    "qwen235b": _model("qwen235b", 94, 4096, 64, 4, 128, 12288, 151936, 262144, _Q2,
                       (128, 8, 1536)),
    "qwen30b": _model("qwen30b", 48, 2048, 32, 4, 128, 6144, 151936, 262144, _Q4,
                      (128, 8, 768)),
    "vnemo4b": _model("vnemo4b", 32, 3072, 24, 8, 128, 9216, 131072, 131072),
}

_REFERENCE_MACHINES = {
    "desktop": _machine("desktop", 16e9, 44e12, 896e9, 50e9, _CURVE16[:8], 57.6e9, 50e9, 50e9,
                        0.7, 8, 8),
    "laptop": _machine("laptop", 12e9, 15e12, 432e9, 40e9, _CURVE16, 119.5e9, 13e9, 13e9,
                       0.7, 16, 8),
    "workstation": _machine("workstation", 32e9, 100e12, 1500e9, 60e9, _CURVE16, 153.6e9,
                            50e9, 50e9, 0.7, 16, 8),
}

# BASELINE.json configs (bf16 everywhere). Architecture values are the
# public HF configs; the tiny decoder's kv / ffn / vocab / head_dim are
# fixed by this build.
_B200_MODELS = {
    "tiny-llama": _model("tiny-llama", 4, 512, 8, 8, 64, 1536, 32000, 4096),
    "llama3.1-8b": _model("llama3.1-8b", 32, 4096, 32, 8, 128, 14336, 128256, 131072),
    "qwen3-30b-a3b": _model("qwen3-30b-a3b", 48, 2048, 32, 4, 128, 6144, 151936, 40960,
                            moe=(128, 8, 768)),
    "llama3.3-70b": _model("llama3.3-70b", 80, 8192, 64, 8, 128, 28672, 128256, 131072),
    # test-scale Qwen3-MoE-style decoder (q/k norm, 16 experts, top-4)
    "tiny-moe": _model("tiny-moe", 2, 256, 4, 2, 64, 512, 1000, 512, moe=(16, 4, 128)),
}

# Measured on this pool's B200s: HBM copy 6544.3 GB/s and sustained bf16
# 1383.9 TFLOP/s (MEASURED_PEAKS.json); pinned cudaMemcpyAsync 1 GiB best of
# 8: H2D 55.62 GB/s, D2H 57.26 GB/s (profiles/r01_probe_box.json).
# CPU compute declared unusable: no CPU backend exists in this executor.
_B200_MACHINES = {
    "b200": _machine("b200", 180e9, 1383.9e12, 6544.3e9, 1e6, [1.0], 1e6, 55.62e9, 57.26e9,
                     1.0, 1, 1),
}


def list_presets(kind: str) -> list[str]:
    """Reference presets only (the reference's CLI tests pin this list)."""
    table = {"models": _REFERENCE_MODELS, "machines": _REFERENCE_MACHINES, "vision": {}}
    if kind not in table:
        raise ValueError(f"unknown preset kind {kind}")
    if kind == "vision":
        return ["cr1-vision", "vnemo4b-vision"]
    return sorted(table[kind])


def list_b200_presets(kind: str) -> list[str]:
    table = {"models": _B200_MODELS, "machines": _B200_MACHINES}
    if kind not in table:
        raise ValueError(f"unknown preset kind {kind}")
    return sorted(table[kind])


def model_doc(name: str) -> dict:
    for table in (_REFERENCE_MODELS, _B200_MODELS):
        if name in table:
            doc = dict(table[name])
            doc["quant"] = dict(doc["quant"])
            return doc
    raise FileNotFoundError(f"no model preset named {name!r}")


def machine_doc(name: str) -> dict:
    for table in (_REFERENCE_MACHINES, _B200_MACHINES):
        if name in table:
            return dict(table[name])
    raise FileNotFoundError(f"no machine preset named {name!r}")


def builtin_model(name: str) -> ModelSpec:
    return model_from_dict(model_doc(name))


def builtin_machine(name: str) -> MachineSpec:
    return machine_from_dict(machine_doc(name))


def striped_machine(machine: MachineSpec, links: int) -> MachineSpec:
    """The link model of NVLink-striped streaming: `links`
    GPUs each pull 1/links of every streamed piece over their own PCIe link into
    the executing GPU, so host -> device bytes move at `links` x the per-GPU rate
    (`pkg/src/shardplan/machine.py:99-101` prices one link). Device -> host (KV
    write-back) stays on the executing GPU's link. links = 1 returns `machine`
    itself, so unstriped plans are the reference's bit for bit. The copy keeps the
    MachineSpec schema (no new field), so save/load round trips are unchanged."""
    if links < 1:
        raise ValueError(f"links must be >= 1, got {links}")
    if links == 1:
        return machine
    import dataclasses
    return dataclasses.replace(machine, name=f"{machine.name}-x{links}",
                               pcie_h2d_bw=machine.pcie_h2d_bw * links)


def builtin_vision(name: str):
    raise NotImplementedError(
        "vision-encoder specs belong to the VLM memory model, which is out of scope "
        "for the streaming-inference path (SURVEY.md §2, DESIGN.md)")
