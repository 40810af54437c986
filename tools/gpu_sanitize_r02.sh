#!/bin/bash
# compute-sanitizer over the concurrency code: racecheck + synccheck on the mbarrier /
# TMA / tcgen05 pipelines (bulk-copy GEMV bf16 + coded, one-pass tcgen05 GEMV, paged
# tcgen05 attention, one-token MoE kernels, hx expand's warp-shared exponent rows, the GPU
# encoders), memcheck on the engine paths that stream (ring, paged KV windows, routed-
# expert fetcher with ps_wait_flag, striping helpers, hx pieces). Summaries -> gpurun_out/san/.
mkdir -p gpurun_out/san
CS=/usr/local/cuda/bin/compute-sanitizer
K="gemv_coded_bit_identical or gemv_tc or attn_prefill or attn_decode or moe_decode or qkv_rope or hx or encoder"
for tool in racecheck synccheck; do
  timeout 1500 $CS --tool $tool --print-limit 10 python -m pytest tests/test_kernels_gpu.py -q -m gpu \
    -p no:cacheprovider -k "$K" > gpurun_out/san/$tool.log 2>&1
  echo "$tool rc=$?"
done
timeout 1800 $CS --tool memcheck --print-limit 10 python -m pytest tests/test_engine_gpu.py -q -m gpu \
  -p no:cacheprovider -k "fetched or paged or coded or striped or batched_varlen or hx" > gpurun_out/san/memcheck.log 2>&1
echo "memcheck rc=$?"
for f in gpurun_out/san/*.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|Invalid|passed|failed" $f | sort | uniq -c | head -12; done
