#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -m gpu -p no:cacheprovider -k "coded" 2>&1 | tail -30 > gpurun_out/kcoded.log
timeout 600 python -m pytest tests/test_engine_gpu.py -q -m gpu -p no:cacheprovider -x -k "batched_gemm or prefill_decode_api or coded" 2>&1 | tail -150 > gpurun_out/engine2.log
timeout 2400 python -m pytest tests/test_full_size_gpu.py -q -m gpu -p no:cacheprovider -k "config2 or config4 or config3" 2>&1 | grep -E "^E |Error|assert|passed|failed" | head -80 > gpurun_out/fullsize2.log
timeout 300 python tools/bench_wcomp.py > gpurun_out/bench_wcomp.jsonl 2>&1
tail -5 gpurun_out/kcoded.log; tail -30 gpurun_out/engine2.log; cat gpurun_out/fullsize2.log; cat gpurun_out/bench_wcomp.jsonl
