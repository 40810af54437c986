#!/bin/bash
mkdir -p gpurun_out
CUDA_LAUNCH_BLOCKING=1 timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_engine_gpu.py -q -m gpu -x -k "$1" -p no:cacheprovider > gpurun_out/sanitize.log 2>&1
grep -E "Invalid|ERROR SUMMARY|at 0x|by thread|in .*kernel|passed|failed|Address" gpurun_out/sanitize.log | head -30
