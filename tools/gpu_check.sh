#!/bin/bash
# One GPU session: kernel parity, engine parity, smoke. Logs -> gpurun_out/
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -m gpu -p no:cacheprovider 2>&1 | tail -60 > gpurun_out/kernels.log
timeout 600 python -m pytest tests/test_engine_gpu.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -60 > gpurun_out/engine.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
for f in kernels engine smoke; do echo == $f; tail -n 3 gpurun_out/$f.log; done
