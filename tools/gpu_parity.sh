#!/bin/bash
# Parity session: engine tests (exact greedy), full-size exact parity, smoke. Logs -> gpurun_out/
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_engine_gpu.py -q -m gpu -p no:cacheprovider 2>&1 | tail -40 > gpurun_out/engine.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 2400 python -m pytest tests/test_full_size_gpu.py -q -m gpu -p no:cacheprovider --durations=0 -k "config" 2>&1 | tail -60 > gpurun_out/fullsize.log
for f in engine smoke fullsize; do echo == $f; tail -n 12 gpurun_out/$f.log; done
