#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_engine_gpu.py -q -m gpu -p no:cacheprovider 2>&1 | tail -80 > gpurun_out/engine.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
for f in engine smoke; do echo == $f; tail -n 4 gpurun_out/$f.log; done
