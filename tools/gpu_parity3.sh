#!/bin/bash
# kernels + engine + full-size parity + coded bench; full logs -> gpurun_out/
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -m gpu -p no:cacheprovider 2>&1 > gpurun_out/k3.log
timeout 1200 python -m pytest tests/test_engine_gpu.py -q -m gpu -p no:cacheprovider 2>&1 > gpurun_out/e3.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke3.log 2>&1
timeout 2400 python -m pytest tests/test_full_size_gpu.py -q -m gpu -p no:cacheprovider --durations=0 2>&1 > gpurun_out/f3.log
timeout 300 python tools/bench_wcomp.py > gpurun_out/bench_wcomp.jsonl 2>&1
for f in k3 e3 f3; do echo "== $f"; grep -E "^E  |^FAILED|passed|failed" gpurun_out/$f.log | cut -c1-400 | head -40; done
tail -2 gpurun_out/smoke3.log; cat gpurun_out/bench_wcomp.jsonl | cut -c1-300
