#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -m gpu -p no:cacheprovider 2>&1 > gpurun_out/k7.log
timeout 1200 python -m pytest tests/test_engine_gpu.py tests/test_replicas_gloo.py -q -m gpu -p no:cacheprovider 2>&1 > gpurun_out/e7.log
timeout 300 python tools/bench_wcomp.py > gpurun_out/wcomp7.jsonl 2>&1
timeout 600 python bench.py --config 1 --no-plan-faithful > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
for f in k7 e7; do echo "== $f"; grep -E "^E  |^FAILED|passed|failed" gpurun_out/$f.log | cut -c1-400 | head -30; done
cut -c1-300 gpurun_out/wcomp7.jsonl
python -c "
import json
d=json.loads(open('gpurun_out/bench_cfg1.json').read().strip().splitlines()[-1])
print({k:d.get(k) for k in ('value','ms_per_step','ttft_ms')}); print(d['roofline']); print(d.get('e2e'))
" 2>&1 | tail -4; tail -3 gpurun_out/bench_cfg1.err
