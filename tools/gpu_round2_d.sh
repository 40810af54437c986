#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -p no:cacheprovider -k "gemv_tc or coded" 2>&1 > gpurun_out/k6.log
timeout 1200 python -m pytest tests/test_engine_gpu.py -q -m gpu -p no:cacheprovider 2>&1 > gpurun_out/e6.log
timeout 300 python tools/bench_wcomp.py > gpurun_out/wcomp6.jsonl 2>&1
timeout 1500 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
for f in k6 e6; do echo "== $f"; grep -E "^E  |^FAILED|passed|failed" gpurun_out/$f.log | cut -c1-600 | head -30; done
cut -c1-300 gpurun_out/wcomp6.jsonl
python -c "
import json
d=json.loads(open('gpurun_out/bench_cfg2.json').read().strip().splitlines()[-1])
print({k:d.get(k) for k in ('value','ms_per_step','ttft_ms')}); print(d['roofline']); print(d['kernel_roofline']); print(d.get('e2e')); print(d.get('plan_faithful')); print(d.get('vram')); print(d.get('ttft'))
" 2>&1 | tail -8; tail -3 gpurun_out/bench_cfg2.err
