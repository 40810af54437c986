#!/bin/bash
# new kernels (one-pass tcgen05 GEMV, coded MoE) + engine tests + configs 3/4 benches
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -p no:cacheprovider -k "gemv_tc or coded" 2>&1 > gpurun_out/k5.log
timeout 1200 python -m pytest tests/test_engine_gpu.py -q -m gpu -p no:cacheprovider -k "batched or moe or coded or paged" 2>&1 > gpurun_out/e5.log
timeout 300 python tools/bench_wcomp.py > gpurun_out/wcomp5.jsonl 2>&1
timeout 1500 python bench.py --config 4 --no-cpu-baseline --no-plan-faithful > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
timeout 1500 python bench.py --config 3 --no-cpu-baseline --no-plan-faithful > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
for f in k5 e5; do echo "== $f"; grep -E "^E  |^FAILED|passed|failed" gpurun_out/$f.log | cut -c1-600 | head -30; done
cut -c1-300 gpurun_out/wcomp5.jsonl
for c in 4 3; do echo "== cfg$c"; python -c "
import json,sys
d=json.loads(open('gpurun_out/bench_cfg$c.json').read().strip().splitlines()[-1])
print({k:d.get(k) for k in ('value','ms_per_step','ttft_ms','link_format')}); print(d['roofline']); print(d.get('e2e'))
" 2>&1 | tail -4; tail -3 gpurun_out/bench_cfg$c.err; done
