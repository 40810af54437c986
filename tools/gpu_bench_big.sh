#!/bin/bash
mkdir -p gpurun_out
free -g | head -2
for c in "$@"; do
  timeout 1200 python bench.py --config $c --steps 8 --warmup 2 --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err
  echo "cfg$c rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_cfg$c.json'))
print({k: d[k] for k in ('value','ms_per_step','ttft_ms','model_load_s')}, d['roofline']['frac'], d['roofline']['achieved'], d['e2e']['value'], d.get('prefill_passes'))" 2>&1 | tail -3; tail -4 gpurun_out/bench_cfg$c.err
done
