#!/bin/bash
mkdir -p gpurun_out
for c in "$@"; do
  timeout 900 python bench.py --config $c --steps 16 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err
  echo "cfg$c rc=$?"; tail -c 1500 gpurun_out/bench_cfg$c.json; tail -5 gpurun_out/bench_cfg$c.err
done
