#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --steps 8 --warmup 2 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "rc=$?"; tail -c 3000 gpurun_out/bench.json; tail -20 gpurun_out/bench.err
