#!/bin/bash
# ncu evidence for the round: launch list of a short bench + full captures of the top kernels.
mkdir -p gpurun_out
export NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  > gpurun_out/launches_bench.log 2>&1
echo "launches rc=$?"
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemv_bf16_kernel -s 400 -c 3 \
  -o gpurun_out/prof_gemv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/prof_gemv.log 2>&1
echo "gemv rc=$?"
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemm_bf16_tcgen05 -s 20 -c 2 \
  -o gpurun_out/prof_gemm python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/prof_gemm.log 2>&1
echo "gemm rc=$?"
ls -la gpurun_out
