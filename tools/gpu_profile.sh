#!/bin/bash
# ncu evidence for the round: launch list of a short bench + full captures of the top kernels.
mkdir -p gpurun_out
export NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  > gpurun_out/launches_bench.log 2>&1
echo "launches rc=$?"
# the bench's kernel-roofline launch (K1 bulk-copy GEMV, SwiGLU epilogue, 28672 x 4096)
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemv_tma_kernel -s 2 -c 1 \
  -o gpurun_out/prof_gemv_tma python tools/gemv_one.py 28672 4096 1 0 2 > gpurun_out/prof_gemv.log 2>&1
echo "gemv rc=$?"
# GEMV launches inside a decode pass (ring pieces)
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemv_tma_kernel -s 600 -c 3 \
  -o gpurun_out/prof_gemv_pass python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/prof_gemv_pass.log 2>&1
echo "gemv pass rc=$?"
# prefill GEMM (CTA-pair tcgen05 kernel) inside the config-4 prefill
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:gemm_bf16_pair -s 8 -c 4 \
  -o gpurun_out/prof_gemm python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/prof_gemm.log 2>&1
echo "gemm rc=$?"
ls -la gpurun_out
