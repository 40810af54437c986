#!/bin/bash
# Round-2 ncu evidence: full captures of the hot kernels (final build) + the launch list of
# the headline bench's decode steps. Summaries -> gpurun_out/ncu/summary.jsonl
mkdir -p gpurun_out/ncu
NCU=/usr/local/cuda/bin/ncu
for t in gemv_bf16:gemv_tma_kernel gemv_coded:gemv_tma_kernel gemv_tc_bf16:gemv_tc_kernel gemv_tc_coded:gemv_tc_kernel \
         hx_expand:hx_expand moe_coded:moe_ attn_tc:attn_prefill_tc; do
  name=${t%%:*}; k=${t##*:}
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/ncu/r02_$name python tools/ncu_targets.py $name > gpurun_out/ncu/$name.log 2>&1
  echo "$name rc=$?"
done
for f in gpurun_out/ncu/*.ncu-rep; do python tools/ncu_summary.py $f; done > gpurun_out/ncu/summary.jsonl 2>&1
cut -c1-300 gpurun_out/ncu/summary.jsonl
