#!/bin/bash
# Round-2 ncu evidence: full captures of the hot kernels + launch list of the headline bench.
mkdir -p gpurun_out/ncu
NCU=/usr/local/cuda/bin/ncu
for t in gemv_bf16:gemv_tma_kernel gemv_coded:gemv_tma_kernel gemv_tc_bf16:gemv_tc_kernel gemv_tc_coded:gemv_tc_kernel \
         moe_coded:moe_ timing attn_tc:attn_prefill_tc expand:expand_coded; do
  name=${t%%:*}; k=${t##*:}
  [ "$name" = "timing" ] && continue
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/ncu/r02_$name python tools/ncu_targets.py $name > gpurun_out/ncu/$name.log 2>&1
  echo "$name rc=$?"
done
timeout 1200 $NCU --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/ncu/r02_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  --no-plan-faithful > gpurun_out/ncu/launches_bench.log 2>&1
echo "launches rc=$?"
for f in gpurun_out/ncu/*.ncu-rep; do python tools/ncu_summary.py $f; done > gpurun_out/ncu/summary.jsonl 2>&1
cut -c1-400 gpurun_out/ncu/summary.jsonl
