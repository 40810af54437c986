#!/bin/bash
# coded GEMV A/B (16 vs 8 consumer warps), engine + replica + full-size parity, headline bench
mkdir -p gpurun_out/parity
timeout 300 python tools/bench_wcomp.py > gpurun_out/wcomp_c16.jsonl 2>&1
PSHARD_LIB=$PWD/paper_2604_26334_b200/_lib/c8/libpshard.so timeout 300 python tools/bench_wcomp.py > gpurun_out/wcomp_c8.jsonl 2>&1
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -p no:cacheprovider -k "gemv" 2>&1 > gpurun_out/k4.log
timeout 1200 python -m pytest tests/test_engine_gpu.py tests/test_replicas_gloo.py -q -m gpu -p no:cacheprovider 2>&1 > gpurun_out/e4.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke4.log 2>&1
PS_PARITY_DIR=gpurun_out/parity timeout 3000 python -m pytest tests/test_full_size_gpu.py -q -m gpu -p no:cacheprovider --durations=0 2>&1 > gpurun_out/f4.log
timeout 1200 python bench.py > gpurun_out/bench4.json 2> gpurun_out/bench4.err
for f in k4 e4 f4; do echo "== $f"; grep -E "^E  |^FAILED|passed|failed" gpurun_out/$f.log | cut -c1-600 | head -30; done
tail -2 gpurun_out/smoke4.log; for f in c16 c8; do echo == $f; cut -c1-260 gpurun_out/wcomp_$f.jsonl; done
cat gpurun_out/parity/*.json; echo; tail -c 1500 gpurun_out/bench4.json; tail -5 gpurun_out/bench4.err
