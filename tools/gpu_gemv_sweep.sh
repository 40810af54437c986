mkdir -p gpurun_out
timeout 200 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x -k gemv -p no:cacheprovider > gpurun_out/gemv_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/gemv_tests.log
for st in 4 6 8 10 12; do
  PS_GEMV_STAGES=$st timeout 200 python tools/bench_gemv.py > gpurun_out/bench_gemv_st$st.log 2>&1
  echo "stages=$st"; grep "\"rows\": 0" gpurun_out/bench_gemv_st$st.log | grep -v "296" | python3 -c "
import sys,json
print(' '.join(f\"{json.loads(l)['shape'].split()[0]}{json.loads(l)['shape'].split()[-1]}:{json.loads(l)['GBps']:.0f}\" for l in sys.stdin))"
done
