python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_blocked.py -q -k "fp32_d128" > gpurun_out/k_fp32.log 2>&1; echo fp32=$?
WC_DEBUG_SYNC=1 timeout 300 python -c "
import os, sys, torch
sys.path.insert(0, os.getcwd())
from wc_harness import run_gpu, qkv
" > /dev/null 2>&1
cd tests && WC_DEBUG_SYNC=1 timeout 300 python -c "
import torch
from wc_harness import run_gpu, qkv
Q, K, V = qkv(1, 2, 1, 100, 3000, 128, 'f32', 'G', seed=13)
print(run_gpu(Q, K, V, 40, 13, block=16)[1])
" > ../gpurun_out/k_fp32_dbg.log 2>&1; cd ..
timeout 1200 python -m pytest tests/test_gpu_blocked.py -q > gpurun_out/k_blocked.log 2>&1; echo blocked_tests=$?
for b in 16 32; do
  timeout 600 python bench.py --block $b --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-variants --no-exact > gpurun_out/k_bench_b${b}.json 2> gpurun_out/k_bench_b${b}.err; echo bench b$b=$?
  WC_SELECT_TRACE=1 timeout 300 python tools/trace_blocked.py $b > /dev/null 2> gpurun_out/k_trace_b$b.txt
done
