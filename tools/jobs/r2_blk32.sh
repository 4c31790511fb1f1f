# blocked selection, 16- and 32-slot plans: parity, racecheck, bench at the headline
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_blocked.py tests/test_gpu_options.py -q -x > gpurun_out/k_blocked.log 2>&1; echo blocked_tests=$?
for b in 16 32; do
  timeout 600 python bench.py --block $b --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/k_bench_b$b.json 2> gpurun_out/k_bench_b$b.err; echo bench b$b=$?
  WC_SELECT_TRACE=1 timeout 300 python -c "
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2602_10056_b200 as wc
from paper_2602_10056_b200.inputs import make_qkv
Q, K, V = make_qkv(1, 1, 1, 65536, 65536, 128, 'bf16', 'G', 0)
dev = torch.device('cuda:0')
sel = wc.select(Q.to(dev), K.to(dev), 256, seed=0, block=$b)
torch.cuda.synchronize()
print('stats', sel.stats[0, :10].tolist(), file=sys.stderr)
" > /dev/null 2> gpurun_out/k_trace_b$b.txt; echo trace=$?
done
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --print-limit 10 python tools/sanitize_case.py blocked > gpurun_out/k_race_blocked.log 2>&1; echo race=$?
