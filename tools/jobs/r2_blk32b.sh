python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_blocked.py -q -x > gpurun_out/k_blocked.log 2>&1; echo blocked_tests=$?
trace() {
  WC_SELECT_TRACE=1 timeout 300 python -c "
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2602_10056_b200 as wc
from paper_2602_10056_b200.inputs import make_qkv
Q, K, V = make_qkv(1, 1, 1, 65536, 65536, 128, 'bf16', 'G', 0)
dev = torch.device('cuda:0')
sel = wc.select(Q.to(dev), K.to(dev), 256, seed=0, block=$1)
torch.cuda.synchronize()
print('stats', sel.stats[0, :10].tolist(), file=sys.stderr)
" > /dev/null 2> gpurun_out/k_trace_b$1$2.txt
}
for keep in 0; do
for b in 16 32; do
  WC_BLK_L2_KEEP_FRAC=$keep timeout 600 python bench.py --block $b --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-variants --no-exact > gpurun_out/k_bench_b${b}_k$keep.json 2> gpurun_out/k_bench_b${b}_k$keep.err; echo bench b$b keep$keep=$?
done
done
trace 16; trace 32
