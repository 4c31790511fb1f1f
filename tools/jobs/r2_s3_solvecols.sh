# session 3: weights solve with 2 vs 8 RHS columns per CTA (headline)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in 2 8 2 8; do
  WC_SOLVE_COLS=$c timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-variants --no-exact 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('cols=$c', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['stages_ms'].items()})"
done
