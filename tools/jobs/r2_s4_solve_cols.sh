# session 4: columns per CTA of the row-parallel solve (headline, llm32k): stage times per C
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for cfg in headline llm32k; do for C in 1 2 4 8; do
  echo "$cfg C=$C $(WC_SOLVE_COLS=$C timeout 300 python bench.py --config $cfg --block 16 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-variants --no-exact 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['stages_ms'].items()})")"
done; done > gpurun_out/solve_cols.txt 2>&1
