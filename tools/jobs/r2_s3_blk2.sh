# session 3: block size sweep with the rejection CTA (headline)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for b in 16 20 24 32 16; do
  timeout 300 python bench.py --block $b --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-variants --no-exact 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('b=$b', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['stages_ms'].items()}, d['selection']['blocks_per_unit'])"
done
