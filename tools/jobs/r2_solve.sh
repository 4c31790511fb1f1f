python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_xweights.py -q -s > gpurun_out/sv_xw.log 2>&1; echo xw=$?
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/sv_tests.log 2>&1; echo tests=$?
for mode in inverse panel; do
  WC_SOLVE=$mode timeout 120 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-variants --no-exact > gpurun_out/sv_bench_headline_$mode.json 2>/dev/null; echo $mode headline=$?
  WC_SOLVE=$mode timeout 180 python bench.py --config llm32k --r 1024 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-variants --no-exact > gpurun_out/sv_bench_llm_$mode.json 2>/dev/null; echo $mode llm=$?
done
