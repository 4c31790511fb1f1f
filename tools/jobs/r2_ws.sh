python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_xweights.py -q -s > gpurun_out/xw.log 2>&1; echo xw=$?
WC_ATTEND=ws timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x > gpurun_out/ws_parity.log 2>&1; echo parity=$?
for r in 256 1024; do
  WC_ATTEND=ws timeout 180 python bench.py --config llm32k --r $r --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-variants --no-exact > gpurun_out/ws_bench_llm_r$r.json 2> gpurun_out/ws_bench_llm_r$r.err; echo ws llm r$r=$?
done
WC_ATTEND=ws timeout 120 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-variants --no-exact > gpurun_out/ws_bench_headline.json 2> gpurun_out/ws_bench_headline.err; echo ws headline=$?
timeout 120 python bench.py --config diffusion --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-variants --no-exact > gpurun_out/tc_bench_diff.json 2>&1; echo tc diff=$?
WC_ATTEND=ws timeout 120 python bench.py --config diffusion --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-variants --no-exact > gpurun_out/ws_bench_diff.json 2>&1; echo ws diff=$?
