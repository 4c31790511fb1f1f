# warp-specialised attend: parity with WC_ATTEND=ws, then timing vs the default path
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
WC_ATTEND=ws timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "vit or diffusion or ragged or large or headline or llm" > gpurun_out/ws_parity.log 2>&1; echo parity=$?
for cfg in headline; do
  WC_ATTEND=ws timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/ws_bench_$cfg.json 2> gpurun_out/ws_bench_$cfg.err; echo ws $cfg=$?
done
for r in 256 1024; do
  WC_ATTEND=ws timeout 600 python bench.py --config llm32k --r $r --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/ws_bench_llm_r$r.json 2> gpurun_out/ws_bench_llm_r$r.err; echo ws llm r$r=$?
done
