# session 3 final evidence (after the write-out change): GPU suite, default bench, reference arm,
# launch list, ncu select, trace, config sweep
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/e_smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/e_gputests.log 2>&1; echo tests=$?
timeout 900 python bench.py > gpurun_out/e_bench.json 2> gpurun_out/e_bench.err; echo bench=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/e_ref.json 2> gpurun_out/e_ref.err; echo ref=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/e_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-exact --no-variants > gpurun_out/e_launch_bench.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rpc_select_blocked -s 1 -c 1 -o gpurun_out/e_select python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-exact --no-variants > /dev/null 2>&1; echo ncu_select=$?
WC_SELECT_TRACE=1 timeout 300 python tools/trace_blocked.py 16 > /dev/null 2> gpurun_out/e_trace.txt; echo trace=$?
for c in vit diffusion llm32k cfg1; do
  timeout 600 python bench.py --config $c --block 16 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/e_cfg_${c}.json 2> gpurun_out/e_cfg_${c}.err; echo $c=$?
done
for c in long256k long1m long4m; do
  timeout 600 python bench.py --config $c --mode units --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-exact --no-variants > gpurun_out/e_long_${c}_units.json 2> gpurun_out/e_long_${c}_units.err; echo $c units=$?
done
