# session 3 round-end evidence: smoke, full GPU suite, default bench, reference arm, launch list, ncu
# captures (select, weights, attend), trace, sanitizers on the blocked case, config + long sweeps
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/e_smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/e_gputests.log 2>&1; echo tests=$?
timeout 900 python bench.py > gpurun_out/e_bench.json 2> gpurun_out/e_bench.err; echo bench=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/e_ref.json 2> gpurun_out/e_ref.err; echo ref=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/e_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-exact --no-variants > gpurun_out/e_launch_bench.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rpc_select_blocked -s 1 -c 1 -o gpurun_out/e_select python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-exact --no-variants > /dev/null 2>&1; echo ncu_select=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:weights_tc_kernel -s 1 -c 1 -o gpurun_out/e_weights python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-exact --no-variants > /dev/null 2>&1; echo ncu_weights=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attend_ws_kernel -s 1 -c 1 -o gpurun_out/e_attend python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-exact --no-variants > /dev/null 2>&1; echo ncu_attend=$?
WC_SELECT_TRACE=1 timeout 300 python tools/trace_blocked.py 16 > /dev/null 2> gpurun_out/e_trace.txt; echo trace=$?
CS=/usr/local/cuda/bin/compute-sanitizer
for t in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $t --print-limit 20 python tools/sanitize_case.py blocked > gpurun_out/e_san_${t}_blocked.log 2>&1; echo $t blocked=$?
done
for c in vit diffusion llm32k cfg1; do
  timeout 600 python bench.py --config $c --block 16 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/e_cfg_${c}.json 2> gpurun_out/e_cfg_${c}.err; echo $c=$?
done
for c in long256k long1m long4m; do
  timeout 600 python bench.py --config $c --mode replicas --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-exact --no-variants > gpurun_out/e_long_${c}_blocked.json 2> gpurun_out/e_long_${c}_blocked.err; echo $c blocked=$?
  timeout 600 python bench.py --config $c --block 16 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-exact > gpurun_out/e_long_${c}_nshard.json 2> gpurun_out/e_long_${c}_nshard.err; echo $c nshard=$?
done
