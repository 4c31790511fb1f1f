# round-end evidence: GPU tests, smoke, default bench, reference arm, launch list, ncu captures
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/f_gputests.log 2>&1; echo tests=$?
timeout 900 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo bench=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f_ref.json 2> gpurun_out/f_ref.err; echo ref=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/f_launch_bench.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attend_tc_kernel -s 1 -c 1 -o gpurun_out/f_attend python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-exact --no-variants > /dev/null 2>&1; echo ncu_attend=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:weights_tc_kernel -s 1 -c 1 -o gpurun_out/f_weights python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-exact --no-variants > /dev/null 2>&1; echo ncu_weights=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rpc_select_blocked -s 1 -c 1 -o gpurun_out/f_select python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-exact --no-variants > /dev/null 2>&1; echo ncu_select=$?
WC_SELECT_TRACE=1 python tools/trace_blocked.py > gpurun_out/f_trace.txt 2>&1; echo trace=$?
