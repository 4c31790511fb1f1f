# session 3 quick loop: build, blocked-selection parity, headline bench + per-block trace
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/q_smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests/test_gpu_blocked.py -q -x > gpurun_out/q_blocked.log 2>&1; echo blocked=$?
tail -2 gpurun_out/q_blocked.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-variants --no-exact > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err; echo bench=$?
WC_SELECT_TRACE=1 timeout 300 python tools/trace_blocked.py 16 > /dev/null 2> gpurun_out/q_trace.txt; echo trace=$?
