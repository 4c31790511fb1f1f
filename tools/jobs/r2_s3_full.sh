# session 3: build, smoke, full GPU suite, headline bench + trace
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke=$?
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-variants --no-exact > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err; echo bench=$?
WC_SELECT_TRACE=1 timeout 300 python tools/trace_blocked.py 16 > /dev/null 2> gpurun_out/q_trace.txt; echo trace=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/f_gputests.log 2>&1; echo tests=$?
tail -3 gpurun_out/f_gputests.log
