python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_blocked.py -q > gpurun_out/g_blocked.log 2>&1; echo blocked_tests=$?
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-variants --no-exact > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err; echo bench=$?
WC_SELECT_TRACE=1 timeout 300 python tools/trace_blocked.py 16 > /dev/null 2> gpurun_out/g_trace.txt; echo trace=$?
