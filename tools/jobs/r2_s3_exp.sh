# session 3 experiment: full-sector quad writes (wrong values in rows < i of the first quad; timing only)
WC_NVCC_EXTRA="-DWC_EXP_FULLQ" python -c "from paper_2602_10056_b200 import build as b; b.build(force=True)" > /dev/null 2>&1; echo build=$?
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-variants --no-exact > gpurun_out/x_bench.json 2> gpurun_out/x_bench.err; echo bench=$?
WC_SELECT_TRACE=1 timeout 300 python tools/trace_blocked.py 16 > /dev/null 2> gpurun_out/x_trace.txt; echo trace=$?
