python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
WC_DEBUG_SYNC=1 timeout 120 python tools/case_gather.py 16 > gpurun_out/c16.log 2>&1; echo c16=$?
WC_DEBUG_SYNC=1 timeout 120 python tools/case_gather.py 8 > gpurun_out/c8.log 2>&1; echo c8=$?
timeout 300 compute-sanitizer --tool memcheck python tools/case_gather.py 16 > gpurun_out/c16_mem.log 2>&1; echo mem=$?
