# session 3: HostPipeline parity + the default bench line
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "host" > gpurun_out/p_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/p_tests.log
timeout 900 python bench.py > gpurun_out/p_bench.json 2> gpurun_out/p_bench.err; echo bench=$?
