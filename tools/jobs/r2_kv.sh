python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_kvcache.py tests/test_gpu_binned.py -q -x > gpurun_out/kv_tests.log 2>&1; echo kv=$?
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/kv_bench.json 2> gpurun_out/kv_bench.err; echo bench=$?
