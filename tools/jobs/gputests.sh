# full GPU test suite, KV tests first (verbose), with a per-call limit
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_kvcache.py -x -q -m gpu > gpurun_out/kv_tests.log 2>&1; echo kv=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo all=$?
