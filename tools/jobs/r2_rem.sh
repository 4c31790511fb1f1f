python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_binned.py tests/test_gpu_kvcache.py -q -x > gpurun_out/rem_tests.log 2>&1; echo rem=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/rem_all.log 2>&1; echo all=$?
