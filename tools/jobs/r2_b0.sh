# round-2 baseline on a fresh box: smoke, GPU tests, default bench, launch list
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/b0_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/b0_gputests.log 2>&1; echo tests=$?
timeout 600 python bench.py > gpurun_out/b0_bench.json 2> gpurun_out/b0_bench.err; echo bench=$?
