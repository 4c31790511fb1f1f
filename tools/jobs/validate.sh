set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/j1_smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/j1_gputests.log 2>&1; echo tests=$?
timeout 600 python bench.py > gpurun_out/j1_bench.json 2> gpurun_out/j1_bench.err; echo bench=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rpc_select_blocked -s 1 -c 1 -o gpurun_out/j1_blocked python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-exact --no-variants > gpurun_out/j1_ncu.log 2>&1; echo ncu=$?
