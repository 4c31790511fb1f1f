# session 4: A/B of the tensor-memory F-row cache in the blocked selection (A = last commit, B = tree),
# headline and LLM 32K; then the blocked / parity GPU tests of the tree and a trace
bash tools/ab.sh 3 > gpurun_out/ab_tmem.txt 2>&1
bash tools/ab.sh 1 --config llm32k --block 16 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-variants --no-exact >> gpurun_out/ab_tmem.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_blocked.py tests/test_gpu_parity.py -q -x > gpurun_out/ab_tmem_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/ab_tmem_tests.log
WC_SELECT_TRACE=1 timeout 300 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-variants --no-exact > /dev/null 2> gpurun_out/trace_bulk.txt
grep btrace gpurun_out/trace_bulk.txt | tail -4
