# session 4: A/B of the reduce with 32 loads in flight and the division-free Dinv chain (A = last commit, B = tree): headline, llm32k, long256k;
# every GPU test; launch list
bash tools/ab.sh 3 > gpurun_out/ab_dinv.txt 2>&1
bash tools/ab.sh 1 --config llm32k --block 16 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-variants --no-exact >> gpurun_out/ab_dinv.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/ab_dinv_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/ab_dinv_tests.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/dinv_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-exact --no-variants > /dev/null 2>&1; echo ncu=$?
