# session 4: A/B of the K_S gather riding in the reduce_dinv launch (A = last commit, B = tree): headline, llm32k, long256k;
# every GPU test; launch list
bash tools/ab.sh 3 > gpurun_out/ab_gks.txt 2>&1
bash tools/ab.sh 1 --config llm32k --block 16 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-variants --no-exact >> gpurun_out/ab_gks.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/ab_gks_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/ab_gks_tests.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/gks_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-exact --no-variants > /dev/null 2>&1; echo ncu=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/gks_smoke.log 2>&1; echo smoke=$?
