# session 3: A/B headline + vit (A = last commit, B = tree), then the blocked tests of the tree
bash tools/ab.sh 2 > gpurun_out/ab2.txt 2>&1
bash tools/ab.sh 2 --config vit --block 16 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-variants --no-exact >> gpurun_out/ab2.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_blocked.py tests/test_gpu_parity.py -q -x > gpurun_out/ab2_tests.log 2>&1; echo tests=$?
tail -1 gpurun_out/ab2_tests.log
