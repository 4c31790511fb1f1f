# session 3: A/B (A = last commit, B = tree) + the weights/select GPU tests of the tree
bash tools/ab.sh 3 > gpurun_out/ab.txt 2>&1; echo ab=$?
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/ab_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/ab_tests.log
