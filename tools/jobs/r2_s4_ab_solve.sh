# session 4: A/B of the row-parallel solve (weights_solve_rows_kernel) for r <= 256 (A = last commit,
# B = tree): headline, llm32k, diffusion, vit; then every GPU test of the tree
bash tools/ab.sh 3 > gpurun_out/ab_solve.txt 2>&1
for c in llm32k diffusion vit; do
  bash tools/ab.sh 1 --config $c --block 16 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-variants --no-exact >> gpurun_out/ab_solve.txt 2>&1
done
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/ab_solve_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/ab_solve_tests.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/solve_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-exact --no-variants > /dev/null 2>&1; echo ncu=$?
