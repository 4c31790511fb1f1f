# session 4: A/B of prologue pass 1 with the Q rows streamed in the K / V iterations (A = last commit,
# B = tree): headline, vit, llm32k; then every GPU test
bash tools/ab.sh 3 > gpurun_out/ab_pass1.txt 2>&1
for c in vit llm32k; do
  bash tools/ab.sh 1 --config $c --block 16 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-variants --no-exact >> gpurun_out/ab_pass1.txt 2>&1
done
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/ab_pass1_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/ab_pass1_tests.log
