python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_nshard.py -q -x > gpurun_out/nsb_tests.log 2>&1; echo nsb=$?
for b in 1 16; do
  timeout 300 python bench.py --config long256k --mode nshard --block $b --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-exact > gpurun_out/nsb_long256k_b$b.json 2> gpurun_out/nsb_long256k_b$b.err; echo long b$b=$?
done
