# session 3: blocked selection at b = 16 / 24 / 32 (bench + per-block trace) on the rebuilt tree
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s3_smoke.log 2>&1; echo smoke=$?
for b in 16 24 32; do
  timeout 300 python bench.py --block $b --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-variants --no-exact > gpurun_out/s3_bench_b${b}.json 2> gpurun_out/s3_bench_b${b}.err; echo bench b$b=$?
  WC_SELECT_TRACE=1 timeout 300 python tools/trace_blocked.py $b > /dev/null 2> gpurun_out/s3_trace_b$b.txt; echo trace b$b=$?
done
