# session 4 final: smoke, default bench, launch list of HEAD
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/g_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err; echo bench=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-exact --no-variants > /dev/null 2>&1; echo launches=$?
