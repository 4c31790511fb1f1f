# session 3: ncu --set full (source-level) of the non-selection kernels at the headline
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"weights_solve|weights_reduce|prologue|attend_ws|weights_tc" -s 8 -c 9 -o gpurun_out/s3_small python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-exact --no-variants > gpurun_out/s3_small.log 2>&1; echo ncu=$?
