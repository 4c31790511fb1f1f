# session 3: ncu --set full of the blocked selection kernel at the headline (source-level stalls)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rpc_select_blocked -s 1 -c 1 -o gpurun_out/s3_select python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-exact --no-variants > gpurun_out/s3_ncu.log 2>&1; echo ncu=$?
