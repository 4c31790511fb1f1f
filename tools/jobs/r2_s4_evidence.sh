# session 4 round-end evidence (row-parallel solve): smoke, full GPU suite, default bench, launch list,
# ncu of the new solve kernel, config lines and the LLM r = 256 rows
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/f_gputests.log 2>&1; echo tests=$?
timeout 900 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo bench=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-exact --no-variants > gpurun_out/f_launch_bench.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:weights_solve_rows -s 1 -c 1 -o gpurun_out/f_solve python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-exact --no-variants > /dev/null 2>&1; echo ncu_solve=$?
for c in vit diffusion llm32k cfg1; do
  timeout 600 python bench.py --config $c --block 16 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/f_cfg_${c}.json 2> gpurun_out/f_cfg_${c}.err; echo $c=$?
done
for n in 65536 131072; do
  timeout 600 python bench.py --config llm32k --n $n --r 256 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/f_llm_n${n}_r256.json 2> gpurun_out/f_llm_n${n}_r256.err; echo llm $n=$?
done
timeout 600 python bench.py --config long256k --mode units --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-exact --no-variants > gpurun_out/f_long256k_units.json 2> gpurun_out/f_long256k_units.err; echo long256k=$?
