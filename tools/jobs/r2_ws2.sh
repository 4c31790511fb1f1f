python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/w_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/w_gputests.log 2>&1; echo tests=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attend_ws -s 1 -c 1 -o gpurun_out/ncu_attend_ws_r1024 python bench.py --config llm32k --r 1024 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-exact --no-variants > gpurun_out/ncu_ws.log 2>&1; echo ncu=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attend_ws -s 1 -c 1 -o gpurun_out/ncu_attend_ws_headline python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-exact --no-variants > gpurun_out/ncu_ws2.log 2>&1; echo ncu2=$?
