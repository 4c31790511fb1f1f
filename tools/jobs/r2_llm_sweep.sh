# LLM KV-cache shapes (BASELINE configs[3]): n in {32K, 64K, 128K} x r in {256, 512, 1024}, GQA 32/8, d = 128
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for n in 32768 65536 131072; do
  for r in 256 512 1024; do
    timeout 900 python bench.py --config llm32k --n $n --r $r --steps 3 --warmup 3 --no-cpu-baseline --no-variants --no-e2e > gpurun_out/llm_n${n}_r${r}.json 2> gpurun_out/llm_n${n}_r${r}.err; echo n$n r$r=$?
  done
done
# tensor-pipe utilisation of the streamed attend at r = 1024
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attend_tc -s 1 -c 1 -o gpurun_out/ncu_attend_r1024 python bench.py --config llm32k --r 1024 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-exact --no-variants > gpurun_out/ncu_attend_r1024.log 2>&1; echo ncu_attend=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:weights_tc -s 1 -c 1 -o gpurun_out/ncu_weights_r1024 python bench.py --config llm32k --r 1024 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-exact --no-variants > gpurun_out/ncu_weights_r1024.log 2>&1; echo ncu_weights=$?
