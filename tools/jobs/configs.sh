# the other BASELINE configs on one GPU (parity-test shapes), blocked b=16 and sequential b=1
for c in vit diffusion llm32k cfg1; do
  for b in 16 1; do
    timeout 600 python bench.py --config $c --block $b --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/cfg_${c}_b${b}.json 2> gpurun_out/cfg_${c}_b${b}.err; echo $c b$b=$?
  done
done
