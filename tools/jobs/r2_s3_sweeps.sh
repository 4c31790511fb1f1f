# session 3: long-sequence single-GPU blocked path, ViT with the ILV flag, and the LLM n x r sweep
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in long256k long1m long4m; do
  timeout 600 python bench.py --config $c --mode units --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-exact --no-variants > gpurun_out/w_long_${c}_units.json 2> gpurun_out/w_long_${c}_units.err; echo $c units=$?
done
timeout 600 python bench.py --config vit --block 16 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/w_cfg_vit.json 2> gpurun_out/w_cfg_vit.err; echo vit=$?
for n in 32768 65536 131072; do for r in 256 512 1024; do
  timeout 600 python bench.py --config llm32k --n $n --r $r --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/w_llm_n${n}_r${r}.json 2> gpurun_out/w_llm_n${n}_r${r}.err; echo llm $n $r=$?
done; done
