# long-sequence sweep on one GPU: n-sharded path (world 1, NCCL) and the single-GPU blocked path
for c in long256k long1m long4m; do
  timeout 600 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-exact > gpurun_out/long_${c}_nshard.json 2> gpurun_out/long_${c}_nshard.err; echo $c nshard=$?
  timeout 600 python bench.py --config $c --mode replicas --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-exact --no-variants > gpurun_out/long_${c}_blocked.json 2> gpurun_out/long_${c}_blocked.err; echo $c blocked=$?
done
