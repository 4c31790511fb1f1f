# GPU tests of the new options, then compute-sanitizer memcheck / racecheck / synccheck on small cases
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_options.py -q > gpurun_out/opt_tests.log 2>&1; echo opt_tests=$?
CS=/usr/local/cuda/bin/compute-sanitizer
for c in cfg1 vit blocked longr binned kv finite; do
  for t in memcheck racecheck synccheck; do
    timeout 900 $CS --tool $t --print-limit 20 python tools/sanitize_case.py $c > gpurun_out/san_${t}_${c}.log 2>&1; echo $t $c=$?
  done
done
