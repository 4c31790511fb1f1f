# full GPU suite + sanitizer re-run on the fixed handshakes / commits
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/c_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/c_gputests.log 2>&1; echo tests=$?
CS=/usr/local/cuda/bin/compute-sanitizer
export CUDA_MODULE_LOADING=EAGER
for c in cfg1 vit blocked longr binned kv finite; do
  for t in memcheck racecheck synccheck; do
    timeout 900 $CS --tool $t --print-limit 10 python tools/sanitize_case.py $c > gpurun_out/san_${t}_${c}.log 2>&1; echo $t $c=$?
  done
done
