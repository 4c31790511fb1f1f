# session 4: compute-sanitizer memcheck / racecheck / synccheck of the final kernels (blocked selection with
# the keyless rejection CTA + relay at n = 16K, 64 CTAs per unit; ViT contiguous slices; cfg1; binned; KV)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
mkdir -p gpurun_out/san
CS=/usr/local/cuda/bin/compute-sanitizer
for c in blocked vit cfg1 binned kv longr finite; do
  for t in memcheck racecheck synccheck; do
    timeout 900 $CS --tool $t --print-limit 20 python tools/sanitize_case.py $c > gpurun_out/san/san_${t}_${c}.log 2>&1; echo $t $c=$?
  done
done
