# A/B timing on one box: variant A = abtest/A_csrc, variant B = the tree's csrc; each built in its own
# copy of the repo, benched alternately (headline, select-stage ms).  usage: bash tools/ab.sh [rounds] [bench args]
R=${1:-3}; shift
ARGS=${@:---steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-variants --no-exact}
for v in A B; do
  rm -rf /tmp/ab$v && mkdir -p /tmp/ab$v && cp -r bench.py __graft_entry__.py oracle paper_2602_10056_b200 include /tmp/ab$v/
  rm -f /tmp/ab$v/paper_2602_10056_b200/libwildcat.so
  [ $v = A ] && rm -rf /tmp/abA/paper_2602_10056_b200/csrc && cp -r abtest/A_csrc /tmp/abA/paper_2602_10056_b200/csrc
  (cd /tmp/ab$v && python -c "from paper_2602_10056_b200 import build as b; b.build(force=True)" > /dev/null 2>&1) || echo "build $v failed"
done
for r in $(seq $R); do
  for v in A B; do
    (cd /tmp/ab$v && timeout 300 python bench.py $ARGS 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('$v', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['stages_ms'].items()}, d.get('clocks',{}).get('sm_mhz'))")
  done
done
