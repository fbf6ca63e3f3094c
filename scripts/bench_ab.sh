# bench.py A/B: in-tree build ("head") vs ab_libs/<variant>, interleaved: bash scripts/bench_ab.sh R variant...
R=$1; shift
LIB=paper_2402_09222_b200/libomcg.so
cp $LIB /tmp/libomcg_head.so
for r in $(seq $R); do
  for v in head "$@"; do
    if [ $v = head ]; then cp /tmp/libomcg_head.so $LIB; else cp ab_libs/$v/libomcg.so $LIB; fi
    timeout 600 python bench.py 2>/dev/null | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('$v', round(l['value']/1e6,3), round(l['e2e']['value']/1e6,3))"
  done
done
cp /tmp/libomcg_head.so $LIB
